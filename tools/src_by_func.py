"""Aggregate `ncu --page source --csv --print-source cuda,sass` line counts
by enclosing device function (executed warp-instructions, stall samples).
Usage: python tools/src_by_func.py gpurun_out/cfg5_src.csv.gz [rows]"""
import csv
import gzip
import io
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = sys.argv[1]
rows_n = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
data = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
rows = list(csv.reader(io.StringIO(data)))
per = {}
f = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0].isdigit() and len(r) > 7 and r[2] == "-":
        try:
            s, e = float(r[4] or 0), float(r[7] or 0)
        except ValueError:
            continue
        per.setdefault(f, {})[int(r[0])] = (s, e)
fn_re = re.compile(r"^(?:template\s*<[^>]*>\s*)?(?:__device__|__global__|static|inline|__host__)[^;{]*?\b([A-Za-z_]\w*)\s*\(")
tot_s = sum(s for d in per.values() for s, e in d.values()) or 1
tot_e = sum(e for d in per.values() for s, e in d.values()) or 1
agg = {}
for fpath, d in per.items():
    local = os.path.join(ROOT, "paper_2601_03159_b200", "csrc", os.path.basename(fpath))
    starts = []
    if os.path.exists(local):
        for i, line in enumerate(open(local), 1):
            m = fn_re.match(line.strip())
            if m and not line.startswith(" "):
                starts.append((i, m.group(1)))
    for ln, (s, e) in d.items():
        name = os.path.basename(fpath) + ":?"
        for i, nm in starts:
            if i <= ln:
                name = os.path.basename(fpath) + ":" + nm
        a = agg.setdefault(name, [0.0, 0.0])
        a[0] += s
        a[1] += e
print(f"total warp-instructions {tot_e:.4g} ({tot_e / rows_n:.0f} per row), stall samples {tot_s:.0f}")
for name, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:45]:
    print(f"{100 * e / tot_e:5.1f}% exec {e / rows_n:8.0f}/row   {100 * s / tot_s:5.1f}% stall   {name}")
