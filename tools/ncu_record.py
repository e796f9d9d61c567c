"""Record a full ncu capture's per-launch DRAM traffic and warp-instruction
count for a workload into profiles/ncu_traffic.json / ncu_instructions.json,
tagged with the hash of the library build that was profiled (bench.py marks
the issue roofline stale when the build changes).
Usage: python tools/ncu_record.py <report.ncu-rep> <key>   (key: config5, transforms, ...)"""
import csv
import hashlib
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, key = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
d, u = dict(zip(h, v)), dict(zip(h, units))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def num(k):
    return float(str(d.get(k, "0")).replace(",", "") or 0)


traffic = num("dram__bytes_read.sum") * scale.get(u.get("dram__bytes_read.sum"), 1) + \
    num("dram__bytes_write.sum") * scale.get(u.get("dram__bytes_write.sum"), 1)
ins = num("smsp__inst_executed.sum")
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (the build identity bench.py compares against: the kernel sources)

sha = bench.build_sha16()
for name, val in (("ncu_traffic.json", traffic), ("ncu_instructions.json", ins)):
    path = os.path.join(ROOT, "profiles", name)
    cur = json.load(open(path)) if os.path.exists(path) else {}
    cur[key] = {"value": val, "build_sha16": sha, "kernel": d.get("Kernel Name", ""),
                "source": f"ncu --set full ({os.path.basename(rep)})"} if name == "ncu_traffic.json" else \
        {"instructions": val, "build_sha16": sha, "kernel": d.get("Kernel Name", ""),
         "source": f"ncu --set full smsp__inst_executed.sum ({os.path.basename(rep)})"}
    json.dump(cur, open(path, "w"), indent=1)
print(json.dumps({"key": key, "traffic": traffic, "instructions": ins, "build_sha16": sha}))
