"""Summarise an ncu --set full report into a committed text file (+ traffic json)."""
import csv, io, json, subprocess, sys
rep, out_txt, label = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v)); u = dict(zip(h, units))
def g(k, default=0.0):
    try: return float(d.get(k, default) or default)
    except ValueError: return default
keys = [k for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")]
tot = sum(g(k) for k in keys) or 1
dram = g("dram__bytes_read.sum") * (1e6 if u.get("dram__bytes_read.sum") == "Mbyte" else (1e9 if u.get("dram__bytes_read.sum") == "Gbyte" else 1))
dramw = g("dram__bytes_write.sum") * (1e6 if u.get("dram__bytes_write.sum") == "Mbyte" else (1e9 if u.get("dram__bytes_write.sum") == "Gbyte" else 1))
dur_ms = g("gpu__time_duration.sum") / (1e6 if u.get("gpu__time_duration.sum") == "ns" else (1e3 if u.get("gpu__time_duration.sum") == "us" else 1))
lines = [f"# ncu --set full summary: {label}", f"# report: {rep}", "",
         f"kernel                     {d.get('Kernel Name', '')}",
         f"duration                   {dur_ms:.3f} ms (under ncu, clocks not locked)",
         f"dram read + write          {dram/1e9:.3f} + {dramw/1e9:.3f} GB = {(dram+dramw)/1e9:.3f} GB per launch",
         f"dram throughput            {g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} % of peak",
         f"issue slots busy           {g('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} %",
         f"warps active / SM          {g('sm__warps_active.avg.per_cycle_active'):.1f}",
         f"registers / thread         {d.get('launch__registers_per_thread')}",
         f"block / grid               {d.get('launch__block_size')} / {d.get('launch__grid_size')}",
         f"dyn smem / block           {d.get('launch__shared_mem_per_block_dynamic')} {u.get('launch__shared_mem_per_block_dynamic','')}",
         f"fp64 pipe util             {g('sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'):.1f} %",
         f"warp-instructions executed {g('smsp__inst_executed.sum'):.4g}",
         "", "stall reasons (share of PC samples):"]
for k in sorted(keys, key=lambda k: -g(k))[:10]:
    lines.append(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100*g(k)/tot:5.1f} %")
open(out_txt, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
if len(sys.argv) > 4:
    tj = sys.argv[4]
    try: data = json.load(open(tj))
    except Exception: data = {}
    data[label.split()[0]] = dram + dramw
    json.dump(data, open(tj, "w"), indent=1)
