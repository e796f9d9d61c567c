"""Summarise an ncu source page (sass) CSV: hottest instruction regions."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
data = rows[2:]
def f(r, k):
    try: return float(r[ix[k]] or 0)
    except Exception: return 0.0
tot_exec = sum(f(r, "Instructions Executed") for r in data)
tot_samp = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print("total warp-instr executed %.3g, samples %.0f" % (tot_exec, tot_samp))
# windows of 32 instructions
W = int(sys.argv[2]) if len(sys.argv) > 2 else 48
best = []
for a in range(0, len(data), W):
    seg = data[a:a + W]
    e = sum(f(r, "Instructions Executed") for r in seg)
    s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in seg)
    best.append((s, e, a, seg))
best.sort(reverse=True)
for s, e, a, seg in best[:int(sys.argv[3]) if len(sys.argv) > 3 else 8]:
    print("---- instr %d..%d  samples %.1f%%  executed %.1f%%" % (a, a + W, 100 * s / tot_samp, 100 * e / tot_exec))
    for r in seg:
        if f(r, "Warp Stall Sampling (All Samples)") > 0.004 * tot_samp or f(r, "Instructions Executed") > 0.004 * tot_exec:
            print("   %-60s exec %8.0f samp %6.0f" % (r[ix["Source"]][:60], f(r, "Instructions Executed"), f(r, "Warp Stall Sampling (All Samples)")))
