"""Source-line hotspots from `ncu --page source --csv --print-source cuda,sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
out = []; f = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r[0] in ("Function Name", "Line No"): continue
    if r[0].isdigit() and len(r) > 7 and r[2] == "-":
        try: s = float(r[4] or 0); e = float(r[7] or 0)
        except ValueError: continue
        out.append((s, e, f, int(r[0]), r[1][:90]))
tot = sum(o[0] for o in out) or 1; tote = sum(o[1] for o in out) or 1
print("stall samples %.0f, warp-instr executed %.3g" % (tot, tote))
agg = {}
for s, e, f, l, src in out:
    agg[f] = (agg.get(f, (0, 0))[0] + s, agg.get(f, (0, 0))[1] + e)
print({k: "%.1f%% / %.1f%%" % (100 * v[0] / tot, 100 * v[1] / tote) for k, v in agg.items()})
for s, e, f, l, src in sorted(out, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print("%5.1f%% samp %5.1f%% exec  %s:%d  %s" % (100 * s / tot, 100 * e / tote, f, l, src.strip()))
