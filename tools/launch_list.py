"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
python tools/launch_list.py gpurun_out/launches.csv profiles/r01_launches_config5.txt "<command>" """
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            v, u = float(d["Metric Value"].replace(",", "")), d["Metric Unit"]
            agg[d["Kernel Name"]].append(v / 1e6 if u == "ns" else (v / 1e3 if u in ("us", "usecond") else v))
tot = sum(sum(v) for v in agg.values())
out = [f"# ncu launch list: {sys.argv[3]}",
       "# gpu__time_duration.sum per launch, --clock-control none; cold-cache and serialised: compare SHARES", ""]
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    out.append("%6.2f%%  launches=%3d  mean=%10.3f ms  %s" % (100 * sum(v) / tot, len(v), sum(v) / len(v), k[:120]))
open(sys.argv[2], "w").write("\n".join(out) + "\n")
print("\n".join(out))
