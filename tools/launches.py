"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(list)
for d in data:
    if d["Metric Name"] == "gpu__time_duration.sum":
        v = float(d["Metric Value"].replace(",", ""))
        if d["Metric Unit"] == "usecond": v *= 1e3
        if d["Metric Unit"] == "msecond": v *= 1e6
        agg[d["Kernel Name"][:70]].append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:70s} n={len(v):3d} mean={sum(v)/len(v)/1e3:11.1f} us  share={sum(v)/tot:6.1%}")
