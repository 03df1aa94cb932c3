"""Per-launch table from an ncu --metrics CSV log: kernel, time, DRAM bytes, achieved GB/s.

    python tools/ncu_kernels.py launches.csv [name-regex]
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
hdr, launches = None, collections.OrderedDict()
scale = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0,
         "s": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if pat and not pat.search(d["Kernel Name"]):
        continue
    key = (d["ID"], d["Kernel Name"])
    v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
    launches.setdefault(key, {})[d["Metric Name"]] = v
tot_t = tot_b = 0.0
for (i, name), m in launches.items():
    t = m.get("gpu__time_duration.sum", 0.0)
    b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot_t += t
    tot_b += b
    short = re.sub(r"\(.*", "", name.replace("sbg::", "").replace("(anonymous namespace)::", ""))[:48]
    print(f"{i:>4} {short:48s} {t * 1e3:9.3f} ms {b / 1e9:8.3f} GB {b / t / 1e9 if t else 0:8.0f} GB/s")
print(f"total {tot_t * 1e3:.3f} ms, {tot_b / 1e9:.3f} GB, {tot_b / tot_t / 1e9 if tot_t else 0:.0f} GB/s")
