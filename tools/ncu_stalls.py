"""Warp-stall samples of an ncu --set full report by SASS instruction: the top instructions with
their leading stall reasons, and the totals per reason for the instructions inside / outside the
address range that holds DMMAs (the DMMA warps' code vs the loader / scatter warps' code in K6).

    python tools/ncu_stalls.py report.ncu-rep [top_n]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
idx = {k: i for i, k in enumerate(h)}
rows = [x for x in r[2:] if len(x) >= len(h)]
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
S = lambda x: float(x[idx["Warp Stall Sampling (All Samples)"]] or 0)
tot = sum(S(x) for x in rows)
dm = [int(x[idx["Address"]], 16) for x in rows if "DMMA" in x[idx["Source"]]]
lo, hi = min(dm) - 0x800, max(dm) + 0x800
agg = {True: collections.Counter(), False: collections.Counter()}
for x in rows:
    inside = lo <= int(x[idx["Address"]], 16) <= hi
    for k in reasons:
        agg[inside][k[6:]] += float(x[idx[k]] or 0)
for inside in (True, False):
    s = sum(agg[inside].values())
    print(("DMMA-warp code" if inside else "other code    "), f"{s / tot:6.1%} of samples:",
          " ".join(f"{k}={v / tot:.1%}" for k, v in agg[inside].most_common(8)))
print("top instructions:")
for x in sorted(rows, key=S, reverse=True)[:top]:
    rs = sorted(((float(x[idx[k]] or 0), k[6:]) for k in reasons), reverse=True)[:3]
    print(f"{S(x) / tot:6.1%} {x[idx['Address']][-5:]:>6} {x[idx['Instructions Executed']]:>11} {x[idx['Source']][:58]:58s}",
          " ".join(f"{k}={v / tot:.1%}" for v, k in rs if v > 0))
