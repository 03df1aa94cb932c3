"""Top SASS instructions by warp-stall samples from an ncu report (needs -lineinfo)."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else None)
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kern:
    args += ["-k", kern]
r = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
h = r[1]; idx = {k: i for i, k in enumerate(h)}
rows = []
for row in r[2:]:
    if len(row) < len(h):
        continue
    try:
        s = float(row[idx["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    rows.append((s, row[idx["Address"]][-5:], row[idx["Source"]][:80], row[idx["Instructions Executed"]]))
tot = sum(x[0] for x in rows) or 1
for x in sorted(rows, reverse=True)[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print(f"{x[0]/tot:6.1%} {x[1]:>6} {x[3]:>12} {x[2]}")
