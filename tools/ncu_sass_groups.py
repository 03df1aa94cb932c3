"""Group warp-stall samples of an ncu report by SASS opcode (and by source line if available)."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
r = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                                                capture_output=True, text=True).stdout)))
h = r[1]; idx = {k: i for i, k in enumerate(h)}
agg = collections.Counter(); cnt = collections.Counter()
tot = 0
for row in r[2:]:
    if len(row) < len(h):
        continue
    s = float(row[idx["Warp Stall Sampling (All Samples)"]] or 0)
    src = row[idx["Source"]].strip()
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    op = op.split(".")[0]
    agg[op] += s; cnt[op] += int(row[idx["Instructions Executed"]] or 0); tot += s
for op, s in agg.most_common(18):
    print(f"{op:10s} {s/tot:6.1%}  executed={cnt[op]}")
