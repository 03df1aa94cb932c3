"""Hot-loop statistics of one kernel in an object file: instruction mix and the sum of the encoded
stall counts (a lower bound of the cycles one warp needs per loop trip when it issues alone).

    python tools/sass_loop.py build/ab/sigma_ab_x.o 'k_sigma_ab_wsILi16ELi32ELb1ELb0ELi2'
"""
import collections
import re
import subprocess
import sys

obj, pat = sys.argv[1], sys.argv[2]
txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
ins, on = [], False
lines = txt.split("\n")
i = 0
while i < len(lines):
    l = lines[i]
    if "Function :" in l:
        on = pat in l
    m = re.match(r"\s*/\*([0-9a-f]{4,5})\*/\s+(.*?);\s*/\* (0x[0-9a-f]+) \*/", l) if on else None
    if m and i + 1 < len(lines):
        m2 = re.match(r"\s*/\* (0x[0-9a-f]+) \*/", lines[i + 1])
        if m2:
            ctrl = int(m2.group(1), 16) >> 41
            ins.append((int(m.group(1), 16), m.group(2).strip(), ctrl & 0xF))
            i += 2
            continue
    i += 1
idx = [k for k, x in enumerate(ins) if "DMMA" in x[1]]
clusters, cur = [], [idx[0]]
for k in idx[1:]:
    if k - cur[-1] < 80:
        cur.append(k)
    else:
        clusters.append(cur)
        cur = [k]
clusters.append(cur)
for c in clusters:
    end = c[-1]
    for j in range(end, min(end + 600, len(ins))):
        t = ins[j][1]
        m = re.search(r"BRA.*0x([0-9a-f]+)", t)
        if m and int(m.group(1), 16) <= ins[c[0]][0]:
            tgt = int(m.group(1), 16)
            start = next(k for k, x in enumerate(ins) if x[0] >= tgt)
            body = ins[start:j + 1]
            ops = collections.Counter()
            st = collections.Counter()
            for a, t2, s in body:
                op = re.sub(r"^@!?U?P\d\s+", "", t2).split()[0].split(".")[0]
                ops[op] += 1
                st[op] += s
            print(f"loop {hex(ins[start][0])}-{hex(ins[j][0])}: {len(body)} instrs, {len(c)} DMMA, stall sum {sum(st.values())}")
            print("   count:", dict(ops.most_common(14)))
            print("   stall:", dict(st.most_common(10)))
            break
