"""Small end-to-end exercise of every kernel family for compute-sanitizer (memcheck / racecheck):
c1 sigma through the host row-block path and the padded device path, SBCI1 / SBCI2 / Davidson with
two roots, <S^2>, and the sharded sigma (world 3, LocalComm) on c0.

    compute-sanitizer --tool memcheck python tools/sanitize_small.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_06101_b200 as P  # noqa: E402
from paper_2603_06101_b200.dist import LocalRankGroup  # noqa: E402

p1 = P.synthetic_problem(10, 10, 2603, 0.05)
op = P.FciOperator(p1, max_determinants=2 ** 62)
x = np.random.default_rng(1).uniform(-1, 1, (2, op.dim()))
y = op.apply(x)
for solve in (P.solve_n_states_sbci1, P.solve_n_states_sbci2, P.davidson_solve):
    r = solve(op, 2, want_vectors=False)
    print(solve.__name__, [pp.energy for pp in r.pairs], [s.s_squared for s in r.summary.states])
op.close()

p0 = P.synthetic_problem(6, 6, 2603, 0.05)
single = P.FciOperator(p0)
x0 = np.random.default_rng(2).uniform(-1, 1, single.dim())
y0 = single.apply(x0)
g = LocalRankGroup(3)
ops = g.operators(p0)
ys = g.run(lambda r, o: o.apply(x0), ops)
nb = single.n_beta_strings
err = max(np.abs(yy[o.row_lo * nb:o.row_hi * nb] - y0[o.row_lo * nb:o.row_hi * nb]).max() for o, yy in zip(ops, ys))
print("sharded sigma max |diff|", err)
for o in ops:
    o.close()
g.close()
single.close()
print("sanitize_small done")
