import sys
import numpy as np
sys.path.insert(0, "oracle")
import paper_2603_06101_b200 as P
from oracle import Restatement, baseline_problem
rest = Restatement()
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
q = baseline_problem(idx, rest)
op = P.FciOperator(P.FciProblem(q.norb, q.nelec, 0, 0.0, q.h1, q.eri), max_determinants=2**62)
n = op.dim(); nb = op.n_beta_strings
x = np.random.default_rng(idx).uniform(-1, 1, n)
ys = [op.apply(x) for _ in range(3)]
for k in (1, 2):
    d = np.abs(ys[k] - ys[0])
    bad = np.nonzero(d > 1e-9)[0]
    print(f"run{k}: max diff {d.max():.3e}, n>1e-9: {len(bad)}", flush=True)
    if len(bad):
        rows = bad[:20]
        ref = rest.sigma_rows(q, x, rows)
        for r, a, b, c in zip(rows, ys[0][rows], ys[k][rows], ref):
            print(f"  ia={r // nb} ib={r % nb} y0={a:.6f} y{k}={b:.6f} ref={c:.6f}")
        ia = bad // nb; ib = bad % nb
        print("  ia hist", np.unique(ia)[:20], "ib range", ib.min(), ib.max(), "count ia", len(np.unique(ia)))
