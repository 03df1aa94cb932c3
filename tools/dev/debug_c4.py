import sys, time
import numpy as np
sys.path.insert(0, "oracle")
import paper_2603_06101_b200 as P
from oracle import Restatement, baseline_problem, Problem
rest = Restatement()
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
q = baseline_problem(idx, rest)
op = P.FciOperator(P.FciProblem(q.norb, q.nelec, 0, 0.0, q.h1, q.eri), max_determinants=2**62)
n = op.dim(); nb = op.n_beta_strings; na = op.n_alpha_strings
rng = np.random.default_rng(idx)
x = rng.uniform(-1, 1, n)
y = op.apply(x)
def check(name, rows):
    rows = np.unique(np.asarray(rows, dtype=np.int64))
    ref = rest.sigma_rows(q, x, rows)
    err = np.abs(y[rows] - ref)
    k = int(np.argmax(err))
    print(f"{name:24s} n={len(rows):5d} maxerr={err.max():.3e} at ia={rows[k]//nb} ib={rows[k]%nb} rel={err.max()/np.abs(ref).max():.2e}", flush=True)
    return rows[err > 1e-9 * np.abs(ref).max()]
bad = []
bad += list(check("random", rng.choice(n, 400, replace=False)))
bad += list(check("last beta cols", [ia * nb + ib for ia in rng.choice(na, 40) for ib in range(nb - 10, nb)]))
bad += list(check("first beta cols", [ia * nb + ib for ia in rng.choice(na, 40) for ib in range(0, 10)]))
bad += list(check("last alpha row", [(na - 1) * nb + ib for ib in rng.choice(nb, 200)]))
bad += list(check("first alpha row", [ib for ib in rng.choice(nb, 200)]))
bad += list(check("tile boundary cols", [ia * nb + ib for ia in rng.choice(na, 20) for ib in range(15, nb, 16)[::40]]))
bad += list(check("diag-ish", [i * nb + i for i in rng.choice(min(na, nb), 200)]))
print("bad count", len(bad), "sample", [(b // nb, b % nb) for b in bad[:20]])
