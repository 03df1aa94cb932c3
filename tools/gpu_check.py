"""Ad-hoc diagnostics on the GPU box: every component vs the oracle, printed, never stops early."""
import sys, time, traceback
import numpy as np
sys.path.insert(0, "oracle")
import paper_2603_06101_b200 as P
from paper_2603_06101_b200 import _lib
from oracle import Restatement, Reference, baseline_problem, CONFIGS

R = Restatement()
L = _lib.lib()
print("selftest rc", L.sbg_selftest(), L.sbg_last_error())

def probs():
    out = []
    for name in ("h4_2e", "h6_4e"):
        out.append(Reference().parse_fcidump(f"tests/golden/{name}.fcidump") if Reference.available() else None)
    return out

def to_P(op):
    return P.FciProblem(op.norb, op.nelec, op.ms2, op.e_core, op.h1, op.eri)

cases = []
for name in ("h4_2e", "h6_4e"):
    p = P.parse_fcidump_file(f"tests/golden/{name}.fcidump")
    cases.append((name, p))
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    q = baseline_problem(i, R)
    cases.append((q.name, P.FciProblem(q.norb, q.nelec, 0, 0.0, q.h1, q.eri)))
# odd sectors
cases.append(("4o1a0b", P.FciProblem(4, 1, 1, -0.75, *R.synthetic(4, 5, 0.05))))
cases.append(("5o3a2b", P.FciProblem(5, 5, 1, 0.3, *R.synthetic(5, 9, 0.05))))
cases.append(("7o2a3b", P.FciProblem(7, 5, -1, 0.0, *R.synthetic(7, 11, 0.05))))

for name, p in cases:
    try:
        from oracle import Problem
        q = Problem(p.norb, p.nelec, p.ms2, p.e_core, p.h1, p.eri, name)
        t = time.time()
        op = P.FciOperator(p, max_determinants=2**62)
        n = op.dim()
        for spin, k in ((0, p.n_alpha()), (1, p.n_beta())):
            s, l = op.string_tables(spin)
            rs = R.strings(p.norb, k); rp, rq, rt, rsg = R.links(p.norb, k)
            ok = (s == rs).all() and (l["p"] == rp).all() and (l["q"] == rq).all() and (l["target"] == rt).all() and (l["sign"] == rsg).all()
            print(name, "spin", spin, "tables bitexact", ok)
        d = op.diagonal(); dr = R.diag(q)
        print(name, "diag bitexact", (d == dr).all(), np.abs(d - dr).max())
        x = np.random.default_rng(7).uniform(-1, 1, n); x /= np.linalg.norm(x)
        t = time.time(); y = op.apply(x); tg = time.time() - t
        if n <= 1_000_000:
            t = time.time(); yr = R.sigma(q, x, block_rows=16, exact=False); tr = time.time() - t
            print(name, "ndet", n, "sigma rel err", np.abs(y - yr).max() / np.abs(yr).max(), "gpu %.3fs oracle %.3fs" % (tg, tr))
        rows = np.sort(np.random.default_rng(3).choice(n, min(n, 64), replace=False))
        yr = R.sigma_rows(q, x, rows)
        print(name, "rows rel err", np.abs(y[rows] - yr).max() / np.abs(yr).max())
        # hermiticity
        a = np.random.default_rng(5).uniform(-1, 1, n); b = np.random.default_rng(6).uniform(-1, 1, n)
        ha, hb = op.apply(np.stack([a, b]))
        print(name, "herm", abs(a @ hb - ha @ b) / (np.linalg.norm(a) * np.linalg.norm(b)))
        if n <= 100_000:
            nr = 3 if name.startswith("h") else (4 if name == "c1" else 1)
            t = time.time()
            res = P.solve_n_states_sbci1(op, nr)
            print(name, "sbci1 E", [pp.energy for pp in res.pairs], "iters", [pp.iterations for pp in res.pairs], "mv", res.summary.matvecs, "%.2fs" % (time.time() - t))
            if n <= 400:
                H = R.dense_h(q); ev = np.linalg.eigvalsh(0.5 * (H + H.T))
                print(name, "dense", ev[:nr], "dE", np.abs(np.array([pp.energy for pp in res.pairs]) - ev[:nr]).max())
        op.close()
    except Exception:
        traceback.print_exc()
