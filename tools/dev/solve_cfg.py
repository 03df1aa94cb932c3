"""One SBCI1 solve of a named bench config (for ncu launch lists): python tools/solve_cfg.py c3 [nroots]."""
import sys
import paper_2603_06101_b200 as P
CFG = {"c1": (10, 10), "c2": (12, 12), "c3": (14, 14), "c4": (16, 16)}
norb, ne = CFG[sys.argv[1]]
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 1
op = P.FciOperator(P.synthetic_problem(norb, ne, 2603, 0.05), max_determinants=2**62)
res = P.solve_n_states_sbci1(op, nr, want_vectors=False)
print([p.energy for p in res.pairs], res.summary.matvecs)
