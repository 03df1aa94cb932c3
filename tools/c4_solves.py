"""(16e,16o) three-root SBCI1 / Davidson / SBCI2 on one GPU (profiles/r01/c4_three_roots.txt)."""
import time
import paper_2603_06101_b200 as P
op = P.FciOperator(P.synthetic_problem(16, 16, 2603, 0.08), max_determinants=2 ** 62)
for name, f in (("sbci1", P.solve_n_states_sbci1), ("davidson", P.davidson_solve), ("sbci2", P.solve_n_states_sbci2)):
    t = time.time()
    r = f(op, 3, want_vectors=False)
    print(f"{name:8s} E = {[p.energy for p in r.pairs]}  iters {[p.iterations for p in r.pairs]}  matvecs "
          f"{r.summary.matvecs}  <S^2> {[round(s.s_squared, 12) for s in r.summary.states]}  wall {time.time() - t:.1f} s",
          flush=True)
