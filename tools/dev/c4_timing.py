import sys, time
sys.path.insert(0, ".")
import paper_2603_06101_b200 as P
op = P.FciOperator(P.synthetic_problem(16, 16, 2603, 0.08), max_determinants=2**62)
t0 = time.perf_counter()
res = P.solve_n_states_sbci1(op, 1, want_vectors=False)
print("wall", time.perf_counter() - t0, "matvecs", res.summary.matvecs, "iters", res.summary.total_iterations, flush=True)
