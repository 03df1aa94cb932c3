"""A few SBCI1 iterations at (16e,16o) (vectors 1.33 GB > L2) for profiling the HBM-bound update
passes (k_precond, k_subspace, k_lincomb, k_reduce_finish) under ncu, plus their CUDA-event
timing without ncu. The solve is cut off by t_max (NonConvergenceError is expected).

    python tools/prof_update.py [iterations]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_06101_b200 as P  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
op = P.FciOperator(P.synthetic_problem(16, 16, 2603, 0.08), max_determinants=2 ** 62)
cfg = P.SolverConfig(t_max=iters)
t0 = time.perf_counter()
try:
    P.solve_n_states_sbci1(op, 1, cfg, want_vectors=False)
except P.NonConvergenceError as e:
    print(f"stopped after {iters} iterations as intended: {e}")
print(f"wall {time.perf_counter() - t0:.2f} s, {op.apply_count()} sigma builds, n_det {op.dim()}")
op.close()
