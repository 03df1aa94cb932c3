"""One c1 (10e,10o) four-root SBCI1 solve (for launch lists / per-iteration profiling)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_06101_b200 as P  # noqa: E402

op = P.FciOperator(P.synthetic_problem(10, 10, 2603, 0.05), max_determinants=2 ** 62)
P.solve_n_states_sbci1(op, 1, want_vectors=False)
r = P.solve_n_states_sbci1(op, 4, want_vectors=False)
print([p.energy for p in r.pairs], r.summary.matvecs, r.summary.total_iterations)
