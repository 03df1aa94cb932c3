import paper_2603_06101_b200 as P
op = P.FciOperator(P.synthetic_problem(12, 12, 2603, 0.05), max_determinants=2**62)
res = P.solve_n_states_sbci1(op, 1, want_vectors=False)
print(res.pairs[0].energy, res.summary.matvecs)
