"""Per-iteration cost of the device-resident SBCI1 solve: total wall vs summed sigma device time."""
import sys, time, ctypes as C
import numpy as np
import paper_2603_06101_b200 as P
from paper_2603_06101_b200 import _lib
L = _lib.lib()
for tag, norb, ne, sc, nr in (("c1", 10, 10, 0.05, 4), ("c2", 12, 12, 0.05, 1), ("c3", 14, 14, 0.05, 2)):
    op = P.FciOperator(P.synthetic_problem(norb, ne, 2603, sc), max_determinants=2**62)
    P.solve_n_states_sbci1(op, 1, want_vectors=False)
    _lib.check(L.sbg_profile_reset(op.handle))
    t0 = time.perf_counter()
    res = P.solve_n_states_sbci1(op, nr, want_vectors=False)
    wall = time.perf_counter() - t0
    prof = (C.c_double * 4)(); calls = C.c_int64()
    _lib.check(L.sbg_profile_read(op.handle, prof, C.byref(calls)))
    it = res.summary.total_iterations
    print(f"{tag}: E={[p.energy for p in res.pairs]} wall {wall:.3f}s iters {it} sigma {res.summary.matvecs} "
          f"sigma_dev {prof[3]/1e3:.3f}s over {calls.value} calls -> non-sigma {1e3*(wall-prof[3]/1e3)/it:.3f} ms/iter "
          f"launches {res.summary.kernel_launches}", flush=True)
    op.close()
