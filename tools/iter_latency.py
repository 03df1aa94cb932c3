"""Per-iteration latency of the device-resident SBCI1 / SBCI2 solves at the small configs against
the sigma time (SURVEY §7 hard part 6): wall time per iteration / device time of one sigma, with
the step-latency features switchable (SBG_SPECULATE, SBG_DEVICE_SCALARS).

    python tools/iter_latency.py            # prints one JSON line per (config, method)
"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_06101_b200 as P  # noqa: E402
from paper_2603_06101_b200 import _lib  # noqa: E402

L = _lib.lib()
for tag, norb, ne, sc, nr in (("c1", 10, 10, 0.05, 4), ("c2", 12, 12, 0.05, 1)):
    op = P.FciOperator(P.synthetic_problem(norb, ne, 2603, sc), max_determinants=2 ** 62)
    for name, solve in (("sbci1", P.solve_n_states_sbci1), ("sbci2", P.solve_n_states_sbci2)):
        if name == "sbci2" and nr == 1:
            continue
        solve(op, nr, want_vectors=False)  # warm-up
        best = None
        for _ in range(3):
            _lib.check(L.sbg_profile_reset(op.handle))
            t0 = time.perf_counter()
            res = solve(op, nr, want_vectors=False)
            wall = time.perf_counter() - t0
            prof = (C.c_double * 4)()
            calls = C.c_int64()
            _lib.check(L.sbg_profile_read(op.handle, prof, C.byref(calls)))
            if best is None or wall < best[0]:
                best = (wall, res, prof[3] / max(calls.value, 1))
        wall, res, sig_ms = best
        it = res.summary.total_iterations
        print(json.dumps({"config": tag, "method": name, "wall_s": wall, "iterations": it, "sigma_builds": res.summary.matvecs,
                          "ms_per_iteration": 1e3 * wall / it, "sigma_ms": sig_ms,
                          "iteration_over_sigma": (1e3 * wall / it) / sig_ms,
                          "energies": [p.energy for p in res.pairs],
                          "speculate": os.environ.get("SBG_SPECULATE", "1"),
                          "device_scalars": os.environ.get("SBG_DEVICE_SCALARS", "1")}), flush=True)
    op.close()
