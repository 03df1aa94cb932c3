"""Non-sigma share of a device-resident solve: wall time of the solver call against the summed device
time of its sigma builds, per method, under environment variants (one subprocess per variant).

    python tools/solver_overhead.py c3 davidson "" "SBG_ZERO_COPY_DOTS=0"
"""
import json
import os
import subprocess
import sys

CFG = {"c1": (10, 10, 0.05, 4), "c2": (12, 12, 0.05, 1), "c3": (14, 14, 0.05, 2), "c4": (16, 16, 0.08, 3)}
CHILD = r'''
import sys, time, json, ctypes as C
sys.path.insert(0, ".")
import paper_2603_06101_b200 as P
from paper_2603_06101_b200 import _lib
norb, ne, sc, nr, method = %d, %d, %r, %d, %r
L = _lib.lib()
op = P.FciOperator(P.synthetic_problem(norb, ne, 2603, sc), max_determinants=2**62)
solve = {"sbci1": P.solve_n_states_sbci1, "sbci2": P.solve_n_states_sbci2, "davidson": P.davidson_solve}[method]
solve(op, nr, want_vectors=False)
_lib.check(L.sbg_profile_reset(op.handle))
t0 = time.perf_counter()
res = solve(op, nr, want_vectors=False)
wall = time.perf_counter() - t0
prof = (C.c_double * 4)(); calls = C.c_int64()
_lib.check(L.sbg_profile_read(op.handle, prof, C.byref(calls)))
print(json.dumps(dict(method=method, wall_s=wall, sigma_dev_s=prof[3] / 1e3, sigma_calls=calls.value,
                      matvecs=res.summary.matvecs, iterations=res.summary.total_iterations,
                      non_sigma_ms_per_iteration=1e3 * (wall - prof[3] / 1e3) / max(res.summary.total_iterations, 1))))
'''
cfg, method = sys.argv[1], sys.argv[2]
norb, ne, sc, nr = CFG[cfg]
for var in sys.argv[3:] or [""]:
    env = dict(os.environ)
    for kv in var.split():
        k, v = kv.split("=", 1)
        env[k] = v
    r = subprocess.run([sys.executable, "-c", CHILD % (norb, ne, sc, nr, method)], env=env, capture_output=True, text=True)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    out = json.loads(line[-1]) if line else {"error": r.stderr[-600:]}
    out.update(config=cfg, variant=var or "default")
    print(json.dumps(out), flush=True)
