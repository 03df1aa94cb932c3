"""End-to-end sigma builds through the host-pointer C ABI (sbg_sigma over pinned host vectors, H2D
and D2H inside the timed call) under environment variants, one subprocess per variant.

    python tools/e2e_modes.py c4 "" "SBG_IO_BLOCKS=8"
"""
import json
import os
import subprocess
import sys

CFG = {"c2": (12, 12, 0.05), "c3": (14, 14, 0.05), "c4": (16, 16, 0.08)}
CHILD = r'''
import json, sys, time, torch, ctypes as C
sys.path.insert(0, ".")
import paper_2603_06101_b200 as P
from paper_2603_06101_b200 import _lib
norb, ne, sc, nvec = %d, %d, %r, %d
L = _lib.lib()
op = P.FciOperator(P.synthetic_problem(norb, ne, 2603, sc), max_determinants=2**62)
n = op.dim()
xh = torch.empty((nvec, n), dtype=torch.float64, pin_memory=True).uniform_(-1, 1)
yh = torch.empty((nvec, n), dtype=torch.float64, pin_memory=True)
dp = C.POINTER(C.c_double)
xp = C.cast(C.c_void_p(xh.data_ptr()), dp); yp = C.cast(C.c_void_p(yh.data_ptr()), dp)
_lib.check(L.sbg_sigma(op.handle, xp, yp, 2))
best = 1e9
for _ in range(3):
    t0 = time.perf_counter(); _lib.check(L.sbg_sigma(op.handle, xp, yp, nvec)); best = min(best, time.perf_counter() - t0)
print(json.dumps(dict(e2e_sigma_per_s=nvec / best, seconds=best)))
'''


def main():
    cfg = sys.argv[1]
    norb, ne, sc = CFG[cfg]
    nvec = {"c2": 64, "c3": 16, "c4": 6}[cfg]
    for var in sys.argv[2:] or [""]:
        env = dict(os.environ)
        for kv in var.split():
            k, v = kv.split("=", 1)
            env[k] = v
        r = subprocess.run([sys.executable, "-c", CHILD % (norb, ne, sc, nvec)], env=env, capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        out = json.loads(line[-1]) if line else {"error": r.stderr[-800:]}
        out.update(config=cfg, variant=var or "default")
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
