"""Times device-resident sigma builds (padded layout, CUDA events) under environment variants, one
subprocess per variant (the variants are read when the operator is planned).

    python tools/sigma_modes.py c4 "SBG_SS_REM=0" "" "SBG_AB_RED=0"
"""
import json
import os
import subprocess
import sys

CFG = {"c1": (10, 10, 0.05), "c2": (12, 12, 0.05), "c3": (14, 14, 0.05), "c4": (16, 16, 0.08)}
CHILD = r'''
import json, sys, torch, ctypes as C
sys.path.insert(0, ".")
import paper_2603_06101_b200 as P
from paper_2603_06101_b200 import _lib
norb, ne, sc, reps = %d, %d, %r, %d
L = _lib.lib()
op = P.FciOperator(P.synthetic_problem(norb, ne, 2603, sc), max_determinants=2**62)
n = op.dim(); pl = L.sbg_padded_len(op.handle)
s = torch.cuda.Stream(); st = C.c_void_p(s.cuda_stream)
xd = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
x = torch.zeros(pl, dtype=torch.float64, device="cuda"); y = torch.zeros_like(x)
torch.cuda.synchronize()
_lib.check(L.sbg_pack(op.handle, C.c_void_p(xd.data_ptr()), C.c_void_p(x.data_ptr()), st))
for _ in range(3):
    _lib.check(L.sbg_sigma_padded(op.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), st))
s.synchronize()
_lib.check(L.sbg_profile_reset(op.handle))
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(reps):
    _lib.check(L.sbg_sigma_padded(op.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), st))
e1.record(s); torch.cuda.synchronize()
prof = (C.c_double * 4)(); calls = C.c_int64()
_lib.check(L.sbg_profile_read(op.handle, prof, C.byref(calls)))
ms = e0.elapsed_time(e1) / reps
print(json.dumps(dict(sigma_ms=ms, ab_ms=prof[0] / calls.value, ss_ms=prof[1] / calls.value, flops=op.sigma_flops())))
'''


def main():
    cfg = sys.argv[1]
    norb, ne, sc = CFG[cfg]
    reps = {"c1": 200, "c2": 50, "c3": 20, "c4": 8}[cfg]
    for var in sys.argv[2:] or [""]:
        env = dict(os.environ)
        for kv in var.split():
            k, v = kv.split("=", 1)
            env[k] = v
        r = subprocess.run([sys.executable, "-c", CHILD % (norb, ne, sc, reps)], env=env, capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        out = json.loads(line[-1]) if line else {"error": r.stderr[-800:]}
        out.update(config=cfg, variant=var or "default")
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
