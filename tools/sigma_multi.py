"""Times sbg_sigma_padded_multi for nvec = 1, 2, 4 (device-resident padded vectors): the per-vector
time falls by the per-row / per-string set-up that several vectors share.

    python tools/sigma_multi.py c4
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_06101_b200 as P  # noqa: E402
from paper_2603_06101_b200 import _lib  # noqa: E402

CFG = {"c2": (12, 12, 0.05), "c3": (14, 14, 0.05), "c4": (16, 16, 0.08)}
tag = sys.argv[1] if len(sys.argv) > 1 else "c4"
norb, ne, sc = CFG[tag]
L = _lib.lib()
op = P.FciOperator(P.synthetic_problem(norb, ne, 2603, sc), max_determinants=2 ** 62)
h = op.handle
pl = L.sbg_padded_len(h)
s = torch.cuda.Stream()
st = C.c_void_p(s.cuda_stream)
xs, ys = [], []
with torch.cuda.stream(s):
    for v in range(4):
        xd = torch.rand(op.dim(), dtype=torch.float64, device="cuda") * 2 - 1
        x = torch.zeros(pl, dtype=torch.float64, device="cuda")
        _lib.check(L.sbg_pack(h, C.c_void_p(xd.data_ptr()), C.c_void_p(x.data_ptr()), st))
        xs.append(x)
        ys.append(torch.zeros_like(x))
s.synchronize()
reps = {"c2": 50, "c3": 20, "c4": 4}[tag]
for nvec in (1, 2, 4):
    xp = (C.c_void_p * nvec)(*[x.data_ptr() for x in xs[:nvec]])
    yp = (C.c_void_p * nvec)(*[y.data_ptr() for y in ys[:nvec]])
    for _ in range(2):
        _lib.check(L.sbg_sigma_padded_multi(h, nvec, xp, yp, st))
    s.synchronize()
    _lib.check(L.sbg_profile_reset(h))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        _lib.check(L.sbg_sigma_padded_multi(h, nvec, xp, yp, st))
    e1.record(s)
    torch.cuda.synchronize()
    prof = (C.c_double * 4)()
    calls = C.c_int64()
    _lib.check(L.sbg_profile_read(h, prof, C.byref(calls)))
    n = max(calls.value, 1)
    print(json.dumps({"config": tag, "nvec": nvec, "ms_per_vector": e0.elapsed_time(e1) / reps / nvec,
                      "ab_ms_per_call": prof[0] / n, "ss_ms_per_call": prof[1] / n, "calls": calls.value}), flush=True)
op.close()
