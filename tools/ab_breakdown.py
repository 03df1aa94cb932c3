"""Per-phase sigma timing (profile slots: alpha-beta, same-spin + transposes, all-gather, total)
with the K6 experiment switches (SBG_AB_DEBUG: 1 = skip scatter, 2 = skip DMMA, 3 = both).

    python tools/ab_breakdown.py [c3,c4] [0,1,2,3,4,5]
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
L = _lib.lib()
for tag in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["c4"]):
    norb, ne, s = CFG[tag]
    op = P.FciOperator(P.synthetic_problem(norb, ne, 2603, s), max_determinants=2 ** 62)
    h = op.handle
    pl = L.sbg_padded_len(h)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        xd = torch.rand(op.dim(), dtype=torch.float64, device="cuda") * 2 - 1
        x = torch.zeros(pl, dtype=torch.float64, device="cuda")
        y = torch.zeros_like(x)
        _lib.check(L.sbg_pack(h, C.c_void_p(xd.data_ptr()), C.c_void_p(x.data_ptr()), C.c_void_p(st.cuda_stream)))
    st.synchronize()
    reps = 5 if tag == "c4" else 20
    for dbg in (sys.argv[2].split(",") if len(sys.argv) > 2 else ("0", "1", "2", "3")):
        os.environ["SBG_AB_DEBUG"] = dbg
        for _ in range(2):
            _lib.check(L.sbg_sigma_padded(h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), C.c_void_p(st.cuda_stream)))
        _lib.check(L.sbg_profile_reset(h))
        for _ in range(reps):
            _lib.check(L.sbg_sigma_padded(h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), C.c_void_p(st.cuda_stream)))
        prof = (C.c_double * 4)()
        calls = C.c_int64()
        _lib.check(L.sbg_profile_read(h, prof, C.byref(calls)))
        n = max(calls.value, 1)
        print(json.dumps({"config": tag, "dbg": int(dbg), "ab_ms": prof[0] / n, "ss_ms": prof[1] / n,
                          "gather_ms": prof[2] / n, "sigma_ms": prof[3] / n}), flush=True)
    os.environ["SBG_AB_DEBUG"] = "0"
    op.close()
