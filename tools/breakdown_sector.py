"""Per-phase sigma timing (alpha-beta / same-spin+transposes / total) on any synthetic sector.

    python tools/breakdown_sector.py NORB NELEC [MS2]
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2603_06101_b200 as P  # noqa: E402
from paper_2603_06101_b200 import _lib  # noqa: E402

norb, ne = int(sys.argv[1]), int(sys.argv[2])
ms2 = int(sys.argv[3]) if len(sys.argv) > 3 else ne % 2
L = _lib.lib()
op = P.FciOperator(P.synthetic_problem(norb, ne, 2603, 0.05, ms2), max_determinants=2 ** 62)
h = op.handle
pl = L.sbg_padded_len(h)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    x = torch.rand(pl, dtype=torch.float64, device="cuda")
    y = torch.zeros_like(x)
st.synchronize()
args = (h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), C.c_void_p(st.cuda_stream))
for _ in range(2):
    _lib.check(L.sbg_sigma_padded(*args))
_lib.check(L.sbg_profile_reset(h))
for _ in range(5):
    _lib.check(L.sbg_sigma_padded(*args))
prof = (C.c_double * 4)()
calls = C.c_int64()
_lib.check(L.sbg_profile_read(h, prof, C.byref(calls)))
n = max(calls.value, 1)
print(json.dumps({"sector": f"({ne}e,{norb}o,ms2={ms2})", "n_det": op.dim(), "ab_ms": prof[0] / n,
                  "ss_ms": prof[1] / n, "sigma_ms": prof[3] / n}))
op.close()
