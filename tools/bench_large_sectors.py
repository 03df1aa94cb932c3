"""sigma time on sectors beyond 16 orbitals: the opposite-spin kernel in 128-row pair blocks
(default) vs the generic link-table kernel (SBG_AB_RED=0).

    python tools/bench_large_sectors.py
"""
import ctypes as C, json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2603_06101_b200 as P
from paper_2603_06101_b200 import _lib
L = _lib.lib()
for norb, ne in ((18, 8), (20, 6)):
    op = P.FciOperator(P.synthetic_problem(norb, ne, 2603, 0.05), max_determinants=2 ** 62)
    h = op.handle; pl = L.sbg_padded_len(h)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        x = torch.rand(pl, dtype=torch.float64, device="cuda"); y = torch.zeros_like(x)
    st.synchronize()
    for _ in range(2): _lib.check(L.sbg_sigma_padded(h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), C.c_void_p(st.cuda_stream)))
    st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5): _lib.check(L.sbg_sigma_padded(h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), C.c_void_p(st.cuda_stream)))
    e1.record(st); torch.cuda.synchronize()
    print(json.dumps({"sector": f"({ne}e,{norb}o)", "n_det": op.dim(), "mode": os.environ.get("SBG_AB_RED", "1"), "sigma_ms": e0.elapsed_time(e1) / 5}), flush=True)
    op.close()
