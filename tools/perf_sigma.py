"""Times sigma builds (device-resident, padded layout) per config with CUDA events."""
import sys, time, json, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_06101_b200 as P
from paper_2603_06101_b200 import _lib

CFG = {2: (12, 12, 0.05), 3: (14, 14, 0.05), 4: (16, 16, 0.08), 1: (10, 10, 0.05)}
which = [int(a) for a in sys.argv[1:]] or [2, 3, 4]
L = _lib.lib()
for c in which:
    norb, ne, s = CFG[c]
    p = P.synthetic_problem(norb, ne, 2603, s)
    t = time.time()
    op = P.FciOperator(p, max_determinants=2**62)
    torch.cuda.synchronize(); tsetup = time.time() - t
    n = op.dim(); pl = L.sbg_padded_len(op.handle)
    x = torch.zeros(pl, dtype=torch.float64, device="cuda"); y = torch.zeros_like(x)
    xd = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
    sm = torch.cuda.Stream(); torch.cuda.set_stream(sm); st = sm.cuda_stream
    _lib.check(L.sbg_pack(op.handle, xd.data_ptr(), x.data_ptr(), st))
    for _ in range(3):
        _lib.check(L.sbg_sigma_padded(op.handle, x.data_ptr(), y.data_ptr(), st))
    torch.cuda.synchronize()
    reps = 20 if c <= 3 else 5
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        _lib.check(L.sbg_sigma_padded(op.handle, x.data_ptr(), y.data_ptr(), st))
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    f = op.sigma_flops()
    print(json.dumps(dict(config=f"c{c}", ndet=n, setup_s=tsetup, sigma_ms=ms, sigma_per_s=1000 / ms,
                          tflops=f["total"] / ms / 1e9, flops=f)), flush=True)
    op.close(); del x, y, xd; torch.cuda.empty_cache()
