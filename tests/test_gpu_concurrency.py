"""The plugin boundary's threading contract: SymmetricOperator::apply is const and
callable from several threads at once, with an atomic apply counter (operator.hpp:14-18, 47),
tested in the reference by 2 threads x 100 applies (test_operator.cpp:49-64). Here the same through
the C ABI (ctypes releases the GIL inside libsbg, so the threads really enter sbg_sigma together),
plus the host-pointer and device-pointer entry points mixed on different streams."""
import ctypes as C
import threading

import numpy as np
import pytest

import paper_2603_06101_b200 as P
from paper_2603_06101_b200 import _lib
from oracle import baseline_problem

pytestmark = pytest.mark.gpu


def to_product(q):
    return P.FciProblem(q.norb, q.nelec, q.ms2, q.e_core, q.h1.copy(), q.eri.copy())


def run_threads(fns):
    err = [None] * len(fns)

    def body(i):
        try:
            fns[i]()
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err[i] = e
    ts = [threading.Thread(target=body, args=(i,)) for i in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in err:
        if e is not None:
            raise e


@pytest.mark.timeout(600)
@pytest.mark.parametrize("idx", [1, 2])
def test_two_threads_hundred_applies(rest, idx):
    q = baseline_problem(idx, rest)
    op = P.FciOperator(to_product(q), max_determinants=2 ** 62)
    n = op.dim()
    xs = [np.random.default_rng(40 + i).uniform(-1, 1, n) for i in range(2)]
    refs = [op.apply(x) for x in xs]
    op.reset_apply_count()
    bad = [0, 0]
    napply = 100 if idx == 1 else 30

    def worker(i):
        def f():
            for _ in range(napply):
                y = op.apply(xs[i])
                # sigma reduces in L2 (red.global.add): equal to rounding, not bit for bit
                if not np.abs(y - refs[i]).max() <= 1e-13 * np.abs(refs[i]).max():
                    bad[i] += 1
        return f
    run_threads([worker(0), worker(1)])
    assert bad == [0, 0]
    assert op.apply_count() == 2 * napply
    op.close()


@pytest.mark.timeout(600)
def test_host_and_device_entry_points_concurrently(rest):
    """Thread A: sbg_sigma (host buffers, library streams). Thread B: sbg_sigma_device and
    sbg_sigma_padded on its own CUDA stream. Both share the context's transposed-operand scratch;
    the context lock plus the device-side ordering event keep every result exact."""
    import torch
    q = baseline_problem(2, rest)
    op = P.FciOperator(to_product(q), max_determinants=2 ** 62)
    L = _lib.lib()
    h = op.handle
    n = op.dim()
    xa = np.random.default_rng(1).uniform(-1, 1, n)
    xb = np.random.default_rng(2).uniform(-1, 1, n)
    ya_ref, yb_ref = op.apply(xa), op.apply(xb)
    dev_x = torch.from_numpy(xb).cuda()
    dev_y = torch.zeros_like(dev_x)
    pl = L.sbg_padded_len(h)
    px = torch.zeros(pl, dtype=torch.float64, device="cuda")
    py = torch.zeros_like(px)
    stream = torch.cuda.Stream()
    _lib.check(L.sbg_pack(h, C.c_void_p(dev_x.data_ptr()), C.c_void_p(px.data_ptr()), C.c_void_p(stream.cuda_stream)))
    stream.synchronize()
    op.reset_apply_count()
    bad = []

    def a():
        for _ in range(40):
            y = op.apply(xa)
            if not np.abs(y - ya_ref).max() <= 1e-13 * np.abs(ya_ref).max():
                bad.append("host")

    def b():
        torch.cuda.set_device(0)
        out = torch.zeros_like(dev_x)
        for it in range(40):
            if it % 2:
                _lib.check(L.sbg_sigma_device(h, C.c_void_p(dev_x.data_ptr()), C.c_void_p(dev_y.data_ptr()),
                                              C.c_void_p(stream.cuda_stream)))
                stream.synchronize()
                y = dev_y.cpu().numpy()
            else:
                _lib.check(L.sbg_sigma_padded(h, C.c_void_p(px.data_ptr()), C.c_void_p(py.data_ptr()),
                                              C.c_void_p(stream.cuda_stream)))
                _lib.check(L.sbg_unpack(h, C.c_void_p(py.data_ptr()), C.c_void_p(out.data_ptr()),
                                        C.c_void_p(stream.cuda_stream)))
                stream.synchronize()
                y = out.cpu().numpy()
            if not np.abs(y - yb_ref).max() <= 1e-13 * np.abs(yb_ref).max():
                bad.append(("device", it))
    run_threads([a, b])
    assert not bad, bad[:5]
    assert op.apply_count() == 80
    op.close()


@pytest.mark.timeout(900)
@pytest.mark.parametrize("env", [{"SBG_AB_RED": "0"}, {"SBG_AB_RED": "0", "SBG_AB_WS": "1"}, {}])
def test_sharded_exchange_beside_nonatomic_alpha_beta(rest, monkeypatch, env):
    """world > 1: the alpha-alpha blocks arrive on the communication stream while the alpha-beta
    kernel runs. The deterministic alpha-beta forms rewrite whole y rows (no atomics), so adding the
    blocks must wait for them; (12e,12o) at world 2 gives a long alpha-beta kernel to overlap."""
    from paper_2603_06101_b200.dist import LocalRankGroup
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    q = baseline_problem(2, rest)
    prob = to_product(q)
    single = P.FciOperator(prob, max_determinants=2 ** 62)
    nb = single.n_beta_strings
    g = LocalRankGroup(2)
    ops = g.operators(prob)
    for seed in (1, 2, 3):
        x = np.random.default_rng(seed).uniform(-1, 1, single.dim())
        y1 = single.apply(x)
        ys = g.run(lambda r, op: op.apply(x), ops)
        for op, y in zip(ops, ys):
            sl = slice(op.row_lo * nb, op.row_hi * nb)
            assert np.abs(y[sl] - y1[sl]).max() <= 1e-12 * np.abs(y1).max(), (seed, op.row_lo)
    for op in ops:
        op.close()
    g.close()
    single.close()
