"""CPU: the C-ABI library loads, exports every symbol include/sbg.h declares, and its host-only
entry points (no GPU needed) behave like the reference's."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2603_06101_b200 as P
from paper_2603_06101_b200 import _lib
from conftest import ROOT


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "sbg.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sbg_[a-z_0-9]+)\s*\(", txt)) - {"sbg_trace_fn"})


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(_lib.EXPORTED) == syms


def test_binomial_and_counts():
    # determinants.hpp:17-37 and the reference tests (test_determinants.cpp:12-31)
    assert P.binomial(26, 5) == 65780 and P.binomial(26, 4) == 14950
    assert P.determinant_count(26, 5, 5) == 4_327_008_400
    assert P.determinant_count(26, 5, 4) == 983_411_000
    assert P.determinant_count(6, 2, 2) == 225
    pascal = [[0] * 31 for _ in range(31)]
    for n in range(31):
        pascal[n][0] = 1
        for k in range(1, n + 1):
            pascal[n][k] = pascal[n - 1][k - 1] + (pascal[n - 1][k] if k <= n - 1 else 0)
    for n in range(31):
        for ka in range(n + 1):
            assert P.determinant_count(n, ka, ka // 2) == pascal[n][ka] * pascal[n][ka // 2]
    with pytest.raises(ValueError):
        P.determinant_count(65, 1, 1)


def test_config_defaults_and_validation():
    d = _lib.lib().sbg_config_default()
    c = P.SolverConfig()
    for f in ("eps0", "r0", "b_th", "eps1", "x_th1", "x_th2", "r1", "max_cycle", "t_max", "lindep", "clamp_delta",
              "hx_refresh_restarts"):
        assert getattr(d, f) == getattr(c, f), f
    assert (c.eps0, c.r0, c.b_th, c.eps1, c.x_th1, c.x_th2, c.r1, c.hx_refresh_restarts) == (
        1e-10, 1e-5, 1e-2, 1e-7, 0.1, 1.2, 1.0, 5)                       # config.hpp:11-22
    c.validate()
    for bad in (dict(eps0=0.0), dict(x_th1=1.5), dict(max_cycle=1), dict(t_max=0), dict(clamp_delta=-1.0)):
        with pytest.raises(ValueError):
            P.SolverConfig(**bad).validate()
    assert P.SolverConfig.preset("loose").eps0 == 1e-8
    with pytest.raises(ValueError):
        P.SolverConfig.preset("medium")


@pytest.mark.parametrize("norb,scale", [(6, 0.05), (10, 0.05), (16, 0.08)])
def test_product_generator_matches_oracle_bitwise(rest, norb, scale):
    p = P.synthetic_problem(norb, norb, 2603, scale)
    h1, eri = rest.synthetic(norb, 2603, scale)
    assert np.array_equal(p.h1, h1) and np.array_equal(p.eri, eri)


@pytest.mark.parametrize("n,world", [(12870, 8), (3432, 3), (20, 8), (5, 8), (924, 1)])
def test_shard_ranges_partition(n, world):
    lo, hi = C.c_int64(), C.c_int64()
    prev = 0
    per = (n + world - 1) // world
    for r in range(world):
        _lib.check(_lib.lib().sbg_shard_range(n, r, world, C.byref(lo), C.byref(hi)))
        assert lo.value == min(n, prev) and hi.value - lo.value <= per
        prev = hi.value
    assert prev == n


def test_guard_message_and_sector_validation():
    with pytest.raises(RuntimeError, match="4327008400"):       # test_sigma.cpp:121-131
        P.as_operator(P.FciProblem(26, 10, 0), 0)
    with pytest.raises(ValueError, match="parity"):
        P.as_operator(P.FciProblem(4, 3, 0))


def test_fcidump_parser_errors(gold_dir):
    with pytest.raises(P.FcidumpError, match="expected &FCI"):
        P.parse_fcidump("garbage\n")
    with pytest.raises(P.FcidumpError, match="missing NELEC"):
        P.parse_fcidump("&FCI NORB=2, MS2=0 &END\n")
    with pytest.raises(P.FcidumpError, match="unterminated"):
        P.parse_fcidump("&FCI NORB=2, NELEC=2, MS2=0\n")
    with pytest.raises(P.FcidumpError, match="two-electron index out of range"):
        P.parse_fcidump("&FCI NORB=2,NELEC=2,MS2=0,\n&END\n1.0 3 1 1 1\n")
    p = P.parse_fcidump_file(os.path.join(gold_dir, "h6_4e.fcidump"))
    assert (p.norb, p.nelec, p.ms2, p.e_core) == (6, 4, 0, 2.25)


def test_no_device_fails_loudly():
    """The product path never falls back to the CPU: without a GPU, operator creation raises."""
    if _lib.lib().sbg_device_count() > 0:
        pytest.skip("a GPU is present")
    p = P.synthetic_problem(6, 6, 2603, 0.05)
    with pytest.raises(Exception):
        P.FciOperator(p)
