"""CPU checks of the opposite-spin kernel's launch plan (host logic in libsbg, no GPU): every sector
the reference accepts either gets a plan that fits the hardware limits the kernel assumes, or is
reported as outside the tensor-core kernel's limits (the operator then uses the link-table kernel).
Restates the sizing rules of DESIGN.md section 4 (K = 1 + n (norb - n) linked alpha rows, npair =
norb (norb + 1) / 2 packed pairs, 32-column tiles, 227 KB of shared memory per CTA)."""
import ctypes as C
import math

import pytest

from paper_2603_06101_b200 import _lib

KEYS = ["KS", "nt", "mb16", "extra", "k0e", "tall", "xs", "dc", "tma", "npass", "smem", "grows", "gstride", "maxE",
        "threads", "red"]


def plan(norb, na, nb):
    out = (C.c_int64 * 16)()
    rc = _lib.lib().sbg_ab_plan_info(norb, na, nb, out)
    return None if rc != 0 else dict(zip(KEYS, list(out)))


def test_baseline_sector_plans():
    c4 = plan(16, 8, 8)       # (16e,16o): uniform stream with split extra rows, k = 0 inside the DGEMM
    assert (c4["xs"], c4["k0e"], c4["KS"], c4["mb16"], c4["extra"], c4["nt"], c4["dc"], c4["tma"]) == (2, 0, 17, 8, 1, 32, 3, 1)
    assert c4["grows"] == 144 and c4["gstride"] == 34 and c4["threads"] == 512 and c4["red"] == 1
    c3 = plan(14, 7, 7)       # (14e,14o): 105 pairs = 7 m16 blocks, TALL, 50 links = 13 k-steps
    assert (c3["tall"], c3["xs"], c3["KS"], c3["mb16"], c3["k0e"]) == (1, 0, 13, 7, 0)
    c2 = plan(12, 6, 6)       # (12e,12o): 78 pairs = 5 blocks, TALL, 36 links = 9 k-steps + rank-1 k = 0
    assert (c2["tall"], c2["KS"], c2["mb16"], c2["k0e"]) == (1, 9, 5, 1)


@pytest.mark.parametrize("norb", list(range(2, 21)))
def test_every_sector_fits_or_is_rejected(norb):
    npair = norb * (norb + 1) // 2
    for na in range(1, norb + 1):
        for nb in range(1, norb + 1):
            if math.comb(norb, na) * math.comb(norb, nb) > 2 ** 40:
                continue
            p = plan(norb, na, nb)
            K = 1 + na * (norb - na)
            if p is None:      # outside the limits: more than 17 k-steps, or more than 32767 beta strings
                assert K > 68 or math.comb(norb, nb) > 32767 or npair > 136, (norb, na, nb)
                continue
            assert p["smem"] <= 227 * 1024, (norb, na, nb, p)
            assert p["nt"] in (16, 32) and p["threads"] in (512, 32 * p["mb16"])
            kcols = 4 * p["KS"] + (1 if p["k0e"] else 0)
            assert kcols >= K and 4 * (p["KS"] - 1) + (1 if p["k0e"] else 0) < K, (norb, na, nb, p)
            rows = 16 * p["mb16"] + (8 if p["extra"] else 0)
            assert rows >= min(npair, 128 if p["npass"] > 1 else npair), (norb, na, nb, p)
            assert p["npass"] * 128 >= npair or p["npass"] == 1
            assert p["grows"] * p["gstride"] * 8 < 65536          # 16-bit byte offsets in the reduction lists
            if p["xs"]:
                assert p["tma"] and p["dc"] in (2, 3) and p["nt"] == 32 and not p["tall"] and not p["k0e"]
                assert p["gstride"] == 34 and p["grows"] == rows + (8 if p["xs"] == 2 else 0)
            if p["xs"] == 2:
                assert p["mb16"] == 8 and p["extra"] == 1 and p["KS"] in (4, 8, 10, 13, 14, 16, 17)
            if p["tall"]:
                assert 5 <= p["mb16"] <= 7 and not p["extra"] and p["KS"] <= 13
