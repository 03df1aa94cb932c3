"""CPU: the oracle restatement pinned against the reference's own fixtures and against the
reference itself (oracle/_ref), before it is trusted as the checker of the CUDA path."""
import json
import os

import numpy as np
import pytest

from oracle import CONFIGS, BASELINE_SEED, Problem, Reference, baseline_problem

HAVE_REF = Reference.available()


def load_gold(gold_dir, tag):
    with open(os.path.join(gold_dir, f"golden_{tag}.json")) as f:
        return json.load(f)


def fixture_problem(gold_dir, name):
    # parse with our python mirror of parse_fcidump (fcidump.hpp:109-169); pinned below vs the reference parser
    from paper_2603_06101_b200.fci import parse_fcidump_file
    p = parse_fcidump_file(os.path.join(gold_dir, f"{name}.fcidump"))
    return Problem(p.norb, p.nelec, p.ms2, p.e_core, p.h1, p.eri, name)


def seeded(n, seed=7):
    x = np.random.default_rng(seed).uniform(-1.0, 1.0, n)
    return x / np.linalg.norm(x)


@pytest.mark.parametrize("name", ["h4_2e", "h6_4e"])
def test_fixture_sigma_diag_golden(rest, gold_dir, name):
    P = fixture_problem(gold_dir, name)
    g = load_gold(gold_dir, name)
    assert (P.norb, P.nelec, P.ms2, P.e_core) == (g["norb"], g["nelec"], g["ms2"], g["e_core"])
    x = seeded(rest.ndet(P))
    sig = rest.sigma(P, x)
    assert np.array_equal(sig, np.load(os.path.join(gold_dir, f"{name}_sigma.npy")))  # bit-exact vs reference
    assert np.array_equal(rest.diag(P), np.load(os.path.join(gold_dir, f"{name}_diag.npy")))
    # independent Slater-Condon dense oracle (dense_oracle.hpp:101-189): abs <= 1e-12 like test_sigma.cpp:39-52
    H = rest.dense_h(P)
    assert np.abs(H @ x - sig).max() <= 1e-12
    ev = np.linalg.eigvalsh(0.5 * (H + H.T))
    assert np.allclose(ev[:6], g["dense_eigs"], atol=1e-12, rtol=0)
    # the reference's SBCI1 energies agree with the dense spectrum to 1e-10 (test_sigma.cpp:109-119)
    assert np.abs(np.array(g["sbci1"]["energies"]) - ev[:3]).max() <= 1e-10


@pytest.mark.parametrize("idx", [0, 1])
def test_baseline_config_golden(rest, gold_dir, idx):
    c = CONFIGS[idx]
    P = baseline_problem(idx, rest)
    g = load_gold(gold_dir, c["name"])
    assert float(P.h1.sum()) == g["h1_sum"] and float(P.eri.sum()) == g["eri_sum"]
    assert P.h1[:4].tolist() == g["h1_first"] and P.eri[:4].tolist() == g["eri_first"]
    assert np.array_equal(rest.strings(P.norb, P.n_alpha), np.load(os.path.join(gold_dir, f"{c['name']}_strings.npy")))
    p, q, t, s = rest.links(P.norb, P.n_alpha)
    assert np.array_equal(t, np.load(os.path.join(gold_dir, f"{c['name']}_links_t.npy")))
    if idx == 0:
        for arr, key in ((p, "p"), (q, "q"), (s, "s")):
            assert np.array_equal(arr, np.load(os.path.join(gold_dir, f"c0_links_{key}.npy")))
    else:
        assert int(np.sum(t.astype(np.int64) * (np.arange(len(t)) % 1009 + 1))) == g["links_checksum"]
        assert float(np.sum(s * (np.arange(len(s)) % 7 + 1))) == g["links_sign_sum"]
    D = rest.diag(P)
    rows = np.load(os.path.join(gold_dir, f"{c['name']}_sigma_rows.npy"))
    assert np.array_equal(D[rows], np.load(os.path.join(gold_dir, f"{c['name']}_diag_vals.npy")))
    order = np.lexsort((np.arange(len(D)), D))
    assert order[:8].tolist() == g["diag_lowest"]
    x = seeded(len(D))
    sig = rest.sigma(P, x, block_rows=16, exact=True)
    assert np.array_equal(sig[rows], np.load(os.path.join(gold_dir, f"{c['name']}_sigma_vals.npy")))
    assert abs(float(sig @ x) - g["sigma_dot_x"]) <= 1e-12 * abs(g["sigma_dot_x"])


def test_sigma_rows_oracle_matches_sigma(rest):
    """The size-independent row oracle used at (14e,14o)/(16e,16o) agrees with the blocked sigma."""
    P = baseline_problem(1, rest)
    x = seeded(rest.ndet(P), 3)
    rows = np.random.default_rng(5).choice(len(x), 64, replace=False)
    full = rest.sigma(P, x, exact=False)
    assert np.abs(rest.sigma_rows(P, x, rows) - full[rows]).max() <= 1e-12 * np.abs(full).max()


def test_c2_golden_pins(rest, gold_dir):
    g = load_gold(gold_dir, "c2")
    P = baseline_problem(2, rest)
    assert float(P.h1.sum()) == g["h1_sum"] and float(P.eri.sum()) == g["eri_sum"]
    rows = np.load(os.path.join(gold_dir, "c2_sigma_rows.npy"))
    x = seeded(rest.ndet(P))
    got = rest.sigma_rows(P, x, rows[:128])
    ref = np.load(os.path.join(gold_dir, "c2_sigma_vals.npy"))[:128]
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("norb,nelec,ms2,seed", [(5, 4, 0, 1), (6, 5, 1, 2), (7, 4, -2, 3), (4, 1, 1, 4)])
def test_restatement_bit_exact_vs_reference(rest, norb, nelec, ms2, seed):
    F = Reference()
    h1, eri = rest.synthetic(norb, seed, 0.07)
    P = Problem(norb, nelec, ms2, 0.37, h1, eri)
    for k in {P.n_alpha, P.n_beta}:
        assert np.array_equal(rest.strings(norb, k), F.strings(norb, k))
        for a, b in zip(rest.links(norb, k), F.links(norb, k)):
            assert np.array_equal(a, b)
    assert np.array_equal(rest.diag(P), F.diag(P))
    x = seeded(rest.ndet(P), seed)
    assert np.array_equal(rest.sigma(P, x, block_rows=3, exact=True), F.sigma(P, x))


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
@pytest.mark.parametrize("name", ["h4_2e", "h6_4e"])
def test_python_fcidump_parser_matches_reference(gold_dir, name):
    F = Reference()
    ref = F.parse_fcidump(os.path.join(gold_dir, f"{name}.fcidump"))
    P = fixture_problem(gold_dir, name)
    assert (P.norb, P.nelec, P.ms2, P.e_core) == (ref.norb, ref.nelec, ref.ms2, ref.e_core)
    assert np.array_equal(P.h1, ref.h1) and np.array_equal(P.eri, ref.eri)


def test_generator_seed_pinned(rest):
    assert BASELINE_SEED == 2603
    h1, eri = rest.synthetic(16, BASELINE_SEED, 0.08)
    E = eri.reshape(256, 256)
    assert np.array_equal(E, E.T)                        # (pq|rs) == (rs|pq) bitwise
    assert np.array_equal(eri.reshape(16, 16, 16, 16), eri.reshape(16, 16, 16, 16).transpose(1, 0, 2, 3))
    assert np.linalg.eigvalsh(E).min() > -1e-12          # PSD (sum of norb rank-1 terms)


# ---------------------------------------------------------------- complete sigma rows (c3/c4 parity)
@pytest.mark.parametrize("spec", [(10, 10, 0, 2603), (7, 4, -2, 3), (6, 5, 1, 2)])
def test_alpha_rows_bit_exact_vs_full_sigma(rest, spec):
    """or_sigma_alpha_rows forms only the intermediate rows that reach the selected alpha rows,
    in contract_sigma's order: its rows equal the full exact sigma (and the reference's) bit for bit."""
    norb, nelec, ms2, seed = spec
    if seed == BASELINE_SEED:
        P = baseline_problem(1, rest)
    else:
        h1, eri = rest.synthetic(norb, seed, 0.07)
        P = Problem(norb, nelec, ms2, 0.37, h1, eri)
    x = seeded(rest.ndet(P), 3)
    full = rest.sigma(P, x, block_rows=5, exact=True)
    if HAVE_REF:
        assert np.array_equal(full, Reference().sigma(P, x))
    na, nb = rest.binomial(norb, P.n_alpha), rest.binomial(norb, P.n_beta)
    rows = np.unique(np.r_[0, na - 1, np.random.default_rng(1).choice(na, min(na, 5), replace=False)])
    got = rest.sigma_alpha_rows(P, x, rows, block_rows=3, nthreads=3)
    for r, g in zip(rows, got):
        assert np.array_equal(g, full[r * nb:(r + 1) * nb])


def test_alpha_rows_c2_bit_exact_vs_reference_golden(rest, gold_dir):
    """(12e,12o): rows of the reference's own sigma (tests/golden/c2_*, from contract_sigma)."""
    P = baseline_problem(2, rest)
    x = seeded(rest.ndet(P))
    rows = np.load(os.path.join(gold_dir, "c2_sigma_rows.npy"))
    vals = np.load(os.path.join(gold_dir, "c2_sigma_vals.npy"))
    nb = rest.binomial(12, 6)
    ia = np.unique(rows // nb)[:6]
    got = rest.sigma_alpha_rows(P, x, ia)
    n = 0
    for a, g in zip(ia, got):
        m = rows // nb == a
        assert np.array_equal(g[rows[m] % nb], vals[m])
        n += m.sum()
    assert n >= 6


@pytest.mark.parametrize("idx", [3, 4])
def test_c34_sigma_row_goldens_vs_slater_condon(rest, gold_dir, idx):
    """The committed complete sigma rows at (14e,14o)/(16e,16o) (oracle/make_golden.py c34) agree with
    the independent Slater-Condon row oracle (dense_oracle.hpp:101-189 restated) on sampled entries,
    and the pinned generator reproduces the integrals they were made from."""
    c = CONFIGS[idx]
    g = load_gold(gold_dir, c["name"])
    P = baseline_problem(idx, rest)
    assert float(P.h1.sum()) == g["h1_sum"] and float(P.eri.sum()) == g["eri_sum"]
    rows = np.load(os.path.join(gold_dir, f"{c['name']}_sigma_alpha_rows.npy"))
    vals = np.load(os.path.join(gold_dir, f"{c['name']}_sigma_alpha_vals.npy"))
    nb = rest.binomial(P.norb, P.n_beta)
    assert vals.shape == (len(rows), nb)
    x = seeded(rest.ndet(P))
    rng = np.random.default_rng(idx)
    sel = [(i, int(b)) for i in range(len(rows)) for b in rng.choice(nb, 4, replace=False)]
    dets = np.array([rows[i] * nb + b for i, b in sel], np.int64)
    sc = rest.sigma_rows(P, x, dets)
    ref = np.array([vals[i, b] for i, b in sel])
    assert np.abs(sc - ref).max() <= 1e-12 * np.abs(vals).max()
