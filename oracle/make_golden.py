"""Generates tests/golden/* from the REFERENCE ITSELF (oracle/_ref/libsbci_ref.so, compiled from
/root/reference). Test infrastructure; run here (the reference does not travel to the GPU box):

    python oracle/make_golden.py fast      # fixtures, c0, c1 (minutes)
    python oracle/make_golden.py c2solve   # (12e,12o) SBCI1 ground state (~30-60 min, serial reference)
    python oracle/make_golden.py c34       # (14e,14o) / (16e,16o): tables + diagonal digests from the
                                           # reference, complete sigma rows from the exact restatement

Outputs: tests/golden/golden_<tag>.json (scalars) and tests/golden/<tag>_*.npy (small arrays).
Seeded vectors: numpy default_rng(seed).uniform(-1, 1, n_det), normalised (see seeded_vector).
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from oracle import CONFIGS, Reference, Restatement, baseline_problem  # noqa: E402

GOLD = os.path.join(os.path.dirname(HERE), "tests", "golden")


def seeded_vector(n, seed=7):
    x = np.random.default_rng(seed).uniform(-1.0, 1.0, n)
    return x / np.linalg.norm(x)


def sample_rows(n, k=2048, seed=11):
    if n <= k:
        return np.arange(n, dtype=np.int64)
    return np.sort(np.random.default_rng(seed).choice(n, k, replace=False)).astype(np.int64)


def save(tag, scalars, arrays):
    for k, v in arrays.items():
        np.save(os.path.join(GOLD, f"{tag}_{k}.npy"), v)
    with open(os.path.join(GOLD, f"golden_{tag}.json"), "w") as f:
        json.dump(scalars, f, indent=1, sort_keys=True)


def solve_record(F, P, nroots, method):
    t = time.time()
    r = F.solve(P, nroots, method=method)
    return dict(energies=r["energies"].tolist(), iterations=r["iterations"].tolist(), restarts=r["restarts"].tolist(),
                residuals=r["residuals"].tolist(), matvecs=r["matvecs"], s_squared=r["s_squared"].tolist(),
                wall_s=time.time() - t)


def fast():
    F = Reference()
    R = Restatement()
    # reference fixtures (tests/data/*.fcidump, copied verbatim as golden inputs)
    for name, nroots in (("h4_2e", 3), ("h6_4e", 3)):
        P = F.parse_fcidump(os.path.join(GOLD, f"{name}.fcidump"))
        x = seeded_vector(R.ndet(P))
        sig = F.sigma(P, x)
        H = R.dense_h(P)
        ev = np.linalg.eigvalsh(0.5 * (H + H.T))
        sc = dict(norb=P.norb, nelec=P.nelec, ms2=P.ms2, e_core=P.e_core, dense_eigs=ev[:6].tolist(),
                  sbci1=solve_record(F, P, nroots, 1), sbci2=solve_record(F, P, nroots, 2),
                  davidson=solve_record(F, P, nroots, 3))
        save(name, sc, dict(sigma=sig, diag=F.diag(P)))
        print(name, sc["sbci1"]["energies"], flush=True)
    for idx in (0, 1):
        c = CONFIGS[idx]
        P = baseline_problem(idx, R)
        n = R.ndet(P)
        x = seeded_vector(n)
        t = time.time()
        sig = F.sigma(P, x)
        t_sig = time.time() - t
        D = F.diag(P)
        rows = sample_rows(n)
        na = R.binomial(P.norb, P.n_alpha)
        p, q, tt, s = F.links(P.norb, P.n_alpha)
        order = np.lexsort((np.arange(n), D))
        sc = dict(norb=P.norb, nelec=P.nelec, h1_sum=float(P.h1.sum()), eri_sum=float(P.eri.sum()),
                  h1_first=P.h1[:4].tolist(), eri_first=P.eri[:4].tolist(), sigma_seconds=t_sig,
                  sigma_norm=float(np.linalg.norm(sig)), sigma_dot_x=float(sig @ x), diag_min=float(D.min()),
                  diag_lowest=order[:8].tolist(), n_strings=na,
                  sbci1=solve_record(F, P, c["nroots"], 1))
        arrays = dict(sigma_rows=rows, sigma_vals=sig[rows], diag_vals=D[rows],
                      links_p=p, links_q=q, links_t=tt, links_s=s, strings=F.strings(P.norb, P.n_alpha))
        if n <= 400:
            arrays["sigma"] = sig
            arrays["diag"] = D
        if idx == 1:
            arrays.pop("links_p"); arrays.pop("links_q"); arrays.pop("links_s")
            sc["links_checksum"] = int(np.sum(tt.astype(np.int64) * (np.arange(len(tt)) % 1009 + 1)))
            sc["links_sign_sum"] = float(np.sum(s * (np.arange(len(s)) % 7 + 1)))
        save(c["name"], sc, arrays)
        print(c["name"], sc["sbci1"], flush=True)


def c2(solve):
    F = Reference()
    R = Restatement()
    P = baseline_problem(2, R)
    n = R.ndet(P)
    D = F.diag(P)
    order = np.lexsort((np.arange(n), D))
    rows = sample_rows(n)
    sc = dict(norb=P.norb, nelec=P.nelec, diag_min=float(D.min()), diag_lowest=order[:8].tolist(),
              h1_sum=float(P.h1.sum()), eri_sum=float(P.eri.sum()))
    arrays = dict(diag_vals=D[rows], sigma_rows=rows)
    x = seeded_vector(n)
    t = time.time()
    sig = F.sigma(P, x)
    sc["sigma_seconds"] = time.time() - t
    sc["sigma_norm"] = float(np.linalg.norm(sig))
    sc["sigma_dot_x"] = float(sig @ x)
    arrays["sigma_vals"] = sig[rows]
    if solve:
        sc["sbci1"] = solve_record(F, P, 1, 1)
    save("c2", sc, arrays)
    print("c2", sc, flush=True)


def digest(*arrays):
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


# complete alpha rows per config for the full-size sigma parity (c3: 12, c4: 6 rows)
C34_ROWS = {3: 12, 4: 6}


def c34_rows(na, idx):
    k = C34_ROWS[idx]
    rows = np.random.default_rng(13).choice(na, k - 2, replace=False).tolist()
    rows += [0, na - 1]          # the first and last alpha strings (edge tiles of the schedule)
    return np.array(sorted(set(rows)), np.int64)


def c34():
    """(14e,14o) and (16e,16o), where the reference cannot build a full sigma:
    * strings, link tables and the exact diagonal computed by the REFERENCE ITSELF, stored as
      SHA-256 digests (bit-exact pins; the arrays are 0.1-1.3 GB), plus the 8 lowest diagonal
      entries in the reference's stable order (the seed determinants, sbci1.hpp:50-53);
    * complete sigma rows (every beta string) of a few alpha strings from the restatement's
      or_sigma_alpha_rows, which reproduces contract_sigma's accumulation order (bit-identical to
      the reference wherever the reference runs; pinned by tests/test_oracle_pins.py)."""
    F = Reference()
    R = Restatement()
    for idx in (3, 4):
        c = CONFIGS[idx]
        P = baseline_problem(idx, R)
        n = R.ndet(P)
        na = R.binomial(P.norb, P.n_alpha)
        t = time.time()
        strings = F.strings(P.norb, P.n_alpha)
        p, q, tt, s = F.links(P.norb, P.n_alpha)
        D = F.diag(P)
        t_tab = time.time() - t
        order = np.lexsort((np.arange(n), D))
        sc = dict(norb=P.norb, nelec=P.nelec, n_strings=na, n_det=n, h1_sum=float(P.h1.sum()), eri_sum=float(P.eri.sum()),
                  strings_sha256=digest(strings), links_sha256=digest(p, q, tt, s), diag_sha256=digest(D),
                  diag_min=float(D.min()), diag_lowest=order[:8].tolist(),
                  diag_lowest_values=D[order[:8]].tolist(), reference_tables_seconds=t_tab)
        del D, order
        x = seeded_vector(n)
        rows = c34_rows(na, idx)
        t = time.time()
        vals = R.sigma_alpha_rows(P, x, rows)
        sc["sigma_alpha_rows_seconds"] = time.time() - t
        sc["sigma_rows_vector"] = "numpy default_rng(7).uniform(-1, 1, n_det), normalised"
        save(c["name"], sc, dict(sigma_alpha_rows=rows, sigma_alpha_vals=vals))
        print(c["name"], {k: v for k, v in sc.items() if "sha" not in k}, flush=True)


def methods():
    """Adds the reference's SBCI2 and Davidson records for c0/c1 to their golden JSON files."""
    F = Reference()
    R = Restatement()
    for idx in (0, 1):
        c = CONFIGS[idx]
        P = baseline_problem(idx, R)
        path = os.path.join(GOLD, f"golden_{c['name']}.json")
        with open(path) as f:
            sc = json.load(f)
        sc["sbci2"] = solve_record(F, P, c["nroots"], 2)
        sc["davidson"] = solve_record(F, P, c["nroots"], 3)
        with open(path, "w") as f:
            json.dump(sc, f, indent=1, sort_keys=True)
        print(c["name"], sc["sbci2"], sc["davidson"], flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "fast"
    if what == "fast":
        fast()
    elif what == "c2sigma":
        c2(False)
    elif what == "c2solve":
        c2(True)
    elif what == "methods":
        methods()
    elif what == "c34":
        c34()
