"""Generates tests/golden/* from the REFERENCE ITSELF (oracle/_ref/libsbci_ref.so, compiled from
/root/reference). Test infrastructure; run here (the reference does not travel to the GPU box):

    python oracle/make_golden.py fast      # fixtures, c0, c1 (minutes)
    python oracle/make_golden.py c2solve   # (12e,12o) SBCI1 ground state (~30-60 min, serial reference)

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
