"""Host-side mirror of the reference's FCI operator surface, backed by the CUDA library.

Reference interfaces mirrored here (same names, argument meaning and error behaviour):
  FciProblem            fci/fcidump.hpp:25-69
  parse_fcidump(_file)  fci/fcidump.hpp:109-175
  binomial / determinant_count   fci/determinants.hpp:17-37
  as_operator           fci/fci_operator.hpp:96-120  (guard kDefaultDeterminantGuard = 5,000,000)
  FciOperator           fci/fci_operator.hpp:60-86 + SymmetricOperator operator.hpp:19-48
  sigma_apply           fci/fci_operator.hpp:89-94
"""
from __future__ import annotations

import ctypes as C
import re
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, lib

K_DEFAULT_DETERMINANT_GUARD = 5_000_000


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class FcidumpError(RuntimeError):
    def __init__(self, line, what):
        super().__init__(f"fcidump, line {line}: {what}")
        self.line = line


@dataclass
class FciProblem:
    """Integrals (hartree): h1[norb^2], chemist-notation eri[norb^4] with all 8 permutations."""
    norb: int = 0
    nelec: int = 0
    ms2: int = 0
    e_core: float = 0.0
    h1: np.ndarray = field(default=None)
    eri: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.norb < 0 or self.norb > 32:
            raise ValueError("FciProblem: norb must be in [0, 32]")
        if self.h1 is None:
            self.h1 = np.zeros(self.norb * self.norb)
        if self.eri is None:
            self.eri = np.zeros(self.norb ** 4)
        self.h1 = np.ascontiguousarray(self.h1, np.float64).reshape(-1)
        self.eri = np.ascontiguousarray(self.eri, np.float64).reshape(-1)

    def h1_at(self, i, j):
        return self.h1[i * self.norb + j]

    def eri_at(self, i, j, k, l):
        return self.eri[((i * self.norb + j) * self.norb + k) * self.norb + l]

    def set_h1(self, i, j, v):
        self.h1[i * self.norb + j] = v
        self.h1[j * self.norb + i] = v

    def set_eri(self, i, j, k, l, v):
        n = self.norb
        for a, b, c, d in ((i, j, k, l), (j, i, k, l), (i, j, l, k), (j, i, l, k),
                           (k, l, i, j), (l, k, i, j), (k, l, j, i), (l, k, j, i)):
            self.eri[((a * n + b) * n + c) * n + d] = v

    def n_alpha(self):
        return (self.nelec + self.ms2) // 2

    def n_beta(self):
        return (self.nelec - self.ms2) // 2


def _namelist_int(header, key):
    for m in re.finditer(re.escape(key), header):
        pos = m.start()
        if pos > 0 and (header[pos - 1].isalnum() or header[pos - 1] == "_"):
            continue
        rest = header[m.end():].lstrip()
        if not rest.startswith("="):
            continue
        mm = re.match(r"\s*([+-]?\d+)", rest[1:])
        if not mm:
            return None
        return int(mm.group(1))
    return None


def parse_fcidump(text: str) -> FciProblem:
    """Molpro FCIDUMP reader with the reference's validation and error messages."""
    lines = text.splitlines()
    header, i, saw, done, line_no = "", 0, False, False, 0
    while not done and i < len(lines):
        line = lines[i]
        i += 1
        line_no += 1
        if not saw:
            if "&FCI" not in line:
                if line.strip() == "":
                    continue
                raise FcidumpError(line_no, "expected &FCI namelist header")
            saw = True
        up = line.upper()
        header += " " + up
        if "&END" in up or "/" in up:
            done = True
    if not saw:
        raise FcidumpError(line_no, "empty input, no &FCI header")
    if not done:
        raise FcidumpError(line_no, "unterminated &FCI namelist (missing &END or /)")
    norb, nelec, ms2 = _namelist_int(header, "NORB"), _namelist_int(header, "NELEC"), _namelist_int(header, "MS2")
    if norb is None:
        raise FcidumpError(line_no, "header missing NORB")
    if nelec is None:
        raise FcidumpError(line_no, "header missing NELEC")
    if ms2 is None:
        raise FcidumpError(line_no, "header missing MS2")
    if norb < 1:
        raise FcidumpError(line_no, "NORB must be positive")
    if nelec < 0 or nelec > 2 * norb:
        raise FcidumpError(line_no, "NELEC out of range")
    if (nelec + ms2) % 2 != 0 or abs(ms2) > nelec:
        raise FcidumpError(line_no, "MS2 inconsistent with NELEC")
    prob = FciProblem(norb, nelec, ms2)
    for line in lines[i:]:
        line_no += 1
        if line.strip() == "":
            continue
        tok = line.split()
        try:
            v = float(tok[0])
            a, b, c, d = (int(t) for t in tok[1:5])
        except (ValueError, IndexError):
            raise FcidumpError(line_no, "expected `value i j k l`") from None
        ok = lambda x: 1 <= x <= norb  # noqa: E731
        if a == b == c == d == 0:
            prob.e_core = v
        elif c == 0 and d == 0:
            if not (ok(a) and ok(b)):
                raise FcidumpError(line_no, "one-electron index out of range")
            prob.set_h1(a - 1, b - 1, v)
        else:
            if not all(ok(x) for x in (a, b, c, d)):
                raise FcidumpError(line_no, "two-electron index out of range")
            prob.set_eri(a - 1, b - 1, c - 1, d - 1, v)
    return prob


def parse_fcidump_file(path: str) -> FciProblem:
    try:
        with open(path) as f:
            return parse_fcidump(f.read())
    except OSError:
        raise RuntimeError(f"cannot open {path}") from None


def binomial(n: int, k: int) -> int:
    return int(lib().sbg_binomial(n, k))


def determinant_count(norb: int, n_alpha: int, n_beta: int) -> int:
    out = C.c_uint64()
    check(lib().sbg_determinant_count(norb, n_alpha, n_beta, C.byref(out)))
    return int(out.value)


def synthetic_problem(norb: int, nelec: int, seed: int, offdiag_scale: float, ms2: int = 0) -> FciProblem:
    """BASELINE.json integrals from the pinned generator."""
    h1 = np.zeros(norb * norb)
    eri = np.zeros(norb ** 4)
    check(lib().sbg_synthetic_integrals(norb, seed, offdiag_scale, _dp(h1), _dp(eri)))
    return FciProblem(norb, nelec, ms2, 0.0, h1, eri)


class FciOperator:
    """Matrix-free determinant CI Hamiltonian on the GPU (drop-in for sbci::fci::FciOperator)."""

    def __init__(self, prob: FciProblem, max_determinants: int = K_DEFAULT_DETERMINANT_GUARD, device: int = 0,
                 rank: int = 0, world: int = 1, nccl_id: bytes | None = None, local_group=None):
        L = lib()
        self.problem = prob
        h = C.c_void_p()
        if local_group is not None:  # ranks as threads of this process (dist.LocalRankGroup)
            rc = L.sbg_create_local(prob.norb, prob.nelec, prob.ms2, prob.e_core, _dp(prob.h1), _dp(prob.eri), device,
                                    int(max_determinants), local_group.handle, rank, C.byref(h))
        elif world == 1:
            rc = L.sbg_create(prob.norb, prob.nelec, prob.ms2, prob.e_core, _dp(prob.h1), _dp(prob.eri), device,
                              int(max_determinants), C.byref(h))
        else:
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
            rc = L.sbg_create_dist(prob.norb, prob.nelec, prob.ms2, prob.e_core, _dp(prob.h1), _dp(prob.eri), device,
                                   int(max_determinants), rank, world, C.cast(idbuf, C.c_void_p), C.byref(h))
        check(rc)
        self._h = h
        norb, na, nb = C.c_int(), C.c_int(), C.c_int()
        nas, nbs = C.c_int64(), C.c_int64()
        check(L.sbg_sector(h, C.byref(norb), C.byref(na), C.byref(nb), C.byref(nas), C.byref(nbs)))
        self.norb, self.n_alpha, self.n_beta = norb.value, na.value, nb.value
        self.n_alpha_strings, self.n_beta_strings = nas.value, nbs.value
        lo, hi = C.c_int64(), C.c_int64()
        check(L.sbg_local_rows(h, C.byref(lo), C.byref(hi)))
        self.row_lo, self.row_hi = lo.value, hi.value
        self._diag = None

    def close(self):
        if getattr(self, "_h", None):
            lib().sbg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def dim(self) -> int:
        return int(lib().sbg_dim(self._h))

    def apply(self, x) -> np.ndarray:
        """SymmetricOperator::apply: dimension check, y = H x, counter += 1 per vector."""
        x = np.ascontiguousarray(x, np.float64)
        if x.shape[-1] != self.dim():
            raise ValueError("SymmetricOperator::apply: dimension mismatch")
        y = np.zeros_like(x)
        nvec = 1 if x.ndim == 1 else x.shape[0]
        check(lib().sbg_sigma(self._h, _dp(x), _dp(y), nvec))
        return y

    def diagonal(self) -> np.ndarray:
        if self._diag is None:
            d = np.zeros(self.dim())
            check(lib().sbg_diagonal(self._h, _dp(d)))
            self._diag = d
        return self._diag

    def spin_squared(self, x) -> float:
        """<S^2> of a CI vector (fci/spin.hpp:17-51), computed on the GPU."""
        x = np.ascontiguousarray(x, np.float64)
        if x.shape != (self.dim(),):
            raise ValueError("spin_squared: vector length mismatch")
        out = C.c_double()
        check(lib().sbg_spin_squared(self._h, _dp(x), C.byref(out)))
        return out.value

    def apply_count(self) -> int:
        return int(lib().sbg_apply_count(self._h))

    def reset_apply_count(self):
        lib().sbg_reset_apply_count(self._h)

    def kernel_launches(self) -> int:
        return int(lib().sbg_kernel_launches(self._h))

    def sigma_flops(self):
        a, s, t = C.c_double(), C.c_double(), C.c_double()
        check(lib().sbg_sigma_flops(self._h, C.byref(a), C.byref(s), C.byref(t)))
        return dict(alpha_beta=a.value, same_spin=s.value, total=t.value)

    def string_tables(self, spin: int):
        """(strings u64[n], links structured array [n*L] of (p, q, target, sign)) for spin 0/1."""
        n, L_ = C.c_int64(), C.c_int64()
        check(lib().sbg_table_sizes(self._h, spin, C.byref(n), C.byref(L_)))
        strings = np.zeros(n.value, np.uint64)
        links = (_lib.Excitation * (n.value * L_.value))()
        check(lib().sbg_string_tables(self._h, spin, strings.ctypes.data_as(C.POINTER(C.c_uint64)), links))
        arr = np.frombuffer(links, dtype=np.dtype([("p", "<u2"), ("q", "<u2"), ("target", "<u4"), ("sign", "<f8")]))
        return strings, arr.copy()


def as_operator(prob: FciProblem, ms2_override: int | None = None,
                max_determinants: int = K_DEFAULT_DETERMINANT_GUARD, **kw) -> FciOperator:
    """fci_operator.hpp:103-120: sector from (nelec, ms2), guard on the determinant count."""
    p = prob
    if ms2_override is not None and ms2_override != prob.ms2:
        p = FciProblem(prob.norb, prob.nelec, ms2_override, prob.e_core, prob.h1.copy(), prob.eri.copy())
    if (p.nelec + p.ms2) % 2 != 0:
        raise ValueError("as_operator: MS2 parity mismatch")
    n = determinant_count(p.norb, p.n_alpha(), p.n_beta())
    if n > max_determinants:
        raise RuntimeError(f"as_operator: sector holds {n} determinants, above the guard of {max_determinants} "
                           "(pass a larger bound to override)")
    return FciOperator(p, max_determinants=max_determinants, **kw)


def sigma_apply(prob: FciProblem, x) -> np.ndarray:
    """H x for a single vector without keeping an operator (fci_operator.hpp:89-94)."""
    op = FciOperator(prob, max_determinants=2 ** 63)
    try:
        return op.apply(x)
    finally:
        op.close()
