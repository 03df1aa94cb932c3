"""ctypes front-end to the TEST-ONLY checkers (see oracle/sbci_oracle.cpp header).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module. The product
(paper_2603_06101_b200) never does: its path is the CUDA library and fails loudly without it.

Two checkers live here:
  * ``Restatement`` — oracle/liboracle.so, our CPU restatement of the reference algorithms;
  * ``Reference``   — oracle/_ref/libsbci_ref.so, the unmodified reference headers compiled in place.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_D = C.POINTER(C.c_double)
_U64 = C.POINTER(C.c_uint64)


def _dp(a):
    return a.ctypes.data_as(_D)


def build():
    """Compile both checkers (the reference only if /root/reference is present)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE], check=True)


@dataclass
class Problem:
    """Mirror of sbci::fci::FciProblem (fcidump.hpp:25-69): dense h1[norb^2], eri[norb^4]."""
    norb: int
    nelec: int
    ms2: int
    e_core: float
    h1: np.ndarray
    eri: np.ndarray
    name: str = field(default="")

    @property
    def n_alpha(self):
        return (self.nelec + self.ms2) // 2

    @property
    def n_beta(self):
        return (self.nelec - self.ms2) // 2

    def args(self):
        return (self.norb, self.nelec, self.ms2, C.c_double(self.e_core), _dp(self.h1), _dp(self.eri))


class Restatement:
    def __init__(self, path=None):
        path = path or os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.or_last_error.restype = C.c_char_p
        L.or_binomial.restype = C.c_uint64
        L.or_sc_element.restype = C.c_double
        L.or_sc_element.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, _D, _D] + [C.c_uint64] * 4

    def _ck(self, rc):
        if rc != 0:
            raise RuntimeError(self.lib.or_last_error().decode())

    def binomial(self, n, k):
        return int(self.lib.or_binomial(n, k))

    def strings(self, norb, k):
        out = np.zeros(self.binomial(norb, k), np.uint64)
        self._ck(self.lib.or_strings(norb, k, out.ctypes.data_as(_U64)))
        return out

    def links(self, norb, k):
        n = self.binomial(norb, k) * k * (norb - k + 1)
        p = np.zeros(n, np.uint16); q = np.zeros(n, np.uint16); t = np.zeros(n, np.uint32); s = np.zeros(n)
        self._ck(self.lib.or_links(norb, k, p.ctypes.data_as(C.c_void_p), q.ctypes.data_as(C.c_void_p),
                                   t.ctypes.data_as(C.c_void_p), _dp(s)))
        return p, q, t, s

    def absorb_h1(self, P):
        out = np.zeros(P.norb ** 4)
        self._ck(self.lib.or_absorb_h1(*P.args(), _dp(out)))
        return out

    def ndet(self, P):
        return self.binomial(P.norb, P.n_alpha) * self.binomial(P.norb, P.n_beta)

    def diag(self, P):
        out = np.zeros(self.ndet(P))
        self._ck(self.lib.or_diag(*P.args(), _dp(out)))
        return out

    def sigma(self, P, x, block_rows=8, exact=True):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros_like(x)
        na = self.binomial(P.norb, P.n_alpha)
        self._ck(self.lib.or_sigma_blocked(*P.args(), _dp(x), _dp(y), int(block_rows), int(bool(exact)),
                                           C.c_int64(0), C.c_int64(na)))
        return y

    def bench(self, P, nthreads):
        """CPU-baseline timing context (or_bench_*): tables and per-thread outputs built once."""
        return SampleBench(self, P, nthreads)

    def sigma_alpha_rows(self, P, x, alpha_rows, block_rows=8, nthreads=None):
        """Complete sigma rows (all beta strings) of the given alpha strings, bit-identical to the
        reference's contract_sigma rows (or_sigma_alpha_rows). Returns len(alpha_rows) x n_beta."""
        x = np.ascontiguousarray(x, np.float64)
        rows = np.ascontiguousarray(alpha_rows, np.int64)
        nb = self.binomial(P.norb, P.n_beta)
        out = np.zeros((len(rows), nb))
        self._ck(self.lib.or_sigma_alpha_rows(*P.args(), _dp(x), rows.ctypes.data_as(C.c_void_p),
                                              C.c_int64(len(rows)), int(block_rows), int(nthreads or os.cpu_count() or 1),
                                              _dp(out)))
        return out

    def dense_h(self, P):
        n = self.ndet(P)
        out = np.zeros((n, n))
        self._ck(self.lib.or_dense_h(*P.args(), _dp(out)))
        return out

    def sigma_rows(self, P, x, rows):
        x = np.ascontiguousarray(x, np.float64)
        rows = np.ascontiguousarray(rows, np.int64)
        out = np.zeros(len(rows))
        self._ck(self.lib.or_sigma_rows(*P.args(), _dp(x), rows.ctypes.data_as(C.c_void_p), C.c_int64(len(rows)), _dp(out)))
        return out

    def synthetic(self, norb, seed, offdiag_scale):
        h1 = np.zeros(norb * norb); eri = np.zeros(norb ** 4)
        self._ck(self.lib.or_synthetic(norb, C.c_uint64(seed), C.c_double(offdiag_scale), _dp(h1), _dp(eri)))
        return h1, eri


class SampleBench:
    """Bounded samples of the blocked contract_sigma restatement on host threads (bench.py's CPU
    legs). Setup (strings, links, absorbed h2e, one n_det output per thread) happens here, outside
    the timed run()."""

    def __init__(self, rest, P, nthreads):
        L = rest.lib
        L.or_bench_create.restype = C.c_void_p
        L.or_bench_destroy.argtypes = [C.c_void_p]
        self.rest, self.nthreads = rest, int(nthreads)
        self.h = L.or_bench_create(*P.args(), self.nthreads)
        if not self.h:
            raise RuntimeError(L.or_last_error().decode())
        self.n_alpha = rest.binomial(P.norb, P.n_alpha)

    def run(self, x, nthreads, rows_per_thread, block_rows=4, row0=0):
        """Wall seconds of nthreads workers x rows_per_thread intermediate alpha rows each."""
        sec = C.c_double()
        self.rest._ck(self.rest.lib.or_bench_run(C.c_void_p(self.h), _dp(x), int(nthreads), C.c_int64(rows_per_thread),
                                                 int(block_rows), C.c_int64(row0), C.byref(sec)))
        return sec.value

    def close(self):
        if self.h:
            self.rest.lib.or_bench_destroy(C.c_void_p(self.h))
            self.h = None

    def __del__(self):
        self.close()


class Reference:
    """The reference library itself (oracle/_ref/libsbci_ref.so)."""

    PATH = os.path.join(HERE, "_ref", "libsbci_ref.so")

    @classmethod
    def available(cls):
        return os.path.exists(cls.PATH)

    def __init__(self):
        L = self.lib = C.CDLL(self.PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_num_strings.restype = C.c_int64

    def _ck(self, rc):
        if rc != 0:
            raise RuntimeError(f"[{rc}] " + self.lib.ref_last_error().decode())

    def strings(self, norb, k):
        out = np.zeros(self.lib.ref_num_strings(norb, k), np.uint64)
        self._ck(self.lib.ref_strings(norb, k, out.ctypes.data_as(_U64)))
        return out

    def links(self, norb, k):
        ns = int(self.lib.ref_num_strings(norb, k))
        n = ns * k * (norb - k + 1)
        p = np.zeros(n, np.uint16); q = np.zeros(n, np.uint16); t = np.zeros(n, np.uint32); s = np.zeros(n)
        rl = np.zeros(ns, np.int64)
        self._ck(self.lib.ref_links(norb, k, p.ctypes.data_as(C.c_void_p), q.ctypes.data_as(C.c_void_p),
                                    t.ctypes.data_as(C.c_void_p), _dp(s), rl.ctypes.data_as(C.c_void_p)))
        return p, q, t, s

    def diag(self, P):
        n = int(self.lib.ref_num_strings(P.norb, P.n_alpha) * self.lib.ref_num_strings(P.norb, P.n_beta))
        out = np.zeros(n)
        self._ck(self.lib.ref_diag(*P.args(), _dp(out)))
        return out

    def sigma(self, P, x):
        x = np.ascontiguousarray(x, np.float64)
        nvec = 1 if x.ndim == 1 else x.shape[0]
        y = np.zeros_like(x)
        self._ck(self.lib.ref_sigma(*P.args(), _dp(x), _dp(y), nvec))
        return y

    def solve(self, P, nroots, method=1, cfg=None, want_vectors=False, trace_csv=None):
        """method 1=sbci1, 2=sbci2, 3=davidson. cfg: dict of SolverConfig fields."""
        cfg = cfg or {}
        d = np.array([cfg.get(k, v) for k, v in (("eps0", 1e-10), ("r0", 1e-5), ("b_th", 1e-2), ("eps1", 1e-7),
                                                  ("x_th1", 0.1), ("x_th2", 1.2), ("r1", 1.0), ("lindep", 1e-14),
                                                  ("clamp_delta", 1e-10))])
        i = np.array([cfg.get("max_cycle", 0), cfg.get("t_max", 10000), cfg.get("hx_refresh_restarts", 5)], np.int64)
        e = np.zeros(nroots); it = np.zeros(nroots, np.int32); rs = np.zeros(nroots, np.int32); res = np.zeros(nroots)
        s2 = np.zeros(nroots); mv = np.zeros(1, np.uint64); wall = np.zeros(1)
        n = int(self.lib.ref_num_strings(P.norb, P.n_alpha) * self.lib.ref_num_strings(P.norb, P.n_beta))
        vec = np.zeros((nroots, n)) if want_vectors else None
        self._ck(self.lib.ref_solve(*P.args(), method, nroots, _dp(d), i.ctypes.data_as(C.c_void_p), _dp(e),
                                    it.ctypes.data_as(C.c_void_p), rs.ctypes.data_as(C.c_void_p), _dp(res),
                                    mv.ctypes.data_as(C.c_void_p), _dp(vec) if vec is not None else None, _dp(s2),
                                    _dp(wall), (trace_csv or "").encode()))
        return dict(energies=e, iterations=it, restarts=rs, residuals=res, matvecs=int(mv[0]), s_squared=s2,
                    wall_s=float(wall[0]), vectors=vec)

    def parse_fcidump(self, path):
        norb = C.c_int(); ne = C.c_int(); ms2 = C.c_int(); ec = C.c_double()
        self._ck(self.lib.ref_parse_fcidump(path.encode(), C.byref(norb), C.byref(ne), C.byref(ms2), C.byref(ec), None, None, 0))
        h1 = np.zeros(norb.value ** 2); eri = np.zeros(norb.value ** 4)
        self._ck(self.lib.ref_parse_fcidump(path.encode(), C.byref(norb), C.byref(ne), C.byref(ms2), C.byref(ec), _dp(h1), _dp(eri), norb.value))
        return Problem(norb.value, ne.value, ms2.value, ec.value, h1, eri, name=os.path.basename(path))

    def spin_squared(self, norb, na, nb, x):
        out = C.c_double()
        self._ck(self.lib.ref_spin_squared(norb, na, nb, _dp(np.ascontiguousarray(x, np.float64)), C.byref(out)))
        return out.value


# BASELINE.json configs. seed is pinned by this repo (BASELINE.json leaves it open).
BASELINE_SEED = 2603
CONFIGS = [
    dict(name="c0", norb=6, nelec=6, nroots=1, offdiag=0.05),
    dict(name="c1", norb=10, nelec=10, nroots=4, offdiag=0.05),
    dict(name="c2", norb=12, nelec=12, nroots=1, offdiag=0.05),
    dict(name="c3", norb=14, nelec=14, nroots=2, offdiag=0.05),
    dict(name="c4", norb=16, nelec=16, nroots=3, offdiag=0.08),
]


def baseline_problem(idx, rest=None):
    c = CONFIGS[idx]
    rest = rest or Restatement()
    h1, eri = rest.synthetic(c["norb"], BASELINE_SEED, c["offdiag"])
    return Problem(c["norb"], c["nelec"], 0, 0.0, h1, eri, name=c["name"])


class RefGpu:
    """oracle/_ref/libsbci_ref_gpu.so: the reference's own drivers on the B200 operator and the
    product's C++ drop-in header include/sbg.hpp (oracle/ref_gpu_shim.cpp)."""

    PATH = os.path.join(HERE, "_ref", "libsbci_ref_gpu.so")

    @classmethod
    def available(cls):
        return os.path.exists(cls.PATH)

    def __init__(self):
        self.lib = C.CDLL(self.PATH)
        self.lib.refgpu_last_error.restype = C.c_char_p

    def _err(self):
        return self.lib.refgpu_last_error().decode()

    def solve(self, P, nroots, method=1):
        e = np.zeros(nroots); it = np.zeros(nroots, np.int32); mv = np.zeros(1, np.uint64)
        rc = self.lib.refgpu_solve(*P.args(), method, nroots, _dp(e), it.ctypes.data_as(C.c_void_p),
                                   mv.ctypes.data_as(C.c_void_p))
        if rc != 0:
            raise RuntimeError(self._err())
        return dict(energies=e, iterations=it, matvecs=int(mv[0]))

    def device_solve(self, P, nroots, method=1, t_max=-1):
        """sbci::gpu::solve_n_states_* (include/sbg.hpp). Returns (rc, result dict)."""
        e = np.zeros(nroots); it = np.zeros(nroots, np.int32); mv = np.zeros(1, np.uint64)
        fs = C.c_int(-1)
        rc = self.lib.refgpu_device_solve(*P.args(), method, nroots, C.c_long(t_max), _dp(e),
                                          it.ctypes.data_as(C.c_void_p), mv.ctypes.data_as(C.c_void_p), C.byref(fs))
        return rc, dict(energies=e, iterations=it, matvecs=int(mv[0]), failed_state=fs.value, error=self._err())

    def concurrent_applies(self, P, nthreads, napply):
        bad = C.c_int(-2)
        rc = self.lib.refgpu_concurrent_applies(*P.args(), int(nthreads), int(napply), C.byref(bad))
        if rc != 0:
            raise RuntimeError(self._err())
        return bad.value

    def warm_start(self, P, with_defl):
        out = np.zeros(8)
        rc = self.lib.refgpu_warm_start(*P.args(), int(with_defl), _dp(out))
        if rc != 0:
            raise RuntimeError(self._err())
        return dict(e_ref=out[0], e_dev=out[1], it_ref=int(out[2]), it_dev=int(out[3]), overlap=out[4],
                    shift_ref=out[5], shift_dev=out[6])
