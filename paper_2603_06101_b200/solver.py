"""Python mirror of the reference's solver surface (config.hpp, sbci1.hpp:27-34/489-579,
trace.hpp:22-221); the solve itself runs in libsbg (C++ host driver + sm_100a kernels)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields

import numpy as np

from ._lib import TRACE_FN, Config, Stats, check, lib

RESTART_REASONS = ("stall_small_b", "norm_out_of_range", "residual_blowup", "max_cycle")


class NonConvergenceError(RuntimeError):
    """sbci::NonConvergenceError (config.hpp:92-100); CLI exit code 2."""

    def __init__(self, msg, state=-1, best_energy=float("nan"), best_residual=float("nan")):
        super().__init__(msg)
        self.state, self.best_energy, self.best_residual = state, best_energy, best_residual


@dataclass
class SolverConfig:
    """Thresholds, defaults = the paper's values (config.hpp:10-22)."""
    eps0: float = 1e-10
    r0: float = 1e-5
    b_th: float = 1e-2
    eps1: float = 1e-7
    x_th1: float = 0.1
    x_th2: float = 1.2
    r1: float = 1.0
    max_cycle: int = 0
    t_max: int = 10000
    lindep: float = 1e-14
    clamp_delta: float = 1e-10
    hx_refresh_restarts: int = 5

    def effective_max_cycle(self, method_default: int) -> int:
        return self.max_cycle if self.max_cycle > 0 else method_default

    def to_c(self) -> Config:
        c = Config()
        for f in fields(self):
            setattr(c, f.name, getattr(self, f.name))
        return c

    def validate(self):
        c = self.to_c()
        check(lib().sbg_config_validate(C.byref(c)))

    @staticmethod
    def preset(name: str) -> "SolverConfig":
        if name == "tight":
            return SolverConfig(eps0=1e-10, r0=1e-5)
        if name == "loose":
            return SolverConfig(eps0=1e-8, r0=1e-4)
        raise ValueError(f"unknown preset '{name}' (expected tight or loose)")


@dataclass
class ConvergedEigenpair:
    state: int
    energy: float
    vector: np.ndarray
    iterations: int
    restarts: int
    final_residual: float


@dataclass
class StateSummary:
    state: int
    energy: float
    iterations: int
    restarts: int
    final_residual: float
    s_squared: float = float("nan")


@dataclass
class RunSummary:
    method: str = "sbci1"
    states: list = field(default_factory=list)
    total_iterations: int = 0
    total_restarts: int = 0
    matvecs: int = 0
    hx_refreshes: int = 0
    peak_vectors: int = 0
    wall_time_s: float = 0.0
    kernel_launches: int = 0
    device_vectors_peak: int = 0   # length-n_det solver vectors resident at once (HBM footprint)

    def energies(self):
        return [s.energy for s in self.states]


@dataclass
class TraceRecord:
    """TraceRecord (trace.hpp:22-44); fields a method does not produce are NaN."""
    method: str
    state: int
    t: int
    energy: float
    dE: float
    res_norm: float
    x_norm: float
    kinetic: float
    matvecs: int
    restart_reason: str
    b: float
    c: float
    pair_partner: int = -1
    b_ab: float = float("nan")
    b_ba: float = float("nan")
    b_bb: float = float("nan")
    c_ab: float = float("nan")
    c_ba: float = float("nan")
    c_bb: float = float("nan")
    a_ab: float = float("nan")
    a_ba: float = float("nan")
    energy_partner: float = float("nan")
    x_norm_partner: float = float("nan")
    res_norm_partner: float = float("nan")


METHODS = {1: "sbci1", 2: "sbci2", 3: "davidson"}


@dataclass
class MultiStateResult:
    pairs: list
    summary: RunSummary


def _trace_cb(sink, name):
    if sink is None:
        return TRACE_FN(0)

    def _cb(rec_p, _user):
        r = rec_p.contents
        sink(TraceRecord(METHODS.get(r.method, name), r.state, r.t, r.energy, r.dE, r.res_norm, r.x_norm,
                         r.kinetic, r.matvecs,
                         RESTART_REASONS[r.restart_reason] if r.restart_reason >= 0 else "", r.b, r.c,
                         r.pair_partner, r.b_ab, r.b_ba, r.b_bb, r.c_ab, r.c_ba, r.c_bb, r.a_ab, r.a_ba,
                         r.energy_partner, r.x_norm_partner, r.res_norm_partner))
    return TRACE_FN(_cb)


def _solve(op, method: int, n: int, cfg: SolverConfig | None, sink, want_vectors: bool, max_space: int = 0):
    cfg = cfg or SolverConfig()
    cfg.validate()
    name = METHODS[method]
    if n < 1:
        raise ValueError(f"solve_n_states_{name}: n must be >= 1")
    dim = op.dim()
    e = np.zeros(n)
    vec = np.zeros((n, dim)) if want_vectors else None
    st = Stats()
    cc = cfg.to_c()
    cb = _trace_cb(sink, name)
    ep = e.ctypes.data_as(C.POINTER(C.c_double))
    vp = vec.ctypes.data_as(C.POINTER(C.c_double)) if vec is not None else None
    if method == 3 and max_space:
        rc = lib().sbg_solve_davidson(op.handle, n, max_space, C.byref(cc), ep, vp, C.byref(st), cb, None)
    else:
        rc = lib().sbg_solve(op.handle, method, n, C.byref(cc), ep, vp, C.byref(st), cb, None)
    if rc == 2:
        raise NonConvergenceError(lib().sbg_last_error().decode(), st.failed_state, st.best_energy, st.best_residual)
    check(rc)
    pairs, states = [], []
    for k in range(n):
        pairs.append(ConvergedEigenpair(k, float(e[k]), vec[k] if vec is not None else None, st.iterations[k],
                                        st.restarts[k], st.final_residual[k]))
        states.append(StateSummary(k, float(e[k]), st.iterations[k], st.restarts[k], st.final_residual[k],
                                   float(st.s_squared[k])))
    summ = RunSummary(name, states, st.total_iterations, st.total_restarts, st.matvecs, st.hx_refreshes,
                      st.peak_vectors, st.wall_time_s, st.kernel_launches, st.device_vectors_peak)
    return MultiStateResult(pairs, summ)


def solve_n_states_sbci1(op, n: int, cfg: SolverConfig | None = None, sink=None, want_vectors: bool = True):
    """Sequential lowest-n SBCI1 driver (sbci1.hpp:526-579) on the GPU operator.
    `sink` is a callable receiving TraceRecord per iteration (TraceSink::record)."""
    return _solve(op, 1, n, cfg, sink, want_vectors)


def solve_n_states_sbci2(op, n: int, cfg: SolverConfig | None = None, sink=None, want_vectors: bool = True):
    """Pair-sequential lowest-n SBCI2 driver (sbci2.hpp:527-623) on the GPU operator: pairs
    (0,1), (1,2), ... with the upper iterate seeding the next pair; the last state runs SBCI1.
    n = 1 routes to SBCI1 (the summary still says "sbci2", as the reference's does)."""
    r = _solve(op, 2, n, cfg, sink, want_vectors)
    return r


def davidson_solve(op, nroots: int, cfg: SolverConfig | None = None, sink=None, want_vectors: bool = True,
                   max_space: int = 0):
    """Block Davidson (davidson.hpp:228-244: eps0/r0/lindep from cfg, 400 iterations) on the GPU
    operator, with the SBCI solvers' (D - E0)^-1 preconditioner. max_space = DavidsonConfig::max_space
    (davidson.hpp:19-38): 0 = 12*nroots, else >= 2*nroots."""
    return _solve(op, 3, nroots, cfg, sink, want_vectors, max_space)


@dataclass
class Sbci1Result:
    """Sbci1Result (sbci1.hpp:344-349) of a single-state solve; next_seed is not exposed."""
    pair: ConvergedEigenpair
    converged_image: np.ndarray
    hx_refreshes: int
    matvecs: int
    s_squared: float
    shift: float    # the preconditioner's shift after the solve (tracks E for alpha == 0)


def solve_state_sbci1(op, x0, E0: float, shift: float, deflation=(), cfg: SolverConfig | None = None, alpha: int = 0,
                      sink=None) -> Sbci1Result:
    """Plain-vector warm start (solve_state_sbci1(op, pre, defl, x0, E0, cfg, alpha, sink),
    sbci1.hpp:477-486): pre = GroundShiftPreconditioner(op.diagonal(), shift, cfg.clamp_delta);
    `deflation` is a sequence of (unit vector, energy) or (vector, image, energy) entries
    (DeflationSet::add / add_with_image, precond.hpp:54-70)."""
    cfg = cfg or SolverConfig()
    cfg.validate()
    n = op.dim()
    x0 = np.ascontiguousarray(x0, np.float64)
    if x0.shape != (n,):
        raise ValueError("SymmetricOperator::apply: dimension mismatch")
    dx = [np.ascontiguousarray(d[0], np.float64) for d in deflation]
    dh = [np.ascontiguousarray(d[1], np.float64) for d in deflation if len(d) == 3]
    de = np.array([float(d[-1]) for d in deflation])
    if dh and len(dh) != len(dx):
        raise ValueError("deflation entries must all carry images, or none")
    X = np.stack(dx) if dx else None
    H = np.stack(dh) if dh else None
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None  # noqa: E731
    sh = C.c_double(shift)
    en = C.c_double()
    vec = np.zeros(n)
    img = np.zeros(n)
    st = Stats()
    cc = cfg.to_c()
    cb = _trace_cb(sink, "sbci1")
    rc = lib().sbg_solve_state_sbci1(op.handle, dp(x0), float(E0), C.byref(sh), int(alpha), len(dx), dp(X), dp(H),
                                     dp(de) if len(dx) else None, C.byref(cc), C.byref(en), dp(vec), dp(img),
                                     C.byref(st), cb, None)
    if rc == 2:
        raise NonConvergenceError(lib().sbg_last_error().decode(), st.failed_state, st.best_energy, st.best_residual)
    check(rc)
    pair = ConvergedEigenpair(int(alpha), en.value, vec, st.iterations[0], st.restarts[0], st.final_residual[0])
    return Sbci1Result(pair, img, st.hx_refreshes, st.matvecs, float(st.s_squared[0]), sh.value)
