#!/usr/bin/env python
"""bench.py — sigma = H.c builds per second for the SBCI hot path (BASELINE.json metric), B200.

Workload (N=1 default): BASELINE configs[4], (16e,16o) Ms=0, 165,636,900 determinants, fp64,
pinned synthetic integrals (seed 2603, L^k off-diagonal scale 0.08) — the largest configuration
and the one the north star's roofline target is quoted on. A "step" is one full sigma build
(y = H x over the whole CI vector, 1.33 GB in / 1.33 GB out, inputs > L2 so no flush needed).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4] [--impl ours|reference]

N > 1 is launched by torchrun: one rank per GPU, the CI vector sharded by alpha-string blocks,
NCCL all-gather of x + all-reduce + alpha-alpha block exchange inside libsbg ("scaling": strong —
the total work per step is fixed). The timed region is bracketed by a barrier + device sync on
both sides and the max over ranks is reported.

--impl reference times the reference's CPU algorithm on the host cores: the reference library
itself cannot build a (16e,16o) sigma (678 GB workspace), so the blocked restatement
of contract_sigma (oracle/sbci_oracle.cpp, bit-exact with the reference at <= (10e,10o)) runs a
bounded sample of intermediate alpha rows on all host threads and the sigma rate is extrapolated.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {"c2": (12, 12, 0.05), "c3": (14, 14, 0.05), "c4": (16, 16, 0.08)}
SEED = 2603
METRIC = "sigma_builds_per_s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tte", action="store_true", help="skip the time-to-energy solves")
    ap.add_argument("--tte-full", action="store_true", help="also solve c4 (3 roots, SBCI1/SBCI2/Davidson, ~15 min)")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.samples, self._stop = index, [], threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
                f = [x.strip() for x in out.strip().split(",")]
                if len(f) == 7:
                    self.samples.append(f)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for s in self.samples:
            for n, v in zip(names, s[3:]):
                if v.strip().lower() in ("active", "1"):
                    reasons.add(n)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": float(self.samples[0][1]),
                "reasons": sorted(reasons), "samples": len(self.samples)}


def cpu_baseline(cfg_name, threads=None, rows_per_thread=None):
    """Reference algorithm (blocked contract_sigma restatement) on the host cores: bounded sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    from oracle import Problem, Restatement
    import paper_2603_06101_b200 as P
    norb, ne, sc = CONFIGS[cfg_name]
    p = P.synthetic_problem(norb, ne, SEED, sc)
    q = Problem(p.norb, p.nelec, p.ms2, p.e_core, p.h1, p.eri)
    rest = Restatement()
    na = rest.binomial(norb, ne // 2)
    threads = threads or os.cpu_count() or 1
    rpt = rows_per_thread or {"c2": 58, "c3": 64, "c4": 12}[cfg_name]
    x = np.random.default_rng(7).uniform(-1, 1, na * na)
    t0 = time.perf_counter()
    rest.sigma_sample(q, x, threads, rpt, block_rows=min(rpt, 4))
    t = time.perf_counter() - t0
    rows = threads * rpt
    sigma_s = t * na / rows          # rows run concurrently on `threads` cores
    return {"value": 1.0 / sigma_s, "unit": "sigma/s", "cores": threads, "kind": "port",
            "sample": f"{rows} of {na} intermediate alpha rows of the blocked contract_sigma restatement "
                      f"(oracle/sbci_oracle.cpp:or_sigma_sample), {threads} threads x {rpt} rows, {t:.1f} s; "
                      f"extrapolated to one full sigma ({sigma_s:.0f} s)",
            "seconds": t}


def dgemm_peak_tflops(torch):
    n = 4096
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn_like(a)
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        a @ b
    e1.record()
    torch.cuda.synchronize()
    return 2 * n ** 3 * 10 / (e0.elapsed_time(e1) * 1e-3) / 1e12


def sigma_roofline(norb, n_el, n_det, flops, ms_step, peak_tflops, world=1):
    """Whole-sigma roofline two ways: (1) this build's executed useful flops against the
    measured DGEMM peak plus 16 n_det bytes against the HBM peak; (2) the SURVEY's algorithmic count
    F_sigma = 2 n_det (norb^2 L + 2 W + L), L = n(norb-n+1), W = 1 + n(norb-n) + C(n,2) C(norb-n,2),
    which the pair-resolved factorization here undercuts (ratio > 1 = faster than that roofline).
    Peaks are per GPU times `world` (the whole job)."""
    if not peak_tflops:
        return None
    from math import comb
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            bw = float(json.load(f)["hbm_gbs"]) * 1e9 * world
    except Exception:
        bw = 7.7e12 * world
    L = n_el * (norb - n_el + 1)
    W = 1 + n_el * (norb - n_el) + comb(n_el, 2) * comb(norb - n_el, 2)
    f_survey = 2.0 * n_det * (norb * norb * L + 2 * W + L)
    t_bytes = 16.0 * n_det / bw
    t_own = flops["total"] / (peak_tflops * 1e12) + t_bytes
    t_survey = f_survey / (peak_tflops * 1e12) + t_bytes
    t = ms_step * 1e-3
    return {"hbm_gbs": bw / 1e9, "fp64_tflops": peak_tflops, "executed_flops": flops["total"],
            "frac_executed": t_own / t, "survey_F_sigma": f_survey, "frac_survey": t_survey / t}


def profile_traffic(cfg_name):
    path = os.path.join(ROOT, "profiles", "ab_kernel_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)[cfg_name]["dram_bytes_per_launch"]   # ncu --set full, per launch
    except Exception:
        return None


def time_to_energy(full=False):
    """Second half of the BASELINE metric: solves on the GPU through the public API (reference
    SolverConfig defaults), wall time of the solver call with the operator built. c1/c2: energies vs
    the reference's own converged energies (tests/golden, produced by the compiled reference on the
    same pinned integrals) and the reference's single-core wall time. c3 (and c4 with --tte-full),
    where the serial reference has no energies: SBCI1 vs GPU block Davidson."""
    import numpy as np
    import paper_2603_06101_b200 as P
    out = {}
    runs = [("c1", (10, 10, 0.05), 4, ("sbci1", "sbci2", "davidson")), ("c2", (12, 12, 0.05), 1, ("sbci1",)),
            ("c3", (14, 14, 0.05), 2, ("sbci1", "davidson"))]
    if full:
        runs.append(("c4", (16, 16, 0.08), 3, ("sbci1", "sbci2", "davidson")))
    solvers = {"sbci1": P.solve_n_states_sbci1, "sbci2": P.solve_n_states_sbci2, "davidson": P.davidson_solve}
    for tag, (norb, ne, sc), nroots, methods in runs:
        ref = {}
        gpath = os.path.join(ROOT, "tests", "golden", f"golden_{tag}.json")
        if os.path.exists(gpath):
            with open(gpath) as f:
                ref = json.load(f)
        op = P.FciOperator(P.synthetic_problem(norb, ne, SEED, sc), max_determinants=2 ** 62)
        P.solve_n_states_sbci1(op, 1, want_vectors=False)          # warm-up (module load, first launches)
        rec = {"nroots": nroots}
        energies = {}
        for m in methods:
            solvers[m](op, nroots, want_vectors=False)    # warm-up: lazy module loading of its kernels
            t0 = time.perf_counter()
            res = solvers[m](op, nroots, want_vectors=False)
            wall = time.perf_counter() - t0
            e = np.array([p.energy for p in res.pairs])
            energies[m] = e
            r = {"seconds": wall, "sigma_builds": res.summary.matvecs, "iterations": res.summary.total_iterations,
                 "energies": e.tolist(), "s_squared": [s.s_squared for s in res.summary.states]}
            if m in ref:
                r["max_abs_dE_vs_reference_Eh"] = float(np.abs(e - np.array(ref[m]["energies"])).max())
                r["reference_seconds_1core"] = ref[m]["wall_s"]
                r["reference_sigma_builds"] = ref[m]["matvecs"]
            rec[m] = r
        # time until every requested state is within 1e-8 Eh of its target: the
        # reference's converged energies where it ran (c1, c2), else the GPU Davidson energies;
        # measured in a second, traced run (the trace callback adds one small pass per iteration)
        target = np.array(ref["sbci1"]["energies"]) if "sbci1" in ref else energies.get("davidson")
        if target is not None:
            for m in methods:
                stamps = []
                base = op.apply_count()
                t0 = time.perf_counter()
                solvers[m](op, nroots, want_vectors=False,
                           sink=lambda rr: stamps.append((time.perf_counter() - t0, rr.energy, rr.matvecs)))
                hit = []
                for ek in target:
                    first = next(((t, mv) for t, en, mv in stamps if abs(en - ek) < 1e-8), None)
                    hit.append(first)
                if all(h is not None for h in hit):
                    rec[m]["seconds_to_1e-8_Eh"] = max(h[0] for h in hit)
                    rec[m]["sigma_builds_to_1e-8_Eh"] = max(h[1] for h in hit) - base
        if "davidson" in energies and "sbci1" in energies and not ("sbci1" in ref):
            rec["max_abs_dE_sbci1_vs_davidson_Eh"] = float(np.abs(energies["sbci1"] - energies["davidson"]).max())
        out[tag] = rec
        op.close()
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # warm-up: one sample (page-in, thread start-up); each timed step is one bounded sample
    cpu_baseline(args.config)
    samples = [cpu_baseline(args.config) for _ in range(args.steps)]
    rates = sorted(s["value"] for s in samples)
    value = rates[len(rates) // 2]
    info = samples[len(samples) // 2]
    norb, ne = CONFIGS[args.config][0], CONFIGS[args.config][1]
    n_det = math.comb(norb, ne // 2) ** 2
    out = {"metric": METRIC, "value": value, "unit": "sigma/s", "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / value, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (pinned BASELINE generator, seed 2603)",
           "config": {"workload": f"{args.config} sigma build (BASELINE configs[{ {'c2': 2, 'c3': 3, 'c4': 4}[args.config]}])",
                      "norb": norb, "nelec": ne, "ms2": 0, "n_det": n_det, "vector_bytes": n_det * 8,
                      "parallelism": f"host cores ({info['cores']} threads)"},
           "cpu_baseline": {k: info[k] for k in ("value", "unit", "cores", "kind", "sample")},
           "e2e": {"value": value, "unit": "sigma/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_ours(args):
    import numpy as np
    import torch
    import paper_2603_06101_b200 as P
    from paper_2603_06101_b200 import _lib, dist as pdist

    rank, world, local = pdist.env_rank_world()
    if world != args.gpus:
        world = max(world, 1)
    torch.cuda.set_device(local)
    tdist = None
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = _lib.lib()
    norb, ne, sc = CONFIGS[args.config]
    prob = P.synthetic_problem(norb, ne, SEED, sc)
    nccl_id = pdist.broadcast_nccl_id(rank) if world > 1 else None
    op = P.FciOperator(prob, max_determinants=2 ** 62, device=local, rank=rank, world=world, nccl_id=nccl_id)
    h = op.handle
    n = op.dim()
    pl = L.sbg_padded_len(h)
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    with torch.cuda.stream(stream):
        xd = torch.empty(n, dtype=torch.float64, device="cuda")
        g = torch.Generator(device="cuda")
        g.manual_seed(7)
        xd.uniform_(-1.0, 1.0, generator=g)
        x = torch.empty(pl, dtype=torch.float64, device="cuda")
        y = torch.empty(pl, dtype=torch.float64, device="cuda")
        _lib.check(L.sbg_pack(h, C.c_void_p(xd.data_ptr()), C.c_void_p(x.data_ptr()), C.c_void_p(sp)))
    stream.synchronize()
    del xd
    flops = op.sigma_flops()

    def barrier():
        if tdist is not None:
            tdist.barrier()

    for _ in range(args.warmup):
        _lib.check(L.sbg_sigma_padded(h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), C.c_void_p(sp)))
    stream.synchronize()
    peak = dgemm_peak_tflops(torch) if rank == 0 else None
    barrier()
    torch.cuda.synchronize()
    _lib.check(L.sbg_profile_reset(h))
    launches0 = op.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            _lib.check(L.sbg_sigma_padded(h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), C.c_void_p(sp)))
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = e0.elapsed_time(e1)
    launches = op.kernel_launches() - launches0
    prof = (C.c_double * 4)()
    calls = C.c_int64()
    _lib.check(L.sbg_profile_read(h, prof, C.byref(calls)))
    ms_ab = prof[0] / max(calls.value, 1)
    ms_ss = prof[1] / max(calls.value, 1)   # same-spin kernels + transposes (+ all-gather wait)
    if tdist is not None:
        t = torch.tensor([ms, ms_ab, ms_ss], dtype=torch.float64, device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms, ms_ab, ms_ss = t.tolist()
    ms_step = ms / args.steps
    value = 1000.0 / ms_step

    # end to end through the public C ABI: pinned host x -> H2D -> sigma -> D2H for every step; one
    # sbg_sigma call over e2e_steps vectors, which overlaps the copies of neighbouring steps with
    # the sigma builds (the library's two-slot pipeline)
    nvec = args.e2e_steps
    while True:   # 2 x nvec pinned host vectors (16 GB at c4 with 6); fewer if the host cannot pin that much
        try:
            xh = torch.empty((nvec, n), dtype=torch.float64, pin_memory=True)
            yh = torch.empty((nvec, n), dtype=torch.float64, pin_memory=True)
            break
        except RuntimeError:
            xh = yh = None
            if nvec <= 2:
                raise
            nvec = max(2, nvec // 2)
    xh.uniform_(-1.0, 1.0)
    dp = C.POINTER(C.c_double)
    xp = C.cast(C.c_void_p(xh.data_ptr()), dp)
    yp = C.cast(C.c_void_p(yh.data_ptr()), dp)
    _lib.check(L.sbg_sigma(h, xp, yp, min(nvec, 2)))   # warm-up (staging buffers, copy streams)
    barrier()
    t0 = time.perf_counter()
    _lib.check(L.sbg_sigma(h, xp, yp, nvec))
    te = time.perf_counter() - t0
    if tdist is not None:
        t = torch.tensor([te], dtype=torch.float64, device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        te = t.item()
    e2e = nvec / te
    local_bytes = (op.row_hi - op.row_lo) * op.n_beta_strings * 8

    if rank == 0:
        clocks = clk.summary()
        achieved = flops["alpha_beta"] / (ms_ab * 1e-3) / 1e12 if ms_ab > 0 else None
        out = {
            "metric": METRIC, "value": value, "unit": "sigma/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (pinned BASELINE generator, seed 2603)",
            "config": {"workload": f"{args.config} sigma build (BASELINE configs[{ {'c2': 2, 'c3': 3, 'c4': 4}[args.config]}])",
                       "norb": norb, "nelec": ne, "ms2": 0, "n_det": n, "vector_bytes": n * 8,
                       "parallelism": f"alpha-row shards x{world}" if world > 1 else "single GPU",
                       "l2": "inputs larger than L2 (no flush needed)"},
            "e2e": {"value": e2e, "unit": "sigma/s", "h2d_bytes_per_step": local_bytes * world,
                    "d2h_bytes_per_step": local_bytes * world},
            "gpu_launches": launches,
            "roofline": {"kernel": "k_sigma_ab (gather -> DMMA -> scatter)", "bound": "tensor",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": (achieved / peak) if (achieved and peak) else None,
                         "peak_source": "cuBLAS DGEMM 4096^3 fp64 measured in this run (MEASURED_PEAKS.json has no fp64)",
                         "flops_per_launch": flops["alpha_beta"], "ms_per_launch": ms_ab,
                         "traffic": profile_traffic(args.config)},
            "roofline_same_spin": {"kernel": "k_sigma_ss x2 + 2 transposes (alpha-alpha, beta-beta)", "bound": "tensor",
                                   "achieved": flops["same_spin"] / (ms_ss * 1e-3) / 1e12 if ms_ss > 0 else None,
                                   "peak": peak, "unit": "TFLOP/s",
                                   "frac": (flops["same_spin"] / (ms_ss * 1e-3) / 1e12 / peak) if (ms_ss > 0 and peak) else None,
                                   "ms_per_sigma": ms_ss},
            "sigma_flops": flops,
            "sigma_tflops": flops["total"] / (ms_step * 1e-3) / 1e12,
            "sigma_roofline": sigma_roofline(norb, ne // 2, n, flops, ms_step, peak * world if peak else None,
                                             world),
            "clocks": clocks,
        }
        if world == 1 and not args.no_tte:
            out["time_to_energy"] = time_to_energy(args.tte_full)
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_baseline(args.config)
            out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        print(json.dumps(out), flush=True)
    op.close()
    if tdist is not None:
        tdist.barrier()
        tdist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
