"""Command-line front end on the GPU operator: the reference's `sbci fci / solve / compare`
(proj/tools/sbci_cli.cpp) with the same flags, config precedence, printed table, JSON summary
schema and exit codes, for FCIDUMP input.

    python -m paper_2603_06101_b200.cli fci --fcidump F [--nroots n] [--method sbci1|sbci2|davidson]
        [--ms2 m] [--trace out.csv] [--summary out.json] [--preset tight|loose] [--config cfg.json]
        [--eps0 ..] [--r0 ..] ... [--max-space m] [--max-determinants N] [--device d]
    python -m paper_2603_06101_b200.cli solve --fcidump F ...      (same as fci)
    python -m paper_2603_06101_b200.cli compare --fcidump F [--nroots n] [--summary out.json]

Behaviour mirrored from the reference:
  * config precedence preset < JSON file < explicit flags, then SolverConfig::validate
    (sbci_cli.cpp:58-96);
  * sector from the FCIDUMP header unless --ms2 (sbci_cli.cpp:103-116), operator through
    as_operator with the 5e6-determinant guard (fci_operator.hpp:103-120) — --max-determinants is
    this build's addition so the (14e,14o)/(16e,16o) sectors can be reached from the command line;
  * summary JSON with exactly the 9 keys of summary_to_json (sbci_cli.cpp:140-166), per-state
    s_squared from fci::spin_squared (attach_spin, :175-181);
  * table print (print_summary, :183-195) with the S^2 column;
  * --trace writes the per-iteration CSV of CsvTraceSink (trace.hpp:69-119);
  * exit codes: 0 ok, 1 usage / parse / I/O / invalid argument, 2 NonConvergenceError
    (sbci_cli.cpp:367-386).
Out of scope: Matrix Market input (`--input`), `gen` and `conserve` — asking for
them exits 1 with a message.
"""
from __future__ import annotations

import argparse
import json
import math
import sys

CONFIG_KEYS = ("eps0", "r0", "b_th", "eps1", "x_th1", "x_th2", "r1", "max_cycle", "t_max", "lindep",
               "clamp_delta", "hx_refresh_restarts")
# flag -> SolverConfig field (add_config_flags, sbci_cli.cpp:35-50)
FLAG_FIELDS = (("--eps0", "eps0", float), ("--r0", "r0", float), ("--b-th", "b_th", float),
               ("--eps1", "eps1", float), ("--x-th1", "x_th1", float), ("--x-th2", "x_th2", float),
               ("--r1", "r1", float), ("--max-cycle", "max_cycle", int), ("--t-max", "t_max", int),
               ("--lindep", "lindep", float), ("--clamp-delta", "clamp_delta", float))
SUMMARY_KEYS = ("method", "energies", "states", "total_iterations", "total_restarts", "matvecs", "hx_refreshes",
                "peak_vectors", "wall_time_s")


class UsageError(Exception):
    """CLI::ParseError / CLI::ValidationError: exit code 1."""


class _Parser(argparse.ArgumentParser):
    def error(self, message):          # argparse would exit 2; the reference's parse errors exit 1
        raise UsageError(message)


def build_parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="sbci", description="SBCI eigensolvers for determinant CI on the B200 sigma operator")
    sub = ap.add_subparsers(dest="cmd")

    def config_flags(p):
        p.add_argument("--preset", choices=("tight", "loose"))
        p.add_argument("--config", dest="config_path", default="")
        for flag, dest, typ in FLAG_FIELDS:
            p.add_argument(flag, dest=dest, type=typ, default=None)
        p.add_argument("--max-space", type=int, default=0, help="davidson subspace cap (default 12*nroots)")

    def input_flags(p, required):
        p.add_argument("--fcidump", required=required, default="")
        p.add_argument("--input", default="", help="Matrix Market input (not supported by the GPU operator)")
        p.add_argument("--ms2", type=int, default=None)
        p.add_argument("--max-determinants", type=int, default=None,
                       help="override the 5e6-determinant guard of as_operator")
        p.add_argument("--device", type=int, default=0)

    for name, req in (("solve", False), ("fci", True)):
        p = sub.add_parser(name)
        input_flags(p, req)
        p.add_argument("--method", default="sbci1", choices=("sbci1", "sbci2", "davidson"))
        p.add_argument("--nroots", type=int, default=1)
        p.add_argument("--trace", default="")
        p.add_argument("--summary", default="")
        config_flags(p)
    p = sub.add_parser("compare")
    input_flags(p, False)
    p.add_argument("--nroots", type=int, default=1)
    p.add_argument("--summary", default="")
    config_flags(p)
    for name in ("gen", "conserve"):
        sub.add_parser(name, add_help=False).add_argument("rest", nargs=argparse.REMAINDER)
    return ap


def resolve_config(args):
    """preset < JSON config file < explicit flags, then validate (sbci_cli.cpp:58-96)."""
    from .solver import SolverConfig
    cfg = SolverConfig.preset(args.preset) if args.preset else SolverConfig()
    if args.config_path:
        try:
            with open(args.config_path) as f:
                j = json.load(f)
        except OSError:
            raise RuntimeError(f"cannot open config file {args.config_path}")
        for key in CONFIG_KEYS:
            if key in j:
                setattr(cfg, key, type(getattr(cfg, key))(j[key]))
    for _, dest, _ in FLAG_FIELDS:
        v = getattr(args, dest)
        if v is not None:
            setattr(cfg, dest, v)
    cfg.validate()
    return cfg


def load_operator(args):
    """load_problem (sbci_cli.cpp:103-116) on the GPU operator."""
    from .fci import K_DEFAULT_DETERMINANT_GUARD, as_operator, parse_fcidump_file
    if bool(args.input) == bool(args.fcidump):
        raise UsageError("exactly one of --input or --fcidump is required")
    if args.input:
        raise UsageError("--input (Matrix Market) is outside this build's scope: the GPU operator is the FCI "
                         "sigma; pass --fcidump")
    prob = parse_fcidump_file(args.fcidump)
    ms2 = prob.ms2 if args.ms2 is None else args.ms2
    guard = args.max_determinants if args.max_determinants is not None else K_DEFAULT_DETERMINANT_GUARD
    return as_operator(prob, ms2, max_determinants=guard, device=args.device)


def run_method(method, op, nroots, cfg, max_space, sink):
    """run_method (sbci_cli.cpp:118-138)."""
    from .solver import davidson_solve, solve_n_states_sbci1, solve_n_states_sbci2
    if method == "sbci1":
        return solve_n_states_sbci1(op, nroots, cfg, sink, want_vectors=False)
    if method == "sbci2":
        return solve_n_states_sbci2(op, nroots, cfg, sink, want_vectors=False)
    if method == "davidson":
        return davidson_solve(op, nroots, cfg, sink, want_vectors=False, max_space=max_space)
    raise UsageError(f"unknown method '{method}'")


def summary_to_json(s) -> dict:
    """summary_to_json (sbci_cli.cpp:140-166): exactly the documented 9 keys, in order."""
    states = []
    for st in s.states:
        states.append({"state": st.state, "energy": st.energy, "iterations": st.iterations,
                       "restarts": st.restarts, "final_residual": st.final_residual,
                       "s_squared": None if math.isnan(st.s_squared) else st.s_squared})
    return {"method": s.method, "energies": s.energies(), "states": states,
            "total_iterations": s.total_iterations, "total_restarts": s.total_restarts, "matvecs": s.matvecs,
            "hx_refreshes": s.hx_refreshes, "peak_vectors": s.peak_vectors, "wall_time_s": s.wall_time_s}


def write_summary_file(path, j):
    if not path:
        return
    try:
        with open(path, "w") as f:
            f.write(json.dumps(j, indent=2) + "\n")
    except OSError:
        raise RuntimeError(f"cannot open {path} for writing")


def print_summary(res, out=None):
    """print_summary (sbci_cli.cpp:183-195), FCI form (with the S^2 column)."""
    out = out or sys.stdout
    out.write(f"{'state':<6} {'energy (hartree)':<20} {'iters':<6} {'restarts':<9} {'|res|':<12}  S^2\n")
    for st in res.summary.states:
        out.write(f"{st.state:<6d} {st.energy:<20.12f} {st.iterations:<6d} {st.restarts:<9d} "
                  f"{st.final_residual:<12.3e}  {st.s_squared:.6f}\n")
    s = res.summary
    out.write(f"matvecs {s.matvecs}, iterations {s.total_iterations}, restarts {s.total_restarts}, "
              f"peak vectors {s.peak_vectors}, wall {s.wall_time_s:.3f} s\n")


def cmd_solve(args) -> int:
    from .trace import CsvTraceSink
    if args.nroots < 1:
        raise UsageError("--nroots must be positive")
    cfg = resolve_config(args)
    op = load_operator(args)
    try:
        if args.trace:
            try:
                sink = CsvTraceSink(args.trace)
            except OSError:
                raise RuntimeError(f"cannot open trace file {args.trace}")
            with sink:
                res = run_method(args.method, op, args.nroots, cfg, args.max_space, sink)
        else:
            res = run_method(args.method, op, args.nroots, cfg, args.max_space, None)
    finally:
        op.close()
    print_summary(res)
    write_summary_file(args.summary, summary_to_json(res.summary))
    return 0


def cmd_compare(args) -> int:
    """cmd_compare (sbci_cli.cpp:216-252): all three methods on one operator."""
    if args.nroots < 1:
        raise UsageError("--nroots must be positive")
    cfg = resolve_config(args)
    op = load_operator(args)
    try:
        results = [run_method(m, op, args.nroots, cfg, args.max_space, None) for m in ("sbci1", "sbci2", "davidson")]
    finally:
        op.close()
    out = sys.stdout
    out.write(f"{'state':<6} {'E_sbci1':<20} {'E_sbci2':<20} {'E_davidson':<20} {'d(1-Dv)':<12} {'d(2-Dv)':<12}\n")
    for k in range(args.nroots):
        e1, e2, ed = (r.pairs[k].energy for r in results)
        out.write(f"{k:<6d} {e1:<20.12f} {e2:<20.12f} {ed:<20.12f} {e1 - ed:<12.3e} {e2 - ed:<12.3e}\n")
    out.write(f"{'method':<10} {'matvecs':<10} {'iterations':<12} {'restarts':<10} {'wall_s':<10}\n")
    for r in results:
        s = r.summary
        out.write(f"{s.method:<10} {s.matvecs:<10d} {s.total_iterations:<12d} {s.total_restarts:<10d} "
                  f"{s.wall_time_s:<10.3f}\n")
    if args.summary:
        write_summary_file(args.summary, {r.summary.method: summary_to_json(r.summary) for r in results})
    return 0


def main(argv=None) -> int:
    from .fci import FcidumpError
    from .solver import NonConvergenceError
    try:
        args = build_parser().parse_args(argv)
        if args.cmd is None:
            raise UsageError("a subcommand is required: solve, fci or compare")
        if args.cmd in ("gen", "conserve"):
            raise UsageError(f"'{args.cmd}' (synthetic sparse matrices / trace conservation report) is outside "
                             "this build's scope")
        if args.cmd == "compare":
            return cmd_compare(args)
        return cmd_solve(args)
    except UsageError as e:
        sys.stderr.write(f"error: {e}\n")
        return 1
    except NonConvergenceError as e:
        sys.stderr.write(f"error: {e}\n")
        return 2
    except (ValueError, RuntimeError, OSError, FcidumpError) as e:
        sys.stderr.write(f"error: {e}\n")
        return 1


if __name__ == "__main__":
    sys.exit(main())
