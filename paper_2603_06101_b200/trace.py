"""Trace sinks (trace.hpp:17-180): the solvers report one TraceRecord per iteration through the
`sink` callable of solve_n_states_sbci1/_sbci2/davidson_solve; these classes are the reference's
MemoryTraceSink, CsvTraceSink (same header, same 17-significant-digit cells, NaN = empty cell),
TeeTraceSink and read_trace_csv."""
from __future__ import annotations

import math

from .solver import TraceRecord

TRACE_CSV_HEADER = ("method,state,pair_partner,t,E,dE,res_norm,x_norm,kinetic,matvecs,restart,"
                    "b,c,b_ab,b_ba,b_bb,c_ab,c_ba,c_bb,a_ab,a_ba,E_partner,x_norm_partner,res_norm_partner")

_TAIL = ("b", "c", "b_ab", "b_ba", "b_bb", "c_ab", "c_ba", "c_bb", "a_ab", "a_ba", "energy_partner",
         "x_norm_partner", "res_norm_partner")


def trace_csv_header() -> str:
    return TRACE_CSV_HEADER


def _cell(v: float) -> str:
    return "" if v is None or math.isnan(v) else "%.17g" % v


class MemoryTraceSink:
    """Keeps records in memory (trace.hpp:57-66)."""

    def __init__(self):
        self.records: list[TraceRecord] = []

    def __call__(self, rec: TraceRecord):
        self.records.append(rec)

    record = __call__


class CsvTraceSink:
    """CSV sink (trace.hpp:68-118): header once, one row per record."""

    def __init__(self, path_or_file):
        if hasattr(path_or_file, "write"):
            self._f, self._own = path_or_file, False
        else:
            try:
                self._f, self._own = open(path_or_file, "w"), True
            except OSError as e:
                raise RuntimeError(f"cannot open trace file {path_or_file}") from e
        self._f.write(TRACE_CSV_HEADER + "\n")

    def __call__(self, r: TraceRecord):
        head = [r.method, str(r.state), str(r.pair_partner) if r.pair_partner >= 0 else "", str(r.t),
                _cell(r.energy), _cell(r.dE), _cell(r.res_norm), _cell(r.x_norm), _cell(r.kinetic),
                str(r.matvecs), r.restart_reason]
        self._f.write(",".join(head + [_cell(getattr(r, k)) for k in _TAIL]) + "\n")

    record = __call__

    def close(self):
        if self._own:
            self._f.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class TeeTraceSink:
    """Fans one record out to several sinks (trace.hpp:120-132)."""

    def __init__(self, *sinks):
        self.sinks = [s for s in sinks if s is not None]

    def add(self, sink):
        if sink is not None:
            self.sinks.append(sink)

    def __call__(self, rec: TraceRecord):
        for s in self.sinks:
            s(rec)

    record = __call__


def read_trace_csv(lines) -> list[TraceRecord]:
    """Parses a CSV trace produced by CsvTraceSink (trace.hpp:136-186)."""
    it = iter(lines)
    try:
        first = next(it).rstrip("\n")
    except StopIteration:
        raise RuntimeError("trace parse: empty input") from None
    if first != TRACE_CSV_HEADER:
        raise RuntimeError("trace parse: unexpected header")
    out = []
    for line_no, line in enumerate(it, start=2):
        line = line.rstrip("\n")
        if not line:
            continue
        f = line.split(",")
        f += [""] * (24 - len(f))
        if len(f) != 24:
            raise RuntimeError(f"trace parse: line {line_no} has {len(f)} fields")

        def num(s):
            return float("nan") if s == "" else float(s)

        tail = {k: num(f[11 + i]) for i, k in enumerate(_TAIL)}
        out.append(TraceRecord(method=f[0], state=int(f[1]), t=int(f[3]), energy=num(f[4]), dE=num(f[5]),
                               res_norm=num(f[6]), x_norm=num(f[7]), kinetic=num(f[8]), matvecs=int(f[9]),
                               restart_reason=f[10], pair_partner=-1 if f[2] == "" else int(f[2]), **tail))
    return out


def read_trace_csv_file(path) -> list[TraceRecord]:
    try:
        with open(path) as fh:
            return read_trace_csv(fh)
    except OSError as e:
        raise RuntimeError(f"cannot open trace file {path}") from e
