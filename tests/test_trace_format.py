"""Trace sink formats (trace.hpp:46-186) — host-only."""
import io
import math

import pytest

import paper_2603_06101_b200 as P

NAN = float("nan")


def rec(method="sbci1", pair=-1, **kw):
    base = dict(method=method, state=1, t=3, energy=-1.25, dE=1e-9, res_norm=2.5e-6, x_norm=1.0, kinetic=0.125,
                matvecs=42, restart_reason="", b=0.5, c=-0.25, pair_partner=pair)
    base.update(kw)
    return P.TraceRecord(**base)


def test_header_matches_reference():
    # trace.hpp:46-49, verbatim column order
    assert P.trace_csv_header() == ("method,state,pair_partner,t,E,dE,res_norm,x_norm,kinetic,matvecs,restart,"
                                    "b,c,b_ab,b_ba,b_bb,c_ab,c_ba,c_bb,a_ab,a_ba,E_partner,x_norm_partner,"
                                    "res_norm_partner")


def test_csv_round_trip_and_cells():
    buf = io.StringIO()
    sink = P.CsvTraceSink(buf)
    mem = P.MemoryTraceSink()
    tee = P.TeeTraceSink(sink, mem)
    tee(rec())
    tee(rec("sbci2", pair=2, b_ab=0.1, b_ba=-0.2, b_bb=1.0, c_ab=3.0, c_ba=4.0, c_bb=5.0, a_ab=6.0, a_ba=7.0,
            energy_partner=-0.75, x_norm_partner=0.9, res_norm_partner=1e-3, restart_reason="max_cycle"))
    tee(rec("davidson", kinetic=NAN, b=NAN, c=NAN, energy=1.0 / 3.0))
    lines = buf.getvalue().splitlines()
    assert len(lines) == 4 and all(len(l.split(",")) == 24 for l in lines)
    # NaN fields are empty cells; the pair partner is empty for -1; 17 significant digits
    assert lines[1].split(",")[2] == "" and lines[1].split(",")[13] == ""
    assert lines[2].split(",")[2] == "2" and lines[2].split(",")[10] == "max_cycle"
    assert lines[3].split(",")[4] == "0.33333333333333331" and lines[3].split(",")[8] == ""
    back = P.read_trace_csv(buf.getvalue().splitlines(keepends=True))
    assert len(back) == 3 and len(mem.records) == 3
    for a, b in zip(mem.records, back):
        for k in a.__dataclass_fields__:
            va, vb = getattr(a, k), getattr(b, k)
            if isinstance(va, float) and math.isnan(va):
                assert math.isnan(vb)
            else:
                assert va == vb, k


def test_read_rejects_bad_header():
    with pytest.raises(RuntimeError, match="unexpected header"):
        P.read_trace_csv(["not,a,header\n"])
    with pytest.raises(RuntimeError, match="empty input"):
        P.read_trace_csv([])
