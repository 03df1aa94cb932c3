"""The command-line front end (paper_2603_06101_b200/cli.py), modelled on the reference's own CLI
checks (proj/tests/test_cli.cpp:43-157): summary schema (exactly 9 keys), trace/summary matvec
agreement, method agreement through `compare`, the S^2 column of `fci`, config precedence and the
exit codes 0 / 1 / 2. CPU tests cover parsing, config resolution and every error path that stops
before the operator is built; the GPU tests run the solves."""
import json
import os
import subprocess
import sys

import pytest

from paper_2603_06101_b200 import cli
from paper_2603_06101_b200.solver import RunSummary, StateSummary

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
H6 = os.path.join(ROOT, "tests", "golden", "h6_4e.fcidump")


def run(argv, capsys):
    rc = cli.main(argv)
    out = capsys.readouterr()
    return rc, out.out + out.err


# ---------------------------------------------------------------- CPU: parsing and error paths
def test_usage_errors_exit_1(capsys, tmp_path):
    assert run([], capsys)[0] == 1
    assert run(["solve"], capsys)[0] == 1                                  # no input (test_cli.cpp:120)
    assert run(["solve", "--fcidump", H6, "--frobnicate"], capsys)[0] == 1  # unknown flag (:121-122)
    assert run(["fci"], capsys)[0] == 1                                    # --fcidump is required
    assert run(["solve", "--fcidump", "/does/not/exist.fcidump"], capsys)[0] == 1   # missing file (:123)
    assert run(["solve", "--fcidump", H6, "--method", "lanczos"], capsys)[0] == 1
    assert run(["solve", "--fcidump", H6, "--preset", "medium"], capsys)[0] == 1
    assert run(["solve", "--fcidump", H6, "--nroots", "0"], capsys)[0] == 1
    assert run(["solve", "--fcidump", H6, "--config", "/does/not/exist.json"], capsys)[0] == 1   # (:142-143)
    assert run(["solve", "--fcidump", H6, "--eps0", "-1"], capsys)[0] == 1  # SolverConfig::validate
    rc, msg = run(["solve", "--input", str(tmp_path / "h.mtx")], capsys)
    assert rc == 1 and "Matrix Market" in msg
    assert run(["solve", "--input", "a.mtx", "--fcidump", H6], capsys)[0] == 1
    assert run(["gen", "--n", "120"], capsys)[0] == 1
    assert run(["conserve", "--trace", "t.csv"], capsys)[0] == 1


def test_module_entry_point_exit_code():
    r = subprocess.run([sys.executable, "-m", "paper_2603_06101_b200.cli", "solve"], cwd=ROOT,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 1 and "error:" in r.stderr


def test_config_precedence(tmp_path):
    """preset < JSON config file < explicit flags (sbci_cli.cpp:79-96)."""
    cfgf = tmp_path / "cfg.json"
    cfgf.write_text(json.dumps({"eps0": 1e-8, "r0": 1e-4, "max_cycle": 15, "hx_refresh_restarts": 3}))
    ap = cli.build_parser()
    c = cli.resolve_config(ap.parse_args(["solve", "--fcidump", H6]))
    assert (c.eps0, c.r0, c.max_cycle) == (1e-10, 1e-5, 0)
    c = cli.resolve_config(ap.parse_args(["solve", "--fcidump", H6, "--preset", "loose"]))
    assert (c.eps0, c.r0) == (1e-8, 1e-4)
    c = cli.resolve_config(ap.parse_args(["solve", "--fcidump", H6, "--preset", "tight", "--config", str(cfgf)]))
    assert (c.eps0, c.r0, c.max_cycle, c.hx_refresh_restarts) == (1e-8, 1e-4, 15, 3)
    c = cli.resolve_config(ap.parse_args(["solve", "--fcidump", H6, "--config", str(cfgf), "--r0", "3e-6",
                                          "--max-cycle", "7", "--b-th", "0.02", "--t-max", "50"]))
    assert (c.eps0, c.r0, c.max_cycle, c.b_th, c.t_max) == (1e-8, 3e-6, 7, 0.02, 50)


def test_summary_json_schema():
    s = RunSummary("sbci2", [StateSummary(0, -1.5, 9, 1, 3e-6, 0.0),
                             StateSummary(1, -1.2, 4, 0, 2e-6, float("nan"))], 13, 1, 17, 0, 11, 0.25)
    j = cli.summary_to_json(s)
    assert tuple(j.keys()) == cli.SUMMARY_KEYS                          # exactly the 9 keys, in order
    assert j["energies"] == [-1.5, -1.2] and j["matvecs"] == 17
    assert j["states"][1]["s_squared"] is None                         # NaN -> null (sbci_cli.cpp:150-153)
    assert set(j["states"][0]) == {"state", "energy", "iterations", "restarts", "final_residual", "s_squared"}
    json.dumps(j)


# ---------------------------------------------------------------- GPU: solves through the CLI
@pytest.mark.gpu
@pytest.mark.parametrize("method", ["sbci1", "sbci2", "davidson"])
def test_fci_solve_summary_and_trace(method, tmp_path, capsys, gold_dir):
    from paper_2603_06101_b200 import read_trace_csv_file
    summ, trace = tmp_path / f"{method}.json", tmp_path / f"{method}.csv"
    rc, out = run(["fci", "--fcidump", H6, "--method", method, "--nroots", "3", "--summary", str(summ),
                   "--trace", str(trace)], capsys)
    assert rc == 0, out
    assert "S^2" in out                                                  # test_cli.cpp:111-115
    j = json.loads(summ.read_text())
    assert tuple(j.keys()) == cli.SUMMARY_KEYS and j["method"] == method and len(j["energies"]) == 3
    rows = read_trace_csv_file(str(trace))
    assert rows and rows[-1].matvecs == j["matvecs"]                    # test_cli.cpp:71-78
    with open(os.path.join(gold_dir, "golden_h6_4e.json")) as f:
        ref = json.load(f)[method]
    assert max(abs(a - b) for a, b in zip(j["energies"], ref["energies"])) <= 1e-10
    assert j["matvecs"] == ref["matvecs"]                              # same trajectory as the reference
    assert [s["iterations"] for s in j["states"]] == ref["iterations"]
    assert abs(j["states"][1]["s_squared"] - 2.0) <= 1e-9              # state 1 is the triplet


@pytest.mark.gpu
def test_compare_and_exit_codes(tmp_path, capsys):
    cmp = tmp_path / "cmp.json"
    rc, out = run(["compare", "--fcidump", H6, "--nroots", "3", "--summary", str(cmp)], capsys)
    assert rc == 0, out
    j = json.loads(cmp.read_text())
    assert set(j) == {"sbci1", "sbci2", "davidson"}
    for k in range(3):                                                   # test_cli.cpp:84-99
        assert abs(j["sbci1"]["energies"][k] - j["davidson"]["energies"][k]) <= 1e-8
        assert abs(j["sbci2"]["energies"][k] - j["davidson"]["energies"][k]) <= 1e-8
    # nonconvergence -> 2 (test_cli.cpp:124-127)
    rc, out = run(["solve", "--fcidump", H6, "--eps0", "1e-300", "--r0", "1e-300", "--t-max", "3"], capsys)
    assert rc == 2, out
    # presets: loose needs no more iterations than tight (test_cli.cpp:147-156)
    t, lo = tmp_path / "tight.json", tmp_path / "loose.json"
    assert run(["solve", "--fcidump", H6, "--preset", "tight", "--summary", str(t)], capsys)[0] == 0
    assert run(["solve", "--fcidump", H6, "--preset", "loose", "--summary", str(lo)], capsys)[0] == 0
    assert json.loads(lo.read_text())["total_iterations"] <= json.loads(t.read_text())["total_iterations"]
    # a JSON config file feeds SolverConfig (test_cli.cpp:131-144); an explicit Davidson space cap
    cfgf = tmp_path / "cfg.json"
    cfgf.write_text('{"eps0": 1e-8, "r0": 1e-4, "max_cycle": 15}\n')
    assert run(["solve", "--fcidump", H6, "--config", str(cfgf), "--nroots", "2"], capsys)[0] == 0
    rc, out = run(["solve", "--fcidump", H6, "--method", "davidson", "--nroots", "2", "--max-space", "4",
                   "--summary", str(tmp_path / "dv.json")], capsys)
    assert rc == 0, out
    assert run(["solve", "--fcidump", H6, "--method", "davidson", "--nroots", "2", "--max-space", "3"],
               capsys)[0] == 1                                           # max_space < 2*nroots
    # the determinant guard and its override (fci_operator.hpp:103-120)
    rc, out = run(["solve", "--fcidump", H6, "--max-determinants", "100"], capsys)
    assert rc == 1 and "guard" in out
