"""The C++ drop-in (include/sbg.hpp) compiled against the reference's own headers
(oracle/ref_gpu_shim.cpp -> oracle/_ref/libsbci_ref_gpu.so), and the plain-vector warm start
(sbci1.hpp:477-486) through the C ABI."""
import numpy as np
import pytest

import paper_2603_06101_b200 as P
from oracle import RefGpu, baseline_problem

pytestmark = pytest.mark.gpu
E_TOL = 1e-8


def gold(gold_dir, tag):
    import json
    import os
    with open(os.path.join(gold_dir, f"golden_{tag}.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def refgpu():
    if not RefGpu.available():
        pytest.fail("oracle/_ref/libsbci_ref_gpu.so not built (oracle/Makefile, needs /root/reference at build time)")
    return RefGpu()


def to_product(q):
    return P.FciProblem(q.norb, q.nelec, q.ms2, q.e_core, q.h1.copy(), q.eri.copy())


@pytest.mark.timeout(600)
def test_cpp_operator_two_threads_hundred_applies(refgpu, rest):
    """test_operator.cpp:49-64 on sbci::gpu::CudaFciOperator: 2 threads x 100 applies through the
    reference's SymmetricOperator::apply; every sigma exact, the atomic counter reads 200."""
    q = baseline_problem(1, rest)
    assert refgpu.concurrent_applies(q, 2, 100) == 0
    assert refgpu.concurrent_applies(q, 4, 25) == 0


@pytest.mark.parametrize("method,key", [(1, "sbci1"), (2, "sbci2"), (3, "davidson")])
def test_cpp_device_drivers_match_reference(refgpu, rest, gold_dir, method, key):
    """sbci::gpu::solve_n_states_* (reference signature, reference result types, TraceSink) against
    the reference's own c1 run: energies and — for SBCI1/SBCI2 — the iteration and sigma counts."""
    q = baseline_problem(1, rest)
    g = gold(gold_dir, "c1")[key]
    rc, r = refgpu.device_solve(q, len(g["energies"]), method)
    assert rc == 0, r["error"]
    assert np.abs(r["energies"] - np.array(g["energies"])).max() <= E_TOL
    assert r["iterations"].tolist() == g["iterations"] and r["matvecs"] == g["matvecs"]


def test_cpp_nonconvergence_maps_to_reference_exception(refgpu, rest):
    q = baseline_problem(1, rest)
    rc, r = refgpu.device_solve(q, 1, 1, t_max=2)
    assert rc == 2 and r["failed_state"] == 0 and "did not converge" in r["error"]


@pytest.mark.parametrize("with_defl", [0, 1])
def test_cpp_warm_start_matches_reference_driver(refgpu, rest, with_defl):
    """sbci::gpu::solve_state_sbci1 vs the reference's solve_state_sbci1 (host driver, same GPU
    operator) from the same plain vector, shift and deflation set."""
    q = baseline_problem(1, rest)
    r = refgpu.warm_start(q, with_defl)
    assert abs(r["e_ref"] - r["e_dev"]) <= E_TOL
    assert r["it_ref"] == r["it_dev"]
    assert abs(r["overlap"] - 1.0) <= 1e-6
    assert abs(r["shift_ref"] - r["shift_dev"]) <= E_TOL


def test_python_warm_start(rest, gold_dir):
    """P.solve_state_sbci1: ground state of c1 from the lowest-diagonal unit vector, then state 1
    from the next one deflated against it (the reference's energies)."""
    q = baseline_problem(1, rest)
    g = gold(gold_dir, "c1")["sbci1"]
    op = P.FciOperator(to_product(q), max_determinants=2 ** 62)
    d = op.diagonal()
    order = np.lexsort((np.arange(len(d)), d))
    e0 = np.zeros(op.dim())
    e0[order[0]] = 1.0
    op.reset_apply_count()
    r0 = P.solve_state_sbci1(op, e0, d[order[0]], d[order[0]])
    assert abs(r0.pair.energy - g["energies"][0]) <= E_TOL
    assert r0.matvecs == op.apply_count()          # the seed image + the solve's sigma builds
    assert abs(np.linalg.norm(r0.pair.vector) - 1.0) <= 1e-12
    assert abs(r0.shift - r0.pair.energy) <= 1e-12  # alpha == 0 tracks the ground shift
    e1 = np.zeros(op.dim())
    e1[order[1]] = 1.0
    r1 = P.solve_state_sbci1(op, e1, d[order[1]], r0.pair.energy,
                             deflation=[(r0.pair.vector, r0.converged_image, r0.pair.energy)], alpha=1)
    assert abs(r1.pair.energy - g["energies"][1]) <= E_TOL
    assert abs(r1.pair.vector @ r0.pair.vector) <= 1e-9
    r1b = P.solve_state_sbci1(op, e1, d[order[1]], r0.pair.energy, deflation=[(r0.pair.vector, r0.pair.energy)],
                              alpha=1)
    assert abs(r1b.pair.energy - r1.pair.energy) <= E_TOL
    with pytest.raises(ValueError):
        P.solve_state_sbci1(op, np.zeros(op.dim()), 0.0, 0.0)
    op.close()
