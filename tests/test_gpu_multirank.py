"""NCCL over several GPUs (one process per GPU): skipped on a one-GPU box. The sharded data path
itself is covered on one GPU by the LocalComm tests (test_gpu_parity.py) and on CPU by gloo."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpu():
    import torch
    return torch.cuda.device_count()


def clean_env():
    return {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}


@pytest.mark.timeout(900)
def test_nccl_two_rank_sigma_and_sbci1():
    if ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", "--master-port=29561", os.path.join(ROOT, "tools", "dist_sigma_check.py"),
                        "c1"], capture_output=True, text=True, timeout=800, env=clean_env(), cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 2
    for d in lines:
        assert d["sigma_rel_err"] <= 1e-12
        assert d["max_abs_dE_vs_reference"] <= 1e-8 and d["matvecs"] == d["reference_matvecs"]


@pytest.mark.timeout(900)
def test_bench_self_spawns_two_ranks():
    if ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "c2", "--steps", "3",
                        "--warmup", "1", "--no-tte", "--no-cpu-baseline", "--e2e-steps", "2"],
                       capture_output=True, text=True, timeout=800, env=clean_env(), cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["n_gpus"] == 2 and d["value"] > 0
