"""CPU: bench.py's multi-rank launcher. `--gpus N` outside torchrun re-launches itself under
torch.distributed.run (127.0.0.1 rendezvous); --dry-run replaces the GPU work by a host step so the
spawn, rendezvous (gloo), barrier and max-over-ranks paths run here without a GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=300):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    return r.returncode, lines, r.stderr


@pytest.mark.timeout(300)
@pytest.mark.parametrize("n", [2, 3])
def test_launcher_spawns_ranks_gloo(n):
    rc, lines, err = run_bench("--gpus", str(n), "--dry-run", "--steps", "2", "--warmup", "1")
    assert rc == 0, err[-2000:]
    assert len(lines) == 1, lines          # rank 0 alone prints, exactly one JSON line
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["ranks"] == list(range(n)) and d["dry_run"]
    assert d["config"]["parallelism"] == f"alpha-row shards x{n}"


@pytest.mark.timeout(300)
def test_launcher_refuses_missing_gpus():
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("this host has enough GPUs")
    rc, lines, _ = run_bench("--gpus", "2", "--steps", "1", "--warmup", "0", "--no-tte", "--no-cpu-baseline")
    assert rc != 0
    assert lines and "error" in json.loads(lines[-1])


def test_both_arms_share_the_config_dict():
    sys.path.insert(0, ROOT)
    import bench
    for world in (1, 2, 8):
        assert bench.config_dict("c4", world) == bench.config_dict("c4", world)
    c = bench.config_dict("c4", 1)
    assert c["n_det"] == 165636900 and c["vector_bytes"] == 8 * 165636900
