"""CPU, world_size 2 and 3 over gloo: the host-side data flow of the sharded sigma / SBCI update
(Context::sigma world>1 path) — alpha-block partition from the library's
sbg_shard_range, all-gather of the sharded CI vector, all-reduced dot buffer, and the
alpha-alpha block exchange — reproduces the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, na, nb, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2603_06101_b200.dist import exchange_blocks, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(1)
    X = rng.uniform(-1, 1, (na, nb))            # the full CI matrix (alpha-major), same seed everywhere
    Wa = rng.uniform(-1, 1, (na, na)); Wa = Wa + Wa.T   # stand-ins for the same-spin operators
    Wb = rng.uniform(-1, 1, (nb, nb)); Wb = Wb + Wb.T
    M = rng.uniform(-1, 1, (na, nb))            # a row-local term (diagonal-like)
    lo, hi = shard_range(na, rank, world)
    per = (na + world - 1) // world
    # 1. all-gather of equal padded blocks (ncclAllGather in Context::gather_full)
    mine = np.zeros((per, nb))
    mine[: hi - lo] = X[lo:hi]
    bufs = [torch.zeros(per * nb, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(bufs, torch.from_numpy(mine.reshape(-1)).clone())
    Xf = torch.cat(bufs).numpy().reshape(world * per, nb)[:na]
    ok_gather = np.array_equal(Xf, X)
    # 2. local rows: beta-beta (row-local) + row-local term
    sig = Xf[lo:hi] @ Wb.T + M[lo:hi] * Xf[lo:hi]
    # 3. alpha-alpha for my beta-column window, all rows; exchange blocks
    blocks = exchange_blocks(na, nb, world)
    (clo, chi) = blocks[rank][1]
    Yw = Wa @ Xf[:, clo:chi]
    reqs, recv = [], {}
    for p, ((plo, phi), (pclo, pchi)) in enumerate(blocks):
        if p == rank:
            sig[:, clo:chi] += Yw[lo:hi]
            continue
        if (phi - plo) * (chi - clo) > 0:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(Yw[plo:phi])), p))
        if (hi - lo) * (pchi - pclo) > 0:
            recv[p] = torch.zeros((hi - lo, pchi - pclo), dtype=torch.float64)
            reqs.append(dist.irecv(recv[p], p))
    for r in reqs:
        r.wait()
    for p, t in recv.items():
        pclo, pchi = blocks[p][1]
        sig[:, pclo:pchi] += t.numpy()
    ref = (Wa @ X + X @ Wb.T + M * X)[lo:hi]
    ok_sigma = np.abs(sig - ref).max(initial=0.0) <= 1e-12 * max(1.0, np.abs(ref).max(initial=0.0))
    # 4. dot buffer all-reduce (finish_dots): identical scalars on every rank
    part = torch.tensor([float(np.sum(X[lo:hi] * ref)), float(np.sum(X[lo:hi] ** 2))], dtype=torch.float64)
    dist.all_reduce(part)
    full = Wa @ X + X @ Wb.T + M * X
    ok_dot = abs(part[0].item() - float(np.sum(X * full))) <= 1e-10 * abs(float(np.sum(X * full))) and \
        abs(part[1].item() - float(np.sum(X * X))) <= 1e-12 * float(np.sum(X * X))
    q.put((rank, ok_gather, ok_sigma, ok_dot, hi - lo))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,na,nb", [(2, 15, 35), (3, 70, 70), (4, 6, 6)])
def test_sharded_sigma_dataflow(world, na, nb):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, na, nb, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sum(r[4] for r in res) == na
    for rank, ok_g, ok_s, ok_d, _ in res:
        assert ok_g and ok_s and ok_d, (rank, ok_g, ok_s, ok_d)
