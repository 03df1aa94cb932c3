"""Multi-GPU plumbing: one process per GPU, torch.distributed for rendezvous only. The data path
(all-gather of the CI vector, all-reduce of the dot buffer, all-to-all of the alpha-alpha blocks)
runs inside libsbg on its own NCCL communicator; this module creates it.

Partition: contiguous alpha-string blocks of ceil(NA/world) rows
(sbg_shard_range); the alpha-alpha same-spin term is computed per beta-column window of the same
partition of NB and exchanged block-wise."""
from __future__ import annotations

import ctypes as C
import os

from ._lib import check, lib


def env_rank_world():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def shard_range(n: int, rank: int, world: int):
    lo, hi = C.c_int64(), C.c_int64()
    check(lib().sbg_shard_range(n, rank, world, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def nccl_unique_id_bytes() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().sbg_nccl_unique_id(buf))
    return buf.raw


def broadcast_nccl_id(rank: int) -> bytes:
    """Rank 0 creates the NCCL unique id; torch.distributed (already initialised) broadcasts it."""
    import torch.distributed as dist
    obj = [nccl_unique_id_bytes() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def exchange_blocks(na: int, nb: int, world: int):
    """(rows of rank r, beta-column window of rank r) for every rank: rank r computes the
    alpha-alpha term for all rows but only its column window, then sends rows(p) x window(r) to p."""
    return [(shard_range(na, r, world), shard_range(nb, r, world)) for r in range(world)]


class LocalRankGroup:
    """Testing aid (sbg_local_group_*): `world` ranks as threads of this process, sharing one GPU
    or several; the collectives go through host barriers and device copies, so the sharded sigma and
    solver data flow runs on the real kernels without several GPUs. Every rank must enter each
    collective entry point (apply, solve, spin_squared) concurrently: use run()."""

    def __init__(self, world: int):
        h = C.c_void_p()
        check(lib().sbg_local_group_create(world, C.byref(h)))
        self.handle, self.world = h, world

    def operators(self, prob, max_determinants: int = 2 ** 62, devices=None):
        from .fci import FciOperator
        devices = devices or [0] * self.world
        return [FciOperator(prob, max_determinants, device=devices[r], rank=r, world=self.world, local_group=self)
                for r in range(self.world)]

    def run(self, fn, ops):
        """fn(rank, op) on every rank concurrently (ctypes releases the GIL inside libsbg); returns the
        per-rank results, re-raising the first failure."""
        import threading
        out, err = [None] * len(ops), [None] * len(ops)

        def body(r):
            try:
                out[r] = fn(r, ops[r])
            except BaseException as e:  # noqa: BLE001 - surfaced below
                err[r] = e
        ts = [threading.Thread(target=body, args=(r,)) for r in range(len(ops))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for e in err:
            if e is not None:
                raise e
        return out

    def close(self):
        if getattr(self, "handle", None):
            lib().sbg_local_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

