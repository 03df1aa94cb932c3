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
