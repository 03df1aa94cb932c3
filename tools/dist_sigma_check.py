"""Sharded sigma and SBCI1 over NCCL (one process per GPU, launched by torch.distributed.run): each
rank's rows of sigma against a single-GPU operator built on the same rank, and the c1 four-root
SBCI1 energies against the reference's golden energies. Prints one JSON line per rank.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_sigma_check.py [c1|c2]
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_06101_b200 as P  # noqa: E402
from paper_2603_06101_b200 import dist as pdist  # noqa: E402

CFG = {"c1": (10, 10, 0.05), "c2": (12, 12, 0.05)}


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "c1"
    rank, world, local = pdist.env_rank_world()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    norb, ne, sc = CFG[tag]
    prob = P.synthetic_problem(norb, ne, 2603, sc)
    nid = pdist.broadcast_nccl_id(rank)
    op = P.FciOperator(prob, max_determinants=2 ** 62, device=local, rank=rank, world=world, nccl_id=nid)
    single = P.FciOperator(prob, max_determinants=2 ** 62, device=local)
    x = np.random.default_rng(5).uniform(-1, 1, op.dim())
    y = op.apply(x)
    y1 = single.apply(x)
    nb = op.n_beta_strings
    sl = slice(op.row_lo * nb, op.row_hi * nb)
    err = float(np.abs(y[sl] - y1[sl]).max() / np.abs(y1).max())
    out = {"rank": rank, "world": world, "rows": [op.row_lo, op.row_hi], "sigma_rel_err": err}
    if tag == "c1":
        with open(os.path.join(ROOT, "tests", "golden", "golden_c1.json")) as f:
            g = json.load(f)["sbci1"]
        res = P.solve_n_states_sbci1(op, 4, want_vectors=False)
        e = np.array([pp.energy for pp in res.pairs])
        out["max_abs_dE_vs_reference"] = float(np.abs(e - np.array(g["energies"])).max())
        out["matvecs"] = res.summary.matvecs
        out["reference_matvecs"] = g["matvecs"]
    print(json.dumps(out), flush=True)
    op.close()
    single.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
