"""One rank of a multi-GPU ring of the stencil workload (launched by
tests/test_gpu_grid.py through torchrun): slices of the grid stream through N_GPU
processes over NVLink (§3.1); rank 0 loads the field and writes the result
to an .npz for comparison with the oracle."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch
import torch.distributed as dist

from paper_2507_11289_b200 import GRID_CONFIGS
from paper_2507_11289_b200.grid import Grid
from tests import inputs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="G8")
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--calls", type=int, default=1)
    ap.add_argument("--block", type=int, default=0)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = GRID_CONFIGS[a.config]
    g = Grid(c.nx, c.ny, c.nz, c.n_slices, c.r, n_gpus=world, rank=rank, device=local,
             workers_per_gpu=a.workers, slices_per_stage=a.block)
    if rank == 0:
        g.set_field(inputs.grid_field(c.nx, c.ny, c.nz, c.seed))
    g.connect(rank, world)
    per = a.steps // a.calls
    for k in range(a.calls):
        g.step(per if k < a.calls - 1 else a.steps - per * (a.calls - 1))
    if rank == 0:
        np.savez(a.out, u=g.field(), hop=np.array([g.stats().hop_bytes]))
    dist.barrier()
    g.disconnect(world)
    g.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
