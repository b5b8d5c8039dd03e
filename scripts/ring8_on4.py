"""8-rank rings on a box with fewer GPUs (two ranks per GPU; gloo for the plumbing --
NCCL refuses two ranks on one GPU -- while the hop itself still uses CUDA IPC + copy
engine + stream flags exactly as on 8 GPUs).  Functional check of the 8-rank plans
(not a performance number): MD P8 / C1 / C4 rings bitwise equal to one GPU, the
stencil G8 ring bit-exact with the oracle.
  torchrun --nproc-per-node 8 scripts/ring8_on4.py <out_dir>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_11289_b200 import CONFIGS, GRID_CONFIGS  # noqa: E402
from paper_2507_11289_b200 import dsea as D  # noqa: E402
from paper_2507_11289_b200.grid import Grid  # noqa: E402


def md(cfg_name, steps, rank, world, dev, block=0):
    c = CONFIGS[cfg_name]
    e = D.Engine(D.Box(c.nx, c.ny, c.nz, c.rho, c.rc, c.dt, c.T0, c.seed))
    e.slice(n_slices=c.n_slices, cells_per_slice_x=c.cells_per_slice_x, n_gpus=world, rank=rank, device=dev,
            slices_per_stage=block)
    D.ring_connect(e.ctx, rank, world, "peer")
    e.step(steps)
    x = e.positions() if rank == 0 else None
    dist.barrier()
    D.ring_disconnect(e.ctx, world)
    e.close()
    if rank == 0:
        s = D.Engine(D.Box(c.nx, c.ny, c.nz, c.rho, c.rc, c.dt, c.T0, c.seed))
        s.slice(n_slices=c.n_slices, cells_per_slice_x=c.cells_per_slice_x, device=dev)
        s.step(steps)
        ok = np.array_equal(x, s.positions())
        s.close()
        return ok
    return True


def grid(steps, rank, world, dev):
    from oracle import grid as OG
    from tests import inputs
    c = GRID_CONFIGS["G8"]
    g = Grid(c.nx, c.ny, c.nz, c.n_slices, c.r, n_gpus=world, rank=rank, device=dev)
    u0 = inputs.grid_field(c.nx, c.ny, c.nz, c.seed)
    if rank == 0:
        g.set_field(u0)
    g.connect(rank, world)
    g.step(steps)
    u = g.field() if rank == 0 else None
    dist.barrier()
    g.disconnect(world)
    g.close()
    return bool(np.array_equal(u, OG.run(u0, c.r, steps))) if rank == 0 else True


def main():
    out = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    res = {}
    for name, fn in [("P8_auto_16", lambda: md("P8", 16, rank, world, dev)),
                     ("P8_B1_16", lambda: md("P8", 16, rank, world, dev, 1)),
                     ("C1_B1_8", lambda: md("C1", 8, rank, world, dev, 1)),
                     ("G8_16", lambda: grid(16, rank, world, dev)),
                     ("C4_auto_16", lambda: md("C4", 16, rank, world, dev))]:
        res[name] = fn()
        dist.barrier()
        if rank == 0:
            print(name, "OK" if res[name] else "MISMATCH", flush=True)
    if rank == 0:
        with open(os.path.join(out, "ring8.txt"), "w") as f:
            for k, v in res.items():
                f.write(f"{k} {'OK' if v else 'MISMATCH'}\n")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
