"""One rank of a ring check (launched by tests/test_gpu_ring.py and
tests/test_gpu_ring_shared.py through torchrun): slices stream through N_GPU processes
(§3.1), one GPU each -- or, with --shared-device, all on GPU 0 (gloo for the
plumbing: NCCL refuses two ranks on one GPU; the hop itself is still the CUDA IPC map,
copy-engine push and stream flags of the peer backend).  Rank 0 writes the final state
to an .npz for comparison with a single-GPU run and with the oracle."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch
import torch.distributed as dist

from paper_2507_11289_b200 import CONFIGS
from paper_2507_11289_b200 import dsea as D


def _log(rank, msg):
    if os.environ.get("DSEA_RING_DEBUG"):
        import time
        print(f"[rank {rank} {time.time():.3f}] {msg}", flush=True)


def main():
    if os.environ.get("DSEA_RING_DEBUG"):
        import faulthandler
        import signal
        faulthandler.register(signal.SIGTERM, all_threads=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="P8")
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--calls", type=int, default=1)
    ap.add_argument("--block", type=int, default=0, help="slices per stage (0 = auto)")
    ap.add_argument("--hop", default="peer", choices=["peer", "nccl"])
    ap.add_argument("--thermo", type=float, default=0.0, help="NVT thermostat T (0 = NVE)")
    ap.add_argument("--shared-device", action="store_true",
                    help="every rank on GPU 0, gloo process group (peer hop only)")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    if a.shared_device:
        local = 0
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = CONFIGS[a.config]
    e = D.Engine(D.Box(c.nx, c.ny, c.nz, c.rho, c.rc, c.dt, c.T0, c.seed))
    e.slice(n_slices=c.n_slices, cells_per_slice_x=c.cells_per_slice_x, n_gpus=world, rank=rank,
            device=local, workers_per_gpu=a.workers, slices_per_stage=a.block)
    _log(rank, "sliced")
    if os.environ.get("DSEA_HANG_DEBUG"):
        D.dsea_set_timing(e.ctx, True)     # per-op events for the library's hang report
    if a.thermo > 0:
        e.set_thermostat(a.thermo)
    D.ring_connect(e.ctx, rank, world, a.hop)
    _log(rank, "connected")
    per = a.steps // a.calls
    for k in range(a.calls):
        e.step(per if k < a.calls - 1 else a.steps - per * (a.calls - 1))
        _log(rank, f"stepped call {k}")
    steps, en = e.energies()
    _log(rank, "energies")
    allv = [None] * world
    prof = e.raw_profiles()
    dist.all_gather_object(allv, (steps.tolist(), en.tolist(),
                                  np.stack([prof[k] for k in ("n_sum", "U_sum", "V_sum", "KE_sum")], 1).tolist()))
    _log(rank, "gathered")
    if rank == 0:
        st = sorted((s, tuple(v)) for s_, v_, _ in allv for s, v in zip(s_, v_))
        prof_sum = np.sum([np.array(p_) for _, _, p_ in allv], axis=0)
        np.savez(a.out, x=e.positions(), v=e.velocities(), f=e.forces(),
                 steps=np.array([s for s, _ in st]), en=np.array([v for _, v in st]),
                 stats=np.array([e.stats().hop_bytes]), prof=prof_sum)
    dist.barrier()
    D.ring_disconnect(e.ctx, world)
    e.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
