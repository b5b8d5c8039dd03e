"""NEXT-3: the paper's largest dataset on one node -- the N_i = 630 FCC
cube, 1,000,188,000 atoms (§4.3; rho* 0.8, rc 2.5: 430 slices by the paper's
rule) -- streamed through a ring of GPUs (one process per GPU, peer copy-engine hop).
The input buffer holds all N_S slots (rank 0 holds the state between calls, Q22); the
working buffers are pools of a few slots (P:121-122 circular slot buffers, s N_b > N_S).
Reports per-GPU device memory, the throughput of K super-cycles, and sampled force
parity against the CPU oracle: forces of atoms sampled in a few slices, against the
oracle's all-pairs sums over the atoms of the neighbouring slices (every atom within
rc of slice j lies in slices j-1..j+1).

  torchrun --nproc-per-node 4 scripts/run_big.py [--ni 630] [--cycles 3] [--out f.json]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_11289_b200 import dsea as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ni", type=int, default=630, help="FCC cells per edge (N = 4 ni^3)")
    ap.add_argument("--cycles", type=int, default=3, help="timed super-cycles")
    ap.add_argument("--samples", type=int, default=32, help="sampled atoms per checked slice")
    ap.add_argument("--slices", default="1,215,428", help="slices whose atoms are checked")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "big_run.json"))
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    t0 = time.time()
    e = D.Engine(D.Box(a.ni, a.ni, a.ni, 0.8, 2.5, 0.0018, 1.0, 11289))
    e.slice(n_slices=0, n_gpus=world, rank=rank, device=local)
    t_slice = time.time() - t0
    if world > 1:
        D.ring_connect(e.ctx, rank, world, "peer")
    free, total = torch.cuda.mem_get_info(local)
    g = e.geometry
    nw = world
    # warm-up super-cycle, then K timed ones
    e.step(nw)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t1 = time.time()
    e.step(a.cycles * nw)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    dt = time.time() - t1
    # parity: positions of the state now, forces of that state after one more step
    checks = []
    sl = [int(s) for s in a.slices.split(",")]
    before = {}
    if rank == 0:
        for j in sl:
            for m in (j - 1, j, j + 1):
                if 0 <= m < g.n_slices and m not in before:
                    before[m] = D.dsea_get_slice(e.ctx, m)
    e.step(1)       # timestep computed by rank 0 (a partial super-cycle, Q15)
    if rank == 0:
        import oracle
        rng = np.random.default_rng(7)
        worst = 0.0
        after = {}
        for m in before:
            after[m] = D.dsea_get_slice(e.ctx, m)
        for j in sl:
            nb = [before[m] for m in (j - 1, j, j + 1) if m in before]
            loc = np.concatenate([b["xyz"] for b in nb])
            loc_id = np.concatenate([b["id"] for b in nb])
            own = before[j]
            pick = rng.choice(len(own["id"]), min(a.samples, len(own["id"])), replace=False)
            # local index of each picked atom in the neighbourhood array
            pos_in_loc = {int(i): k for k, i in enumerate(loc_id)}
            idx = np.array([pos_in_loc[int(own["id"][p])] for p in pick], dtype=np.int64)
            Fo, _ = oracle.forces_subset(loc, g.b, 2.5, idx)
            # the picked atoms after the step (one may have crossed into a neighbour slice)
            aid = np.concatenate([after[m]["id"] for m in (j - 1, j, j + 1) if m in after])
            af = np.concatenate([after[m]["f"] for m in (j - 1, j, j + 1) if m in after])
            fmap = {int(i): k for k, i in enumerate(aid)}
            Fg = np.array([af[fmap[int(own["id"][p])]] for p in pick])
            frms = np.sqrt((Fo ** 2).sum(1).mean())
            err = np.sqrt(((Fg - Fo) ** 2).sum(1)) / np.maximum(np.sqrt((Fo ** 2).sum(1)), frms)
            worst = max(worst, float(err.max()))
            checks.append({"slice": j, "atoms": int(len(pick)), "neighbourhood": int(len(loc)),
                           "max_rel_err": float(err.max())})
    mem = torch.tensor([float(total - free), float(total)], dtype=torch.float64)
    allmem = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
    if world > 1:
        dist.all_gather(allmem, mem)
    else:
        allmem = [mem]
    if rank == 0:
        res = {"n_atoms": int(g.n_atoms), "box": list(g.b), "n_slices": int(g.n_slices),
               "slot_capacity": int(g.slot_capacity), "gpus": world,
               "device_memory_used_gb": [round(float(m[0]) / 1e9, 2) for m in allmem],
               "device_memory_total_gb": round(float(allmem[0][1]) / 1e9, 2),
               "slice_seconds": round(t_slice, 1), "timed_super_cycles": a.cycles,
               "timed_seconds": dt, "atom_timesteps_per_s": g.n_atoms * a.cycles * nw / dt,
               "parity": checks, "parity_max_rel_err": max(c["max_rel_err"] for c in checks),
               "note": "wall-clock timing around a blocking dsea_step (includes the ring's fill/drain)"}
        print(json.dumps(res, indent=1), flush=True)
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        with open(a.out, "w") as fh:
            json.dump(res, fh, indent=1)
    if world > 1:
        dist.barrier()
        D.ring_disconnect(e.ctx, world)
    e.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
