#!/usr/bin/env python
"""Benchmark of the DSEAmd hot path (arXiv 2507.11289) on B200.

Metric (BASELINE.json; §4.3): atom-timesteps/s = molecules processed by all
workers in one super-cycle / super-cycle time.  One bench "step" is one super-cycle
(N_w = N_GPU * W timesteps of every atom: force, kick, drift, migration, finalise
and ring hop of every slice -- all §8(a) rows).

Default workload: C4 of BASELINE.json (16,384,000-atom LJ cube, rho* 0.8, T* 1.0,
rc 2.5, 109 slices; strong scaling at 1/2/4/8 GPUs).  Inputs are larger than L2
(1.25 GB of state), so no L2 flush is needed between steps.  Before the warm-up the
lattice is melted for --equil timesteps (untimed; the perfect lattice has
unrealistically uniform cell occupancy).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl dsea|reference]
  N > 1: python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

--impl reference times the CPU oracle (oracle/, O(N^2) all pairs) on the host cores on
a bounded sample of the same workload: each step computes the Algorithm 1 forces of a
sample of atoms against all N atoms.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
# bytes one atom costs the fused force+integrate kernel at minimum: read r, v, F_old (72 B)
# + id (4 B); write r', v', F_new (72 B) + id (4 B) + destination key (4 B)
FORCE_BYTES_PER_ATOM = 156
# FP64 flops of Algorithm 1 per in-cutoff ordered pair (FMA = 2)
FP64_FLOPS_PER_PAIR = 33
FP64_LANES_PER_SM = 64
N_SMS = 148


def measured_traffic_per_atom():
    """DRAM bytes per atom of the force kernel from the committed ncu capture (or None)."""
    import glob
    best = None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "force_traffic.json"))):
        try:
            with open(f) as fh:
                best = float(json.load(fh)["bytes_per_atom"])
        except Exception:
            pass
    return best


def peaks():
    try:
        with open(MEASURED_PEAKS) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every 5 ms
    during the timed region (the recipe's clocks line, without nvidia-smi start-up lag)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join(timeout=2)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": self.max_mhz or 1965.0, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml, 5 ms"}


def cpu_oracle_rate(cfg, seconds_target=15.0, max_sample=None):
    """Time the oracle (as it stands) on the host cores: Algorithm 1 forces of a sample
    of atoms against all N atoms (the O(N) per-atom work of its O(N^2) step)."""
    import numpy as np
    import oracle
    g = oracle.geometry(cfg.nx, cfg.ny, cfg.nz, cfg.rho, cfg.rc, cfg.n_slices, cfg.cells_per_slice_x)
    x = oracle.lattice(cfg.nx, cfg.ny, cfg.nz, g.a)
    n = x.shape[0]
    threads = oracle.default_threads()
    rng = np.random.default_rng(0)
    k = 8
    while True:
        idx = np.sort(rng.choice(n, min(k, n), replace=False))
        t0 = time.perf_counter()
        oracle.forces_subset(x, g.b, cfg.rc, idx, threads)
        dt = time.perf_counter() - t0
        if dt > seconds_target / 4 or k >= n or (max_sample and k >= max_sample):
            break
        k = min(n, int(k * max(2.0, (seconds_target / 4) / max(dt, 1e-4))))
    # final timed sample sized for ~seconds_target
    k = min(n, max(k, int(k * seconds_target / max(dt, 1e-4) / 2)))
    if max_sample:
        k = min(k, max_sample)
    idx = np.sort(rng.choice(n, k, replace=False))
    t0 = time.perf_counter()
    oracle.forces_subset(x, g.b, cfg.rc, idx, threads)
    dt = time.perf_counter() - t0
    return k / dt, threads, k, dt


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle, timed on the host cores (rank 0 only)."""
    if rank != 0:
        return
    import numpy as np
    import oracle
    g = oracle.geometry(cfg.nx, cfg.ny, cfg.nz, cfg.rho, cfg.rc, cfg.n_slices, cfg.cells_per_slice_x)
    x = oracle.lattice(cfg.nx, cfg.ny, cfg.nz, g.a)
    n = x.shape[0]
    threads = oracle.default_threads()
    # size one step for ~ 8 s so warmup + steps ends within a few minutes
    rate, _, _, _ = cpu_oracle_rate(cfg, seconds_target=4.0)
    per_step = int(max(1, min(n, rate * 8.0 / max(1, args.steps + args.warmup) * 4)))
    per_step = max(1, min(per_step, n))
    rng = np.random.default_rng(1)
    for _ in range(args.warmup):
        idx = np.sort(rng.choice(n, per_step, replace=False))
        oracle.forces_subset(x, g.b, cfg.rc, idx, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        idx = np.sort(rng.choice(n, per_step, replace=False))
        oracle.forces_subset(x, g.b, cfg.rc, idx, threads)
    dt = time.perf_counter() - t0
    value = per_step * args.steps / dt
    sample = (f"forces-only, sampled -- per step: Algorithm 1 forces of {per_step} sampled atoms of {n:,} "
              f"against all {n:,} "
              f"(all-pairs O(N) each, minimum image y/z) on the {cfg.name} lattice")
    line = {"metric": "atom-timesteps/s", "value": value, "unit": "atom-timesteps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (FCC lattice, seeded velocities)",
            "config": {"workload": cfg.name, "n_atoms": n, "n_slices": g.n_slices, "rho": cfg.rho,
                       "rc": cfg.rc},
            "impl": "reference",
            "comparability": "not the same work as the GPU arm: Algorithm 1 forces of sampled atoms on the "
                             "unmelted lattice (no kick, drift, migration or binning), while the GPU arm "
                             "times the full step on a melted state; an upper bound of the oracle's rate",
            "cpu_baseline": {"value": value, "unit": "atom-timesteps/s", "cores": threads,
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "atom-timesteps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


STENCIL_BYTES_PER_CELL = 16   # one read + one write of a double per cell-step


def run_stencil(args, rank, world, local_rank):
    """--config G*: the stencil workload (include/dsea_grid.h) on
    the same ring plan: metric cell-timesteps/s, roofline = HBM (16 B per cell-step)."""
    import numpy as np
    import torch
    from paper_2507_11289_b200 import GRID_CONFIGS
    from paper_2507_11289_b200 import grid as G
    cfg = GRID_CONFIGS[args.config]
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    W = args.workers
    g = G.Grid(cfg.nx, cfg.ny, cfg.nz, cfg.n_slices, cfg.r, n_gpus=world, rank=rank, device=local_rank,
               workers_per_gpu=W, slices_per_stage=args.block)
    u0 = np.random.default_rng(cfg.seed).random((cfg.nx, cfg.ny, cfg.nz))
    if rank == 0:
        g.set_field(u0)
    g.connect(rank, world)
    nw = world * W

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    for _ in range(args.warmup):
        g.step(nw)
    barrier()
    G.dsea_grid_reset_stats(g.g)
    G.dsea_grid_set_timing(g.g, True)
    hbm_peak, sm_max, peak_kind = peaks()
    with ClockSampler(local_rank) as clk:
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        g.step(args.steps * nw)
        ev1.record()
        barrier()
    ms = ev0.elapsed_time(ev1)
    st = g.stats()
    G.dsea_grid_set_timing(g.g, False)
    t = torch.tensor([ms, float(st.kernel_launches)], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
    ms_total, launches = float(t[0]), int(t[1])
    cells = cfg.n_cells
    value = cells * args.steps * nw / (ms_total * 1e-3)
    per_launch_ms = st.stencil_ms / max(1, st.stencil_launches)
    cells_per_launch = st.cell_steps / max(1, st.stencil_launches)
    achieved = STENCIL_BYTES_PER_CELL * cells_per_launch / (per_launch_ms * 1e-3) / 1e9
    e2e = None
    if not args.no_e2e:
        uh = torch.empty((cfg.nx, cfg.ny, cfg.nz), dtype=torch.float64, pin_memory=True).numpy()
        uh[...] = u0
        uo = torch.empty_like(torch.from_numpy(uh)).pin_memory().numpy()
        barrier()
        t0 = time.perf_counter()
        if rank == 0:
            G.dsea_grid_set_field(g.g, uh)
        g.step(args.steps * nw)
        if rank == 0:
            G.lib.dsea_grid_get_field(g.g, uo.ctypes.data_as(G._pd), uo.size)
        barrier()
        dt = time.perf_counter() - t0
        if dist is not None:
            tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt[0])
        e2e = {"value": cells * args.steps * nw / dt, "unit": "cell-timesteps/s",
               "h2d_bytes_per_step": int(cells * 8 / args.steps), "d2h_bytes_per_step": int(cells * 8 / args.steps),
               "note": "set_field(pinned host) + step(K super-cycles) + get_field (pinned); bytes amortised"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import grid as OG
        slab = np.ascontiguousarray(u0[: max(8, min(cfg.nx, 64))])
        t0 = time.perf_counter()
        k = 0
        while time.perf_counter() - t0 < 10.0:
            slab = OG.ftcs_step(slab, cfg.r)
            k += 1
        secs = time.perf_counter() - t0
        cpu = {"value": slab.size * k / secs, "unit": "cell-timesteps/s", "cores": 1, "kind": "oracle",
               "sample": f"{k} numpy FTCS steps of a {slab.shape} slab of the {cfg.name} grid ({secs:.1f} s)"}
    if rank == 0:
        line = {
            "metric": "cell-timesteps/s", "value": value, "unit": "cell-timesteps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded uniform random field",
            "config": {"workload": cfg.name, "cells": [cfg.nx, cfg.ny, cfg.nz], "n_slices": cfg.n_slices,
                       "r": cfg.r, "workers_per_gpu": W, "timesteps_per_step": nw,
                       "mode": "fused" if world == 1 and W == 1 else "staged-ring",
                       "l2": "inputs larger than L2 (field %.2f GB)" % (cells * 8 / 1e9),
                       "parallelism": f"ring{world}"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": None, "kernel": "k_ftcs",
                         "bytes_per_cell": STENCIL_BYTES_PER_CELL, "peak_kind": peak_kind,
                         "stencil_ms_per_launch": per_launch_ms},
            "clocks": clk.summary(), "gpu_launches": launches, "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
    g.disconnect(world)
    g.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="dsea", choices=["dsea", "reference"])
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--equil", type=int, default=200, help="untimed melting timesteps before warm-up")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-steady", action="store_true", help="skip the steady-state super-cycle rate (N > 1)")
    ap.add_argument("--staged", action="store_true",
                    help="force the staged schedule on one GPU (the ring of one: the baseline of ring efficiency)")
    ap.add_argument("--hop", default="peer", choices=["peer", "nccl"],
                    help="ring hop: NVLink copy-engine push with stream flags (peer) or NCCL send/recv")
    ap.add_argument("--block", type=int, default=0, help="slices per stage (0 = auto)")
    ap.add_argument("--thermostat", type=float, default=0.0,
                    help="NVT per-slice isokinetic thermostat at this T (P:314-316; 0 = NVE, the default)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config.startswith("G"):
        if args.impl == "reference":
            if rank == 0:
                print(json.dumps({"impl": "reference", "unavailable": "stencil workload: use the default "
                                  "MD workload for the reference arm"}), flush=True)
            return
        run_stencil(args, rank, world, local_rank)
        return
    from paper_2507_11289_b200 import CONFIGS
    cfg = CONFIGS[args.config]

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import numpy as np
    import torch
    from paper_2507_11289_b200 import dsea as D

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    W = args.workers
    e = D.Engine(D.Box(cfg.nx, cfg.ny, cfg.nz, cfg.rho, cfg.rc, cfg.dt, cfg.T0, cfg.seed))
    e.slice(n_slices=cfg.n_slices, cells_per_slice_x=cfg.cells_per_slice_x, n_gpus=world, rank=rank,
            device=local_rank, workers_per_gpu=W, slices_per_stage=args.block,
            mode=D.DSEA_MODE_STAGED if args.staged else D.DSEA_MODE_AUTO)
    if args.thermostat > 0:
        e.set_thermostat(args.thermostat)
    if world > 1:
        D.ring_connect(e.ctx, rank, world, args.hop)
    geo = e.geometry
    nw = world * W

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # melt the lattice (untimed), then warm up (untimed)
    if args.equil > 0:
        e.step(((args.equil + nw - 1) // nw) * nw)
    barrier()
    for _ in range(args.warmup):
        e.step(nw)
    barrier()

    # ---- timed region: K super-cycles, device-timed with CUDA events ----------------
    D.dsea_reset_stats(e.ctx)
    D.dsea_set_timing(e.ctx, True)
    hbm_peak, sm_max, peak_kind = peaks()
    with ClockSampler(local_rank) as clk:
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        e.step(args.steps * nw)
        ev1.record()
        barrier()
    ms = ev0.elapsed_time(ev1)
    st = e.stats()
    D.dsea_set_timing(e.ctx, False)

    # ---- steady state (the paper's metric: molecules processed by all workers in
    # one super-cycle / super-cycle time): a call of K super-cycles includes the ring's
    # pipeline fill and drain (rank g starts (2 + W) blocks after rank g-1); a second call
    # of 2K super-cycles has the same fill and drain, so the difference of the two calls
    # times K super-cycles alone.  Reported beside the K-cycle value, never instead of it.
    steady = None
    if world > 1 and not args.no_steady:
        barrier()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record()
        e.step(2 * args.steps * nw)
        s1.record()
        barrier()
        ms2 = torch.tensor([s0.elapsed_time(s1)], dtype=torch.float64, device="cuda")
        ms1 = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(ms2, op=dist.ReduceOp.MAX)
        dist.all_reduce(ms1, op=dist.ReduceOp.MAX)
        dms = float(ms2[0] - ms1[0])
        if dms > 0:
            steady = {"value": geo.n_atoms * args.steps * nw / (dms * 1e-3), "unit": "atom-timesteps/s",
                      "ms_per_super_cycle": dms / args.steps,
                      "method": f"(T({2 * args.steps} super-cycles) - T({args.steps})) / {args.steps}: "
                                "one call's pipeline fill and drain cancel (P:344 metric)"}
    t = torch.tensor([ms, float(st.kernel_launches)], dtype=torch.float64, device="cuda")
    if dist is not None:
        tmax = t.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tmax[1:], op=dist.ReduceOp.SUM)
        t = tmax
    ms_total = float(t[0])
    launches = int(t[1])
    atoms = int(geo.n_atoms)
    value = atoms * args.steps * nw / (ms_total * 1e-3)

    # dominant kernel: fused force+integrate (per-launch average on its own stream)
    force_ms_avg = st.force_ms / max(1, st.force_launches)
    # atoms per force launch on this rank: the fused pass covers every slice, a ring
    # stage B slices (counted exactly: atom-steps computed / force launches)
    atoms_per_launch = st.atom_steps / max(1, st.force_launches)
    pairs_per_atom = st.force_pairs / max(1, atoms)
    fp64_peak = N_SMS * FP64_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12  # TFLOP/s
    fp64_achieved = pairs_per_atom * atoms_per_launch * FP64_FLOPS_PER_PAIR / (force_ms_avg * 1e-3) / 1e12
    hbm_achieved = FORCE_BYTES_PER_ATOM * atoms_per_launch / (force_ms_avg * 1e-3) / 1e9
    force_share = st.force_ms / max(1e-9, st.force_ms + st.bin_ms)
    traffic_pa = measured_traffic_per_atom()

    # ---- e2e through the public API with host buffers ------------------------------
    e2e = None
    if not args.no_e2e:
        # page-locked host buffers (what a user streaming states would allocate)
        xh = torch.empty((atoms, 3), dtype=torch.float64, pin_memory=True).numpy()
        vh = torch.empty((atoms, 3), dtype=torch.float64, pin_memory=True).numpy()
        xo = torch.empty((atoms, 3), dtype=torch.float64, pin_memory=True).numpy()
        if rank == 0:
            D.dsea_get_positions(e.ctx, atoms, out=xh)
            D.dsea_get_velocities(e.ctx, atoms, out=vh)
        barrier()
        t0 = time.perf_counter()
        e.set_state(xh, vh)                       # H2D of the inputs + device binning
        e.step(args.steps * nw)
        if rank == 0:
            D.dsea_get_positions(e.ctx, atoms, out=xo)   # D2H of the result
            _ = e.energies()
        barrier()
        dt = time.perf_counter() - t0
        if dist is not None:
            tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt[0])
        e2e = {"value": atoms * args.steps * nw / dt, "unit": "atom-timesteps/s",
               "h2d_bytes_per_step": int(atoms * 48 / args.steps),
               "d2h_bytes_per_step": int((atoms * 24 + args.steps * nw * 32) / args.steps),
               "note": "set_state(pinned host r, v) + step(K super-cycles) + get_positions (pinned) "
                       "+ energies; bytes amortised over the K steps"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, cores, k, secs = cpu_oracle_rate(cfg, seconds_target=15.0)
        cpu = {"value": rate, "unit": "atom-timesteps/s", "cores": cores, "kind": "oracle",
               "sample": f"forces-only, sampled: Algorithm 1 forces of {k} sampled atoms of {atoms:,} "
                         f"against all atoms (O(N^2) oracle, no kick/drift/binning; {secs:.1f} s on "
                         f"{cores} threads)"}

    if rank == 0:
        line = {
            "metric": "atom-timesteps/s", "value": value, "unit": "atom-timesteps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_total / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: FCC lattice (P:224) + seeded Maxwell-Boltzmann velocities, "
                    f"melted {args.equil} steps",
            "config": {"workload": cfg.name, "n_atoms": atoms, "n_slices": geo.n_slices,
                       "cells": list(geo.cells), "rho": cfg.rho, "rc": cfg.rc, "dt": cfg.dt,
                       "workers_per_gpu": W, "timesteps_per_step": nw,
                       "ensemble": f"NVT(T={args.thermostat})" if args.thermostat > 0 else "NVE",
                       "mode": "fused" if world == 1 and W == 1 and not args.staged else "staged-ring",
                       "l2": "inputs larger than L2 (state %.2f GB)" % (atoms * 76 / 1e9),
                       "parallelism": f"ring{world}", "ring_hop": args.hop if world > 1 else None},
            "roofline": {"bound": "alu", "achieved": fp64_achieved, "peak": fp64_peak,
                         "unit": "TFLOP/s", "frac": fp64_achieved / fp64_peak,
                         "traffic": (None if traffic_pa is None else traffic_pa * atoms_per_launch),
                         "traffic_note": "dram read+write bytes per launch: ncu per-atom figure "
                                         "(profiles/r*/force_traffic.json) x atoms per launch",
                         "kernel": "k_force_tile (force + kick + drift + migration key; NVT: "
                                   "force + kick, drift in k_drift)",
                         "peak_note": f"FP64: {N_SMS} SMs x {FP64_LANES_PER_SM} lanes x 2 x {sm_max:.0f} MHz",
                         "hbm": {"achieved": hbm_achieved, "peak": hbm_peak, "unit": "GB/s",
                                 "frac": hbm_achieved / hbm_peak, "peak_kind": peak_kind,
                                 "bytes_per_atom": FORCE_BYTES_PER_ATOM},
                         "force_ms_per_launch": force_ms_avg, "force_share_of_step": force_share,
                         "pairs_per_atom": pairs_per_atom},
            "steady_state": steady,
            "clocks": clk.summary(),
            "gpu_launches": launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        D.ring_disconnect(e.ctx, world)
    e.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
