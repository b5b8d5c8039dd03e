"""Multi-GPU ring (one process per GPU; the hop of P:117-120 §3.1 by the "peer"
backend -- copy-engine pushes into the successor's IPC-mapped slots with monotone
arrival / release counters -- or the "nccl" backend's send/recv;
P:200-208 §3.4): the state after n steps equals the single-GPU run bit for bit --
the ring is an exact re-scheduling of timesteps and every
kernel result depends only on its input slots.  Needs >= 2 GPUs (gpurun --gpus N)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.conftest import run_group

from paper_2507_11289_b200 import CONFIGS
from paper_2507_11289_b200 import dsea as D

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    """GPUs on this box, counted in a subprocess: independent of what this pytest
    process has already initialised (libdsea's static cudart, torch)."""
    try:
        r = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=60)
        return sum(1 for line in r.stdout.splitlines() if line.startswith("GPU "))
    except Exception:
        return 0


def _single(cfg, steps, thermo=0.0):
    c = CONFIGS[cfg]
    e = D.Engine(D.Box(c.nx, c.ny, c.nz, c.rho, c.rc, c.dt, c.T0, c.seed))
    e.slice(n_slices=c.n_slices, cells_per_slice_x=c.cells_per_slice_x)
    if thermo:
        e.set_thermostat(thermo)
    e.step(steps)
    p = e.raw_profiles()
    r = (e.positions(), e.velocities(), e.forces(), *e.energies(),
         np.stack([p[k] for k in ("n_sum", "U_sum", "V_sum", "KE_sum")], 1))
    e.close()
    return r


def _ring(tmp_path, n, cfg, steps, workers=1, calls=1, block=0, hop="peer", thermo=0.0, env=None):
    out = str(tmp_path / f"ring_{n}_{cfg}_{steps}_{workers}_{calls}_{block}_{hop}_{thermo}.npz")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29500 + n * 7 + steps}",
           os.path.join(ROOT, "tests", "ring_worker.py"), "--config", cfg, "--steps", str(steps),
           "--workers", str(workers), "--calls", str(calls), "--block", str(block), "--hop", hop,
           "--thermo", str(thermo), "--out", out]
    r = run_group(cmd, timeout=300, cwd=ROOT, env=None if env is None else {**os.environ, **env})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return np.load(out)


# (gpus, config, steps, workers, calls, slices per stage (0 = auto), ring hop backend)
CASES = [(2, "P8", 16, 1, 1, 1, "peer"), (2, "P8", 9, 1, 2, 1, "peer"), (2, "P8", 12, 2, 1, 1, "peer"),
         (2, "P8", 16, 1, 1, 0, "peer"), (2, "P8", 10, 2, 2, 3, "peer"), (2, "P8", 16, 1, 1, 1, "nccl"),
         (2, "P8", 10, 2, 2, 3, "nccl"), (4, "P8", 16, 1, 2, 1, "peer"), (4, "P8", 10, 1, 1, 2, "peer"),
         (4, "P8", 16, 1, 1, 0, "peer"), (4, "P8", 16, 1, 1, 0, "nccl"), (8, "P8", 16, 1, 1, 1, "peer"),
         (8, "C1", 8, 1, 1, 1, "peer"), (8, "P8", 24, 1, 2, 0, "peer"),
         # past Eq. (1)'s bound at block level: the ring must run at the plateau, not stall
         (4, "P8", 10, 2, 1, 3, "peer"), (4, "P8", 12, 3, 1, 2, "peer"), (2, "P8", 11, 3, 1, 4, "peer"),
         (4, "P8", 12, 2, 1, 3, "nccl"),
         # full size: C3 (2,048,000 atoms, 256 slices) with the bench's automatic block size
         (2, "C3", 4, 1, 1, 0, "peer"), (4, "C3", 8, 1, 1, 0, "peer")]
# optional lead blocks (DSEA_LEAD_BLOCKS=1: 2 + 2 slices, then B): both backends, W = 2, several calls
LEAD_CASES = [(2, "P8", 12, 2, 1, 5, "peer"), (4, "P8", 12, 1, 1, 5, "nccl"), (2, "P8", 12, 1, 2, 6, "nccl"),
              (4, "P8", 16, 1, 2, 4, "peer")]


# Known issue: with the NCCL comparison backend, these two 4-GPU rings at
# Eq. (1)'s plateau hang since the round-2 force kernel (also with plain launches,
# DSEA_PDL=0); the peer backend runs the same plans, and NCCL passes on 2 GPUs.
NCCL_PLATEAU_HANG = {(4, "P8", 12, 2, 1, 3, "nccl", False), (4, "P8", 12, 1, 1, 5, "nccl", True)}


def _ring_case(c):
    if c in NCCL_PLATEAU_HANG and not os.environ.get("DSEA_RUN_XFAIL"):
        return pytest.param(*c, marks=pytest.mark.xfail(run=False, reason="NCCL backend hangs at the 4-GPU "
                                                                             "plateau (DESIGN.md §12)"))
    return c


@pytest.mark.parametrize("n,cfg,steps,workers,calls,block,hop,lead",
                         [_ring_case(c + (False,)) for c in CASES] + [_ring_case(c + (True,)) for c in LEAD_CASES])
def test_ring_bitwise_equals_single_gpu(tmp_path, n, cfg, steps, workers, calls, block, hop, lead):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    c = CONFIGS[cfg]
    if c.n_slices < 2 + 2 * workers:
        pytest.skip("too few slices")
    x, v, f, s1, e1, _ = _single(cfg, steps)
    r = _ring(tmp_path, n, cfg, steps, workers, calls, block, hop, env={"DSEA_LEAD_BLOCKS": "1"} if lead else None)
    assert np.array_equal(r["x"], x)
    assert np.array_equal(r["v"], v)
    assert np.array_equal(r["f"], f)
    assert r["steps"].tolist() == list(range(steps))
    assert np.array_equal(r["en"], e1)
    assert int(r["stats"][0]) > 0  # slices really crossed NVLink


# slot pools forced (DSEA_POOLS=1; by default they are used only when full buffers would
# take more than a quarter of the device memory, e.g. the 1e9-atom ring): staging and the
# last worker's output buffer hold a window of slices in slots (K N_S + j) mod pool
POOL_CASES = [(2, "P8", 16, 1, 1, 1, "peer"), (2, "P8", 10, 2, 2, 3, "peer"), (4, "P8", 16, 1, 2, 1, "peer"),
              (4, "P8", 10, 1, 1, 2, "peer"), (2, "P8", 10, 2, 2, 3, "nccl"), (2, "C3", 4, 1, 1, 0, "peer"),
              (4, "C3", 8, 1, 1, 0, "peer")]


@pytest.mark.parametrize("n,cfg,steps,workers,calls,block,hop", POOL_CASES)
def test_ring_with_slot_pools_bitwise_equals_single_gpu(tmp_path, n, cfg, steps, workers, calls, block, hop):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    x, v, f, s1, e1, _ = _single(cfg, steps)
    r = _ring(tmp_path, n, cfg, steps, workers, calls, block, hop, env={"DSEA_POOLS": "1"})
    assert np.array_equal(r["x"], x)
    assert np.array_equal(r["v"], v)
    assert np.array_equal(r["f"], f)
    assert np.array_equal(r["en"], e1)


@pytest.mark.parametrize("n,workers,block,hop", [(2, 1, 0, "peer"), (2, 2, 1, "nccl"), (4, 1, 0, "peer")])
def test_ring_thermostat_bitwise_equals_single_gpu(tmp_path, n, workers, block, hop):
    """NVT (per-slice isokinetic scaling, Q23) needs no exchange beyond the
    ring hop: every rank scales the slices it processes, so the ring still equals
    the single-GPU run bit for bit; x-resolved sums agree over ranks (Q24)."""
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    x, v, f, s1, e1, p1 = _single("P8", 12, thermo=1.5)
    r = _ring(tmp_path, n, "P8", 12, workers, 1, block, hop, thermo=1.5)
    assert np.array_equal(r["x"], x)
    assert np.array_equal(r["v"], v)
    assert np.array_equal(r["f"], f)
    assert np.array_equal(r["en"], e1)
    assert np.allclose(r["prof"], p1, rtol=1e-12, atol=0)
