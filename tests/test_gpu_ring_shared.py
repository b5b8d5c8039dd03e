"""The ring on ONE B200: 2 and 3 ranks (processes) share GPU 0, so the round-end
driver box exercises the real ring hop -- CUDA IPC mapping of the successor's slot
buffer, copy-engine push, monotone arrival/release counters as stream flags
(§3.1, §3.4) -- that the multi-GPU tests (tests/test_gpu_ring.py)
cover only on boxes with 2+ GPUs.  gloo carries the plumbing (handle exchange,
barriers); NCCL refuses two ranks on one device.

Each case is compared element by element with the CPU oracle (the plain sequential
integrator: the ring is an exact re-scheduling of timesteps) --
positions within 1e-8 sigma (Q14), forces within 1e-10 relative (Q13), the energy
series within 1e-10 -- and bitwise with the single-GPU run."""
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.conftest import run_group

import oracle
from paper_2507_11289_b200 import CONFIGS
from paper_2507_11289_b200 import dsea as D

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _single(cfg, steps):
    c = CONFIGS[cfg]
    e = D.Engine(D.Box(c.nx, c.ny, c.nz, c.rho, c.rc, c.dt, c.T0, c.seed))
    e.slice(n_slices=c.n_slices, cells_per_slice_x=c.cells_per_slice_x)
    x0, v0 = e.positions(), e.velocities()
    e.step(steps)
    r = dict(x0=x0, v0=v0, x=e.positions(), v=e.velocities(), f=e.forces(), en=e.energies()[1])
    e.close()
    return r


def _ring(tmp_path, n, cfg, steps, workers, calls, block, pools=False):
    out = str(tmp_path / f"shared_{n}_{cfg}_{steps}_{workers}_{calls}_{block}_{int(pools)}.npz")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29600 + 11 * n + steps + 3 * workers + block}",
           os.path.join(ROOT, "tests", "ring_worker.py"), "--config", cfg, "--steps", str(steps),
           "--workers", str(workers), "--calls", str(calls), "--block", str(block), "--hop", "peer",
           "--shared-device", "--out", out]
    env = {**os.environ, "DSEA_POOLS": "1"} if pools else None
    r = run_group(cmd, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return np.load(out)


# (ranks, config, steps, workers per rank, calls, slices per stage (0 = auto), slot pools
# forced (DSEA_POOLS=1: staging and the last output buffer hold a window of slices))
CASES = [(2, "P8", 12, 1, 2, 1, False), (2, "P8", 12, 2, 1, 0, False), (3, "P8", 13, 1, 1, 0, False),
         (3, "P8", 12, 2, 2, 2, False), (2, "C1", 10, 1, 1, 0, False), (3, "C1", 9, 2, 2, 1, False),
         (2, "P8", 12, 1, 2, 1, True), (3, "P8", 12, 2, 2, 2, True), (3, "C1", 9, 2, 2, 1, True)]


@pytest.mark.parametrize("n,cfg,steps,workers,calls,block,pools", CASES)
def test_shared_device_ring_equals_oracle_and_single_gpu(tmp_path, n, cfg, steps, workers, calls, block, pools):
    c = CONFIGS[cfg]
    s = _single(cfg, steps)
    r = _ring(tmp_path, n, cfg, steps, workers, calls, block, pools)
    g = oracle.geometry(c.nx, c.ny, c.nz, c.rho, c.rc, c.n_slices, c.cells_per_slice_x)
    xo, vo, Fo, eo = oracle.run(s["x0"], s["v0"], np.zeros_like(s["x0"]), g.b, c.rc, c.dt, steps)
    # against the oracle
    d = r["x"] - xo
    d[:, 1:] -= g.b[1:] * np.round(d[:, 1:] / g.b[1:])
    assert np.abs(d).max() <= 1e-8
    frms = np.sqrt((Fo ** 2).sum(1).mean())
    ferr = np.sqrt(((r["f"] - Fo) ** 2).sum(1)) / np.maximum(np.sqrt((Fo ** 2).sum(1)), frms)
    assert ferr.max() <= 1e-10, ferr.max()
    assert r["steps"].tolist() == list(range(steps))
    assert np.allclose(r["en"][:, 3], eo[:, 3], rtol=1e-10)
    # bitwise against the single-GPU run
    assert np.array_equal(r["x"], s["x"])
    assert np.array_equal(r["v"], s["v"])
    assert np.array_equal(r["f"], s["f"])
    assert np.array_equal(r["en"], s["en"])
    assert int(r["stats"][0]) > 0          # slices really took the ring hop
