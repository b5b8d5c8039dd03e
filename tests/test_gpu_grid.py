"""GPU parity of the stencil workload (include/dsea_grid.h)
against oracle/grid.py: the CUDA path evaluates the same IEEE operations in the same
order (reading G1), so every comparison is bit-exact -- single-GPU fused sweeps on
ragged shapes, the stage plan on a ring of one (W workers, B slices per stage,
pass-through cycles), rings of 2-8 GPUs over NVLink, and the full-size bench grid on
sampled planes (a slab with a halo of n planes is exact after n steps)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.conftest import run_group

from oracle import grid as OG
from paper_2507_11289_b200 import GRID_CONFIGS, GridConfig
from paper_2507_11289_b200.grid import DSEA_GRID_MODE_STAGED, Grid
from tests import inputs

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count()


def _run(c, steps, **kw):
    g = Grid(c.nx, c.ny, c.nz, c.n_slices, c.r, **kw)
    u0 = inputs.grid_field(c.nx, c.ny, c.nz, c.seed)
    g.set_field(u0)
    g.step(steps)
    out = g.field()
    st = g.stats()
    g.close()
    return u0, out, st


@pytest.mark.parametrize("shape,ns,r", [((48, 12, 10), 12, 0.1), ((33, 5, 33), 11, 1.0 / 6.0),
                                         ((20, 64, 40), 5, 0.07), ((9, 3, 3), 3, 0.15)])
def test_fused_bit_exact_vs_oracle(shape, ns, r):
    c = GridConfig("t", *shape, ns, r=r, seed=4)
    u0, out, st = _run(c, 7)
    assert np.array_equal(out, OG.run(u0, r, 7))
    assert st.cell_steps == 7 * c.n_cells


@pytest.mark.parametrize("W,B,steps", [(1, 1, 9), (2, 1, 8), (3, 1, 7), (1, 3, 6), (2, 2, 5), (3, 4, 9), (1, 0, 4)])
def test_ring_of_one_plan_bit_exact_vs_oracle(W, B, steps):
    """The Table-1 stage plan (shared with MD) with the stencil worker on one GPU:
    W workers, B slices per stage, steps not a multiple of W (pass-through, Q15)."""
    c = GRID_CONFIGS["G8"]
    u0, out, _ = _run(c, steps, workers_per_gpu=W, slices_per_stage=B, mode=DSEA_GRID_MODE_STAGED)
    assert np.array_equal(out, OG.run(u0, c.r, steps))


def test_repeated_calls_and_zero_steps():
    c = GRID_CONFIGS["G0"]
    g = Grid(c.nx, c.ny, c.nz, c.n_slices, c.r, workers_per_gpu=2, mode=DSEA_GRID_MODE_STAGED)
    u0 = inputs.grid_field(c.nx, c.ny, c.nz, 1)
    g.set_field(u0)
    for n in (3, 0, 1, 4):
        g.step(n)
    assert np.array_equal(g.field(), OG.run(u0, c.r, 8))
    g.close()


def _ring(tmp_path, n, cfg, steps, workers=1, calls=1, block=0):
    out = str(tmp_path / f"grid_{n}_{cfg}_{steps}_{workers}_{calls}_{block}.npz")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29700 + n * 11 + steps}",
           os.path.join(ROOT, "tests", "grid_ring_worker.py"), "--config", cfg, "--steps", str(steps),
           "--workers", str(workers), "--calls", str(calls), "--block", str(block), "--out", out]
    r = run_group(cmd, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("n,steps,workers,calls,block", [(2, 12, 1, 1, 0), (2, 9, 2, 2, 1), (2, 10, 1, 2, 3),
                                                         (4, 16, 1, 1, 0), (4, 10, 2, 1, 2), (8, 16, 1, 1, 0)])
def test_ring_bit_exact_vs_oracle(tmp_path, n, steps, workers, calls, block):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    c = GRID_CONFIGS["G8"]
    r = _ring(tmp_path, n, "G8", steps, workers, calls, block)
    u0 = inputs.grid_field(c.nx, c.ny, c.nz, c.seed)
    assert np.array_equal(r["u"], OG.run(u0, c.r, steps))
    assert int(r["hop"][0]) > 0           # slices really crossed NVLink


def test_full_size_bench_grid_sampled_planes():
    """G1 (512^3 cells, 128 slices) in the bench's launch configuration: after 3
    steps, plane slabs at both walls and in the interior equal the oracle run on the
    slab with a 3-plane halo, bit for bit."""
    c = GRID_CONFIGS["G1"]
    n = 3
    u0, out, _ = _run(c, n)
    for a, b in ((0, 2), (255, 258), (c.nx - 2, c.nx)):
        lo, hi = max(a - n, 0), min(b + n, c.nx)
        ref = OG.run(u0[lo:hi], c.r, n)[a - lo:b - lo]
        assert np.array_equal(out[a:b], ref), (a, b)


@pytest.mark.parametrize("env", [{"DSEA_FTCS": "col"}, {"DSEA_FTCS_GRID": "3", "DSEA_FTCS_ROWS": "2"},
                                 {"DSEA_FTCS_NS": "2", "DSEA_FTCS_ROWS": "1", "DSEA_FTCS_GRID": "5"},
                                 {"DSEA_FTCS_NS": "4", "DSEA_FTCS_ROWS": "3"}])
@pytest.mark.parametrize("shape,ns", [((48, 12, 10), 12), ((20, 64, 40), 5), ((33, 7, 34), 11)])
def test_stencil_kernel_variants_bit_exact(monkeypatch, env, shape, ns):
    """The bulk-copy plane pipeline (k_ftcs_tma) with forced tilings -- one-row y-tiles,
    several items per CTA (the load sequence running on across items), 2 and 4 stages
    -- and the register-column kernel (odd nz always takes it): bit-exact vs the
    oracle on ragged shapes, fused and on the staged plan."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    c = GridConfig("t", *shape, ns, r=0.11, seed=5)
    u0, out, _ = _run(c, 5)
    assert np.array_equal(out, OG.run(u0, c.r, 5))
    W = 2 if ns >= 8 else 1               # the staged plan needs >= 2 + W blocks
    u0, out, _ = _run(c, 5, workers_per_gpu=W, slices_per_stage=2, mode=DSEA_GRID_MODE_STAGED)
    assert np.array_equal(out, OG.run(u0, c.r, 5))
