"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same
seeded inputs.  Tolerances from the north star (BASELINE.json) with readings
Q13/Q14:
  cells and slice membership ............ bit-exact (oracle binning of the GPU positions)
  per-atom forces (fp64) ................ |dF| <= 1e-10 * max(|F_oracle|, F_rms)
  positions after 10 steps .............. <= 1e-8 sigma (minimum image in y/z)
  energy drift over 1000 NVE steps ...... |dE/E| < 1e-4
Run on a B200 with -m gpu."""
import numpy as np
import pytest

import oracle
from paper_2507_11289_b200 import CONFIGS
from paper_2507_11289_b200 import dsea as D
from tests import inputs

pytestmark = pytest.mark.gpu


def _engine(cfg, seed=None, **kw):
    c = CONFIGS[cfg] if isinstance(cfg, str) else cfg
    e = D.Engine(D.Box(c.nx, c.ny, c.nz, c.rho, c.rc, c.dt, c.T0, c.seed if seed is None else seed))
    kw.setdefault("n_slices", c.n_slices)
    kw.setdefault("cells_per_slice_x", c.cells_per_slice_x)
    e.slice(**kw)
    return e, c


def _geom(c):
    return oracle.geometry(c.nx, c.ny, c.nz, c.rho, c.rc, c.n_slices, c.cells_per_slice_x)


def _force_close(Fg, Fo, tol=1e-10):
    frms = np.sqrt((Fo ** 2).sum(1).mean())
    err = np.sqrt(((Fg - Fo) ** 2).sum(1))
    ref = np.maximum(np.sqrt((Fo ** 2).sum(1)), frms)
    worst = (err / ref).max()
    assert worst <= tol, worst
    return worst


def _min_image(d, b):
    d = d.copy()
    d[:, 1:] -= b[1:] * np.round(d[:, 1:] / b[1:])
    return d


def _cells_exact(e, c):
    g = _geom(c)
    x = e.positions()
    cg, sg = e.cells()
    co, so = oracle.bin_atoms(x, g.l, g.cells, c.cells_per_slice_x)
    assert np.array_equal(cg, co)
    assert np.array_equal(sg, so)
    counts = np.bincount(sg, minlength=g.n_slices)
    assert counts.sum() == c.n_atoms


@pytest.mark.parametrize("cfg", ["C1", "P8"])
def test_initial_binning_bit_exact(cfg):
    e, c = _engine(cfg)
    x0 = oracle.lattice(c.nx, c.ny, c.nz, _geom(c).a)
    assert np.array_equal(e.positions(), x0)
    _cells_exact(e, c)


@pytest.mark.parametrize("cfg", ["C1", "P8"])
def test_first_step_forces_energies_lattice(cfg):
    """Step 0 from the lattice: F_new(r_0), U, V, KE against the oracle."""
    e, c = _engine(cfg)
    g = _geom(c)
    x0 = e.positions()
    v0 = e.velocities()
    e.step(1)
    xo, vo, Fo, eo = oracle.run(x0, v0, np.zeros_like(x0), g.b, c.rc, c.dt, 1)
    _force_close(e.forces(), Fo)
    steps, en = e.energies()
    assert steps.tolist() == [0]
    assert np.allclose(en[0, :3], eo[0, :3], rtol=1e-10, atol=1e-9)
    assert np.max(np.abs(e.positions() - xo)) < 1e-12
    _cells_exact(e, c)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_forces_thermalised_state(seed):
    """Q13 on a disordered state: lattice jittered by up to 0.25 sigma, Gaussian
    velocities, injected through dsea_set_state."""
    e, c = _engine("C1")
    g = _geom(c)
    x = inputs.jitter(oracle.lattice(c.nx, c.ny, c.nz, g.a), g.b, 0.25, seed)
    v = inputs.gaussian_velocities(c.n_atoms, 1.0, seed)
    e.set_state(x, v)
    _cells_exact(e, c)
    e.step(1)
    _, _, Fo, eo = oracle.run(x, v, np.zeros_like(x), g.b, c.rc, c.dt, 1)
    _force_close(e.forces(), Fo)
    _, en = e.energies()
    assert np.allclose(en[-1, :3], eo[0, :3], rtol=1e-10)


@pytest.mark.parametrize("cfg,seed", [("C1", 11289), ("C1", 5), ("P8", 7)])
def test_positions_after_10_steps(cfg, seed):
    """Q14: positions after 10 steps within 1e-8 sigma of the oracle; cells exact."""
    e, c = _engine(cfg, seed=seed)
    g = _geom(c)
    x0, v0 = e.positions(), e.velocities()
    e.step(10)
    xo, vo, Fo, eo = oracle.run(x0, v0, np.zeros_like(x0), g.b, c.rc, c.dt, 10)
    d = _min_image(e.positions() - xo, g.b)
    assert np.max(np.abs(d)) < 1e-8
    assert np.max(np.abs(e.velocities() - vo)) < 1e-8
    _force_close(e.forces(), Fo, tol=1e-8)
    _, en = e.energies()
    assert np.allclose(en[:, 3], eo[:, 3], rtol=1e-10)
    _cells_exact(e, c)


def test_wall_hits_match_oracle():
    """Mirror walls (reading Q2) against the oracle: edge atoms driven into
    both walls, 60 steps, positions within 1e-8."""
    e, c = _engine("C1")
    g = _geom(c)
    x = oracle.lattice(c.nx, c.ny, c.nz, g.a)
    v = oracle.velocities(c.n_atoms, 9, 1.0)
    v[x[:, 0] < 0.5 * g.a, 0] = -6.0
    v[x[:, 0] > g.b[0] - 0.5 * g.a, 0] = 6.0
    e.set_state(x, v)
    e.step(60)
    xo, vo, Fo, _ = oracle.run(x, v, np.zeros_like(x), g.b, c.rc, c.dt, 60)
    assert np.max(np.abs(_min_image(e.positions() - xo, g.b))) < 1e-8
    assert np.max(np.abs(e.velocities() - vo)) < 1e-7
    _cells_exact(e, c)


@pytest.mark.parametrize("rc,c_per,ns", [(4.0, 1, 0), (2.5, 2, 4), (2.5, 3, 0), (4.0, 2, 0)])
def test_cutoff_and_slice_thickness_variants(rc, c_per, ns):
    """C5-style variants at oracle size: rc = 4.0 and 2-3 cells per slice."""
    from paper_2507_11289_b200.configs import Config
    c = Config("v", 24 if rc < 3 else 30, 8, 8, ns, rc=rc, cells_per_slice_x=c_per)
    g = _geom(c)
    assert g.feasible
    e, _ = _engine(c, seed=3)
    x = inputs.jitter(oracle.lattice(c.nx, c.ny, c.nz, g.a), g.b, 0.15, 4)
    v = inputs.gaussian_velocities(c.n_atoms, 0.8, 4)
    e.set_state(x, v)
    e.step(3)
    xo, vo, Fo, eo = oracle.run(x, v, np.zeros_like(x), g.b, c.rc, c.dt, 3)
    _force_close(e.forces(), Fo, tol=1e-9)
    assert np.max(np.abs(_min_image(e.positions() - xo, g.b))) < 1e-10
    _, en = e.energies()
    assert np.allclose(en[:, 3], eo[:, 3], rtol=1e-10)
    _cells_exact(e, c)


@pytest.mark.parametrize("W,B,pools", [(1, 1, 0), (2, 1, 0), (3, 1, 0), (1, 3, 0), (2, 4, 0), (3, 2, 0), (3, 5, 0),
                                       (1, 1, 1), (1, 3, 1), (2, 4, 1), (3, 5, 1)])
def test_ring_of_one_bitwise_equals_fused(monkeypatch, W, B, pools):
    """The stage schedule (Table 1 for B = 1; B slices per stage otherwise; W workers
    sequential on one GPU) and the fused whole-domain pass compute the same
    unit results: bitwise equal states after 7 steps (7 is not a multiple of W = 2, 3:
    pass-through workers, Q15).  pools = 1: staging buffers of 2 B + 4 slices (slots
    (K N_S + j) mod pool; the previous super-cycle's last slice is binned after the
    next one's first block)."""
    ref, c = _engine("P8")
    ref.step(7)
    monkeypatch.setenv("DSEA_POOLS", "1" if pools else "")
    e, _ = _engine("P8", workers_per_gpu=W, mode=D.DSEA_MODE_STAGED, slices_per_stage=B)
    e.step(7)
    assert np.array_equal(e.positions(), ref.positions())
    assert np.array_equal(e.velocities(), ref.velocities())
    assert np.array_equal(e.forces(), ref.forces())
    s1, e1 = ref.energies()
    s2, e2 = e.energies()
    assert s1.tolist() == s2.tolist() == list(range(7))
    assert np.array_equal(e1, e2)


@pytest.mark.parametrize("W,B", [(2, 4), (3, 3)])
def test_ring_of_one_single_slice_last_block(W, B):
    """13 slices in blocks of B leave a last block of one slice; with W > 1 the next
    worker's pass on the previous block needs that slice in the same stage, so the
    plan finalises it with its own block (found by tests/test_plan_sim.py): bitwise
    equal to the fused pass."""
    from paper_2507_11289_b200.configs import Config
    c = Config("r13", 20, 5, 5, 13)
    ref, _ = _engine(c)
    ref.step(5)
    e, _ = _engine(c, workers_per_gpu=W, mode=D.DSEA_MODE_STAGED, slices_per_stage=B)
    e.step(5)
    assert np.array_equal(e.positions(), ref.positions())
    assert np.array_equal(e.velocities(), ref.velocities())
    assert np.array_equal(e.energies()[1], ref.energies()[1])


@pytest.mark.parametrize("maxh,rc", [("24", 2.5), ("40", 2.5), ("", 4.0)])
def test_deterministic_with_mid_chunk_flushes(monkeypatch, maxh, rc):
    """Hit lists shorter than one chunk's hits (small DSEA_MAXH, or rc = 4.0 with ~107
    hits per lane) force flushes in the middle of a chunk; the result must still not
    depend on which warp or CTA took the chunk: reruns and the staged path are
    bitwise equal to the fused path."""
    from paper_2507_11289_b200.configs import Config
    if maxh:
        monkeypatch.setenv("DSEA_MAXH", maxh)
    c = Config("d", 30 if rc > 3 else 20, 8, 8, 0, rc=rc)

    def run(**kw):
        e, _ = _engine(c, **kw)
        e.step(4)
        r = e.positions(), e.velocities(), e.forces(), e.energies()[1]
        e.close()
        return r
    a, b = run(), run()
    s = run(workers_per_gpu=2, mode=D.DSEA_MODE_STAGED, slices_per_stage=1)
    for x, y, z in zip(a, b, s):
        assert np.array_equal(x, y)
        assert np.array_equal(x, z)


def test_deterministic_rerun():
    a, _ = _engine("C1")
    b, _ = _engine("C1")
    a.step(20)
    b.step(10)
    b.step(10)
    assert np.array_equal(a.positions(), b.positions())
    assert np.array_equal(a.energies()[1], b.energies()[1])


@pytest.mark.slow
def test_nve_energy_drift_1000_steps():
    """North star: |dE/E| < 1e-4 over 1000 steps on C1 (Q19), and the GPU energy
    series tracks the oracle's for the first 50 steps."""
    e, c = _engine("C1")
    g = _geom(c)
    x0, v0 = e.positions(), e.velocities()
    e.step(1000)
    _, en = e.energies()
    E = en[:, 3]
    drift = np.max(np.abs(E - E[0])) / abs(E[0])
    assert drift < 1e-4, drift
    _, _, _, eo = oracle.run(x0, v0, np.zeros_like(x0), g.b, c.rc, c.dt, 50)
    assert np.allclose(E[:50], eo[:, 3], rtol=1e-9)


def test_full_size_c2_sampled_forces_and_cells():
    """C2 (256,000 atoms, 64 slices) in the launch configuration bench.py times:
    forces on 512 sampled atoms against the oracle's all-pairs sums, every atom's
    cell bit-exact, atom count conserved."""
    e, c = _engine("C2")
    g = _geom(c)
    x = inputs.jitter(oracle.lattice(c.nx, c.ny, c.nz, g.a), g.b, 0.2, 8)
    v = inputs.gaussian_velocities(c.n_atoms, 1.0, 8)
    e.set_state(x, v)
    e.step(1)
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(c.n_atoms, 512, replace=False))
    Fo, _ = oracle.forces_subset(x, g.b, c.rc, idx)
    Fg = e.forces()[idx]
    frms = np.sqrt((Fo ** 2).sum(1).mean())
    err = np.sqrt(((Fg - Fo) ** 2).sum(1)) / np.maximum(np.sqrt((Fo ** 2).sum(1)), frms)
    assert err.max() <= 1e-10
    _cells_exact(e, c)


def test_full_size_c4_bench_workload():
    """C4 -- the bench workload (16,384,000 atoms, 109 slices, paper slicing rule) -- in
    the launch configuration bench.py times (fused, one GPU): forces on 256 sampled
    atoms against the oracle's all-pairs sums (Q13), every atom's cell and slice
    bit-exact (Q4), and over 10 further steps the properties that hold at any size:
    atom count, zero net force (the walls exert none, Alg. 1 pairs cancel) and
    conserved y/z momentum (the walls only flip v_x, Q1/Q2)."""
    e, c = _engine("C4")
    g = _geom(c)
    x = inputs.jitter(oracle.lattice(c.nx, c.ny, c.nz, g.a), g.b, 0.2, 9)
    v = inputs.gaussian_velocities(c.n_atoms, 1.0, 9)
    e.set_state(x, v)
    e.step(1)
    rng = np.random.default_rng(1)
    idx = np.sort(rng.choice(c.n_atoms, 256, replace=False))
    Fo, _ = oracle.forces_subset(x, g.b, c.rc, idx)
    F = e.forces()
    frms_o = np.sqrt((Fo ** 2).sum(1).mean())
    err = np.sqrt(((F[idx] - Fo) ** 2).sum(1)) / np.maximum(np.sqrt((Fo ** 2).sum(1)), frms_o)
    assert err.max() <= 1e-10, err.max()
    _cells_exact(e, c)
    p0 = e.velocities().sum(0)
    e.step(10)
    F = e.forces()
    frms = np.sqrt((F ** 2).sum(1).mean())
    assert np.abs(F.sum(0)).max() <= 1e-12 * c.n_atoms * frms
    v1 = e.velocities()
    assert v1.shape[0] == c.n_atoms
    assert np.abs(v1.sum(0)[1:] - p0[1:]).max() <= 1e-10 * np.abs(v1).sum(0)[1:].max()
    _cells_exact(e, c)
    e.close()


def test_error_paths():
    e, c = _engine("C1")
    g = _geom(c)
    # step 0 is a no-op
    e.step(0)
    assert e.energies()[0].size == 0
    # outside the box -> EINVAL
    x = oracle.lattice(c.nx, c.ny, c.nz, g.a)
    v = np.zeros_like(x)
    bad = x.copy()
    bad[5, 1] = -1.0
    with pytest.raises(D.DseaError) as ei:
        e.set_state(bad, v)
    assert ei.value.status == D.DSEA_EINVAL
    # all atoms squeezed into slice 0 -> ECAPACITY
    sq = x.copy()
    sq[:, 0] = sq[:, 0] * (g.w * 0.99 / g.b[0])
    with pytest.raises(D.DseaError) as ei:
        e.set_state(sq, v)
    assert ei.value.status == D.DSEA_ECAPACITY
    # an atom jumping more than one slice -> EUNSTABLE
    e2, _ = _engine("C1")
    v2 = np.zeros_like(x)
    v2[100, 0] = 5000.0
    e2.set_state(x, v2)
    with pytest.raises(D.DseaError) as ei:
        e2.step(1)
    assert ei.value.status == D.DSEA_EUNSTABLE
    # stepping before slicing -> ESTATE
    ctx = D.dsea_init(c.nx, c.ny, c.nz, c.rho, c.rc)
    with pytest.raises(D.DseaError) as ei:
        D.dsea_step(ctx, 1)
    assert ei.value.status == D.DSEA_ESTATE
    D.dsea_destroy(ctx)


def test_overfull_cell_binned_exactly():
    """A cell far above its expected occupancy (100 atoms where ~18 are typical) is
    ranked by k_bin_gather's global-memory path: positions round-trip exactly by id,
    every cell is bit-exact against the oracle's binning, and a step runs on it."""
    e, c = _engine("C1")
    g = _geom(c)
    x = oracle.lattice(c.nx, c.ny, c.nz, g.a)
    rng = np.random.default_rng(3)
    lo = np.array([2, 2, 2]) * g.l
    idx = rng.choice(c.n_atoms, 100, replace=False)
    x[idx] = lo + rng.random((100, 3)) * g.l * 0.999
    v = np.zeros_like(x)
    e.set_state(x, v)
    assert np.array_equal(e.positions(), x)
    _cells_exact(e, c)
    cg, _ = e.cells()
    assert np.sum(np.all(cg == [2, 2, 2], axis=1)) >= 100


@pytest.mark.parametrize("mode,W,B", [(D.DSEA_MODE_FUSED, 1, 0), (D.DSEA_MODE_STAGED, 2, 3)])
def test_empty_slices(mode, W, B):
    """Edge case: half the slices hold no atoms.  A rho = 0.3 box (P8 shape) whose lattice
    is compressed into the left half along x (local density 0.6): slices 16-31 are
    empty, the occupied ones hold twice the mean (capacity_factor 3).  Forces, positions
    after 5 steps and cells against the oracle (Q13, Q14, Q4), in the fused pass and on
    a staged ring of one."""
    from paper_2507_11289_b200 import Config
    c = Config("E", 48, 5, 5, 32, rho=0.3)
    g = _geom(c)
    x = oracle.lattice(c.nx, c.ny, c.nz, g.a)
    x[:, 0] *= 0.5
    v = inputs.gaussian_velocities(c.n_atoms, 0.3, 4)
    e, _ = _engine(c, mode=mode, workers_per_gpu=W, slices_per_stage=B, capacity_factor=3.0)
    e.set_state(x, v)
    _, sl = e.cells()
    assert sl.max() < c.n_slices // 2 + 1
    e.step(5)
    xo, vo, Fo, _ = oracle.run(x, v, np.zeros_like(x), g.b, c.rc, c.dt, 5)
    _force_close(e.forces(), Fo)
    d = _min_image(e.positions() - xo, g.b)
    assert np.abs(d).max() <= 1e-8
    _cells_exact(e, c)
    e.close()


def test_melted_state_parity():
    """Reading Q13 asks for thermalised states: C1 melted for 200 steps by the ORACLE
    (T* drops from 1.0 to ~0.55, the lattice order is gone), injected through
    dsea_set_state with its F_new (the next kick needs F_old), then 10 GPU steps against
    10 more oracle steps: first-step forces within 1e-10 (Q13), positions within 1e-8
    after 10 steps (Q14), energies within 1e-10, cells bit-exact."""
    c = CONFIGS["C1"]
    g = _geom(c)
    x0 = oracle.lattice(c.nx, c.ny, c.nz, g.a)
    v0 = oracle.velocities(c.n_atoms, c.seed, c.T0)
    xm, vm, Fm, _ = oracle.run(x0, v0, np.zeros_like(x0), g.b, c.rc, c.dt, 200)
    e, _ = _engine("C1")
    e.set_state(xm, vm, Fm)
    _cells_exact(e, c)
    e.step(1)
    x1, v1, F1, e1 = oracle.run(xm, vm, Fm, g.b, c.rc, c.dt, 1)
    _force_close(e.forces(), F1)
    assert np.allclose(e.energies()[1][-1, :3], e1[0, :3], rtol=1e-10)
    e.step(9)
    x10, v10, F10, e10 = oracle.run(x1, v1, F1, g.b, c.rc, c.dt, 9)
    assert np.abs(_min_image(e.positions() - x10, g.b)).max() <= 1e-8
    assert np.abs(e.velocities() - v10).max() <= 1e-8
    _, en = e.energies()
    assert np.allclose(en[-9:, 3], e10[:, 3], rtol=1e-10)
    _cells_exact(e, c)


def test_full_size_c4_melted_bench_state():
    """The exact state bench.py times: C4 from the lattice, melted 200 GPU steps (the
    bench's --equil default).  Forces of that state (one more step) on 256 sampled
    atoms against the oracle's all-pairs sums (Q13), every cell and slice bit-exact."""
    e, c = _engine("C4")
    g = _geom(c)
    e.step(200)
    x = e.positions()
    _cells_exact(e, c)
    e.step(1)
    rng = np.random.default_rng(2)
    idx = np.sort(rng.choice(c.n_atoms, 256, replace=False))
    Fo, _ = oracle.forces_subset(x, g.b, c.rc, idx)
    F = e.forces()[idx]
    frms = np.sqrt((Fo ** 2).sum(1).mean())
    err = np.sqrt(((F - Fo) ** 2).sum(1)) / np.maximum(np.sqrt((Fo ** 2).sum(1)), frms)
    assert err.max() <= 1e-10, err.max()
    e.close()


def test_pair_exactly_at_cutoff():
    """Inclusive cutoff r^2 <= rc^2 (reading Q5) on the GPU: a pair at exactly
    rc = 2.5 along x contributes the attractive force 24 (2 rc^-13 - rc^-7) and zero
    energy, a pair one ulp beyond rc contributes nothing.  Every other atom sits on a
    simple cubic grid of spacing > rc, more than rc away from the pairs, so the pair
    terms are the only ones; results against the oracle."""
    from paper_2507_11289_b200.configs import Config
    c = Config("cut", 10, 10, 10, 0, rho=0.05)
    g = _geom(c)
    n = c.n_atoms
    pa = np.array([[10.0, 11.0, 12.0], [12.5, 11.0, 12.0],            # exactly rc apart
                   [30.0, 31.0, 30.0], [np.nextafter(32.5, 40.0), 31.0, 30.0]])   # 1 ulp beyond
    # one grid plane per slice along x (spacing w), 16 x 16 per plane: every slot holds
    # at most 256 + 4 atoms
    ns = g.n_slices
    gx, gy = g.b[0] / ns, g.b[1] / 16
    grid = np.stack(np.meshgrid((np.arange(ns) + 0.5) * gx, (np.arange(16) + 0.5) * gy,
                                (np.arange(16) + 0.5) * gy, indexing="ij"), -1).reshape(-1, 3)
    far = np.min(np.linalg.norm(grid[:, None, :] - pa[None, :, :], axis=2), axis=1) > 3.0
    x = np.concatenate([pa, grid[far][: n - 4]])
    assert x.shape[0] == n and min(gx, gy) > c.rc
    v = np.zeros_like(x)
    e, _ = _engine(c, capacity_factor=2.0)   # the start lattice puts two planes in some slices
    e.set_state(x, v)
    e.step(1)
    _, _, Fo, eo = oracle.run(x, v, np.zeros_like(x), g.b, c.rc, c.dt, 1)
    F = e.forces()
    mag = 24 * (2 * c.rc ** -13 - c.rc ** -7)   # F_abs r at rc: negative (attractive)
    tol = 1e-12 * abs(mag)          # the GPU's 1/r^2: rcp + one Newton step
    assert abs(F[0, 0] + mag) <= tol and abs(F[1, 0] - mag) <= tol    # atom 0 pulled to +x
    assert np.all(F[2:] == 0.0) and np.all(Fo[2:] == 0.0)
    assert np.abs(F - Fo).max() <= tol
    _, en = e.energies()
    # U(rc) = 0: both sides cancel terms of ~4e-3 (s6^2 - s6 + U_shift), so the zero is
    # only resolved to ~1e-15 -- a few ulps of the terms
    assert abs(en[0, 0]) <= 1e-14 and abs(eo[0, 0]) <= 1e-14


def test_first_step_forces_rc4():
    """rc = 4.0 (C5's long cutoff: ~214 in-cutoff pairs per atom, several hit-list
    flushes per chunk) on a jittered state: first-step forces within 1e-10 (Q13) and
    energies within 1e-10 of the oracle."""
    from paper_2507_11289_b200.configs import Config
    c = Config("r4", 30, 8, 8, 0, rc=4.0)
    g = _geom(c)
    e, _ = _engine(c, seed=3)
    x = inputs.jitter(oracle.lattice(c.nx, c.ny, c.nz, g.a), g.b, 0.2, 6)
    v = inputs.gaussian_velocities(c.n_atoms, 0.8, 6)
    e.set_state(x, v)
    e.step(1)
    _, _, Fo, eo = oracle.run(x, v, np.zeros_like(x), g.b, c.rc, c.dt, 1)
    _force_close(e.forces(), Fo, tol=1e-10)
    _, en = e.energies()
    assert np.allclose(en[0, :3], eo[0, :3], rtol=1e-10)


def test_get_slice_matches_by_id_readback():
    """dsea_get_slice (one slot at a time, the read-back for states too large to gather
    by id): every slice's atoms, ids and vectors equal the by-id arrays; the slices
    partition the atoms."""
    e, c = _engine("C1")
    e.step(3)
    x, v, f = e.positions(), e.velocities(), e.forces()
    seen = []
    for j in range(c.n_slices):
        s = D.dsea_get_slice(e.ctx, j)
        assert np.array_equal(s["xyz"], x[s["id"]])
        assert np.array_equal(s["v"], v[s["id"]])
        assert np.array_equal(s["f"], f[s["id"]])
        seen.append(s["id"])
    ids = np.sort(np.concatenate(seen))
    assert np.array_equal(ids, np.arange(c.n_atoms))
    with pytest.raises(D.DseaError):
        D.dsea_get_slice(e.ctx, c.n_slices)
