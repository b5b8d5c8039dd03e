"""GPU parity for NEXT-1: the per-slice NVT thermostat (§4.1,
reading Q23), x-resolved profiles and the virial pressure (Q24),
through the C ABI, against the CPU oracle (oracle.run_ex / oracle.pressure) on the
same seeded inputs.  Tolerances as for NVE (Q13/Q14).  -m gpu."""
import numpy as np
import pytest

import oracle
from paper_2507_11289_b200 import CONFIGS
from paper_2507_11289_b200 import dsea as D
from tests import inputs

pytestmark = pytest.mark.gpu


def _engine(cfg, **kw):
    c = CONFIGS[cfg] if isinstance(cfg, str) else cfg
    e = D.Engine(D.Box(c.nx, c.ny, c.nz, c.rho, c.rc, c.dt, c.T0, c.seed))
    kw.setdefault("n_slices", c.n_slices)
    kw.setdefault("cells_per_slice_x", c.cells_per_slice_x)
    e.slice(**kw)
    return e, c


def _geom(c):
    return oracle.geometry(c.nx, c.ny, c.nz, c.rho, c.rc, c.n_slices, c.cells_per_slice_x)


def _min_image(d, b):
    d = d.copy()
    d[:, 1:] -= b[1:] * np.round(d[:, 1:] / b[1:])
    return d


def _prof_sums(e):
    p = e.raw_profiles()
    return np.stack([p[k] for k in ("n_sum", "U_sum", "V_sum", "KE_sum")], 1), p["samples"]


@pytest.mark.parametrize("cfg,T", [("C1", 1.5), ("P8", 0.7)])
def test_nvt_matches_oracle(cfg, T):
    """10 NVT steps from a jittered state at T0 = 1.0: positions and velocities within
    1e-8 (Q14), energies, per-slice sums of {n, U, V, KE} and the pressure series
    against the oracle."""
    e, c = _engine(cfg)
    g = _geom(c)
    x = inputs.jitter(oracle.lattice(c.nx, c.ny, c.nz, g.a), g.b, 0.2, 5)
    v = inputs.gaussian_velocities(c.n_atoms, 1.0, 5)
    e.set_state(x, v)
    e.set_thermostat(T)
    e.step(10)
    xo, vo, Fo, eo, rec = oracle.run_ex(x, v, np.zeros_like(x), g.b, c.rc, c.dt, 10, g, T_target=T)
    assert np.max(np.abs(_min_image(e.positions() - xo, g.b))) < 1e-8
    assert np.max(np.abs(e.velocities() - vo)) < 1e-8
    _, en = e.energies()
    assert np.allclose(en[:, :3], eo[:, :3], rtol=1e-9, atol=1e-9)
    sums, samples = _prof_sums(e)
    assert np.all(samples == 10)
    ref = rec.sum(0)
    assert np.array_equal(sums[:, 0], ref[:, 0])                       # atom counts exact
    assert np.allclose(sums[:, 1:], ref[:, 1:], rtol=1e-9, atol=1e-9)
    vol = g.b.prod()
    p_ref = oracle.pressure(eo[:, 1], eo[:, 2], c.n_atoms, vol)
    assert np.allclose(e.pressure(), p_ref, rtol=1e-10)


def test_nvt_every_slice_at_target_on_gpu():
    """After each NVT step the velocities of every slice -- grouped by the GPU's own
    slice membership at the start of the step -- have sum v.v / (3 n_j) = T_target."""
    e, c = _engine("C1")
    e.set_thermostat(1.25)
    for _ in range(3):
        _, sl = e.cells()
        e.step(1)
        v = e.velocities()
        for j in range(c.n_slices):
            m = sl == j
            assert abs((v[m] ** 2).sum() / (3 * m.sum()) - 1.25) < 1e-12


@pytest.mark.parametrize("W,B", [(1, 1), (2, 1), (2, 3)])
def test_nvt_staged_bitwise_equals_fused(W, B):
    """The thermostat is per (slice, timestep): the stage schedule and the fused pass
    give bitwise equal states, energies and per-slice sums."""
    ref, _ = _engine("P8")
    ref.set_thermostat(1.5)
    ref.step(7)
    e, _ = _engine("P8", workers_per_gpu=W, mode=D.DSEA_MODE_STAGED, slices_per_stage=B)
    e.set_thermostat(1.5)
    e.step(7)
    assert np.array_equal(e.positions(), ref.positions())
    assert np.array_equal(e.velocities(), ref.velocities())
    assert np.array_equal(e.energies()[1], ref.energies()[1])
    assert np.array_equal(_prof_sums(e)[0], _prof_sums(ref)[0])


def test_nvt_long_run_mean_temperature():
    """SPEC S:322 anchored on P:322 (T = 1.5): C1 from T0 = 1.0, mean kinetic
    temperature over steps 500-1500 within 1 % of 1.5; turning the thermostat off
    afterwards returns to NVE (energy drift < 1e-4 over the next 500 steps)."""
    e, c = _engine("C1")
    e.set_thermostat(1.5)
    e.step(1500)
    _, en = e.energies()
    T = 2 * en[500:, 1] / (3 * c.n_atoms)
    assert abs(T.mean() / 1.5 - 1) < 0.01, T.mean()
    e.set_thermostat(None)
    e.step(500)
    E = e.energies()[1][1500:, 3]
    assert np.max(np.abs(E - E[0])) / abs(E[0]) < 1e-4


def test_nve_profiles_and_pressure_match_oracle():
    """NVE: per-slice sums over 6 steps and the pressure series against the oracle;
    slice sums add up to the domain totals every step."""
    e, c = _engine("P8")
    g = _geom(c)
    x0, v0 = e.positions(), e.velocities()
    e.step(6)
    _, _, _, eo, rec = oracle.run_ex(x0, v0, np.zeros_like(x0), g.b, c.rc, c.dt, 6, g)
    sums, _ = _prof_sums(e)
    ref = rec.sum(0)
    assert np.array_equal(sums[:, 0], ref[:, 0])
    assert np.allclose(sums[:, 1:], ref[:, 1:], rtol=1e-9, atol=1e-9)
    _, en = e.energies()
    assert np.allclose(sums[:, 1].sum(), en[:, 0].sum(), rtol=1e-12)
    assert np.allclose(sums[:, 2].sum(), en[:, 2].sum(), rtol=1e-12)
    prof = e.profiles()
    assert np.allclose(prof["rho"].mean(), c.n_atoms / g.b.prod(), rtol=1e-12)
    assert np.allclose(e.pressure(), oracle.pressure(eo[:, 1], eo[:, 2], c.n_atoms, g.b.prod()),
                       rtol=1e-10)
    e.reset_profiles()
    assert np.all(e.raw_profiles()["samples"] == 0)


def test_thermostat_error_paths():
    c = CONFIGS["C1"]
    ctx = D.dsea_init(c.nx, c.ny, c.nz, c.rho, c.rc)
    with pytest.raises(D.DseaError) as ei:          # before dsea_slice
        D.dsea_set_thermostat(ctx, 1.0)
    assert ei.value.status == D.DSEA_ESTATE
    D.dsea_destroy(ctx)
    e, _ = _engine("C1")
    for bad in (-1.0, float("nan"), float("inf")):
        with pytest.raises(D.DseaError) as ei:
            e.set_thermostat(bad)
        assert ei.value.status == D.DSEA_EINVAL
    with pytest.raises(D.DseaError) as ei:
        D.dsea_get_profiles(e.ctx, c.n_slices + 1)
    assert ei.value.status == D.DSEA_EINVAL
