"""Pins for the CPU oracle (oracle/oracle.c) against what the paper and the
mathematics fix -- never against the oracle itself.

Each test names the passage (P:n = PAPER.md line) or the closed form it pins and
the plausible oracle mistake it would catch.  CPU only (-m "not gpu")."""
import os

import numpy as np
import pytest

import oracle
from tests import inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
RC = 2.5


def _golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


BIG = np.array([40.0, 40.0, 40.0])  # box so large that no image or wall matters


def _pair(r, axis=0):
    xyz = np.full((2, 3), 20.0)
    xyz[1, axis] += r
    return xyz


# --------------------------------------------------------------------------- generator
def test_splitmix64_published_vector():
    """Q9 generator: SplitMix64 reference outputs for state 0 (golden/splitmix64.txt).
    Catches a wrong constant, shift or increment."""
    rows = _golden("splitmix64.txt")
    seed, count = int(rows[0][0]), int(rows[0][1])
    want = [int(r[0], 16) for r in rows[1:1 + count]]
    assert oracle.splitmix64(seed, count) == want


def test_box_muller_is_standard_normal():
    """Q9: normals are N(0,1).  Moments and the 1-sigma mass (0.6827) of 2e5 draws.
    Catches a sin/cos mix-up with wrong scale, a missing sqrt or -2 factor."""
    z = oracle.normals(7, 200000)
    assert abs(z.mean()) < 0.01
    assert abs(z.var() - 1.0) < 0.015
    assert abs(np.mean(np.abs(z) < 1.0) - 0.682689) < 0.005
    assert abs(np.mean(z ** 4) - 3.0) < 0.08


def test_velocities_zero_momentum_and_exact_temperature():
    """P:225 'initialized according to the temperature' + Q9: zero total momentum,
    instantaneous T = sum v^2 / (3N) equal to T0 (k_B = m = 1, Q11)."""
    for n, T0 in [(4000, 1.0), (500, 1.5)]:
        v = oracle.velocities(n, 11289, T0)
        assert np.all(np.abs(v.sum(axis=0)) < 1e-10)
        assert abs((v ** 2).sum() / (3 * n) - T0) < 1e-12 * T0


# --------------------------------------------------------------------------- geometry
def test_geometry_paper_formulas():
    """b = N_i (4/rho)^(1/3), N = 4 N_i^3, N_xyz = floor(b/rc), l = b/N_xyz.
    Worked values: N_i=2, rho=0.5 -> a=2, b=4, N=32; N_i=5 -> b=10, N_xyz=4, l=2.5."""
    g = oracle.geometry(2, 2, 2, 0.5, RC, 1, 1)
    assert g.a == 2.0 and np.all(g.b == 4.0) and g.n_atoms == 32
    g = oracle.geometry(5, 5, 5, 0.5, RC, 0, 1)
    assert np.all(g.b == 10.0) and g.n_atoms == 500
    assert g.n_slices == 4 and list(g.cells) == [4, 4, 4] and np.all(g.l == 2.5)
    assert g.feasible  # l = rc accepted (Q18)
    # C4: 160^3 FCC cells at rho 0.8, paper rule -> 109 slices
    g = oracle.geometry(160, 160, 160, 0.8, RC, 0, 1)
    assert g.n_slices == 109 and g.n_atoms == 16384000 and list(g.cells) == [109, 109, 109]
    # too few cells in y -> infeasible
    assert not oracle.geometry(20, 2, 5, 0.8, RC, 8, 1).feasible
    # slices thinner than rc -> infeasible
    assert not oracle.geometry(10, 10, 10, 0.8, RC, 8, 1).feasible


def test_lattice_is_fcc():
    """FCC with four molecules per cell: every site has its 12 nearest
    neighbours at a/sqrt(2) (minimum image in y/z), none closer; offset a/4 (Q10)."""
    nx, ny, nz = 4, 4, 4
    g = oracle.geometry(nx, ny, nz, 0.8, RC, 1, 1)
    x = oracle.lattice(nx, ny, nz, g.a)
    assert x.shape == (256, 3)
    assert np.allclose(x[0], [0.25 * g.a] * 3, rtol=0, atol=0)
    d = x[:, None, :] - x[None, :, :]
    d[..., 1:] -= g.b[1:] * np.round(d[..., 1:] / g.b[1:])
    r = np.sqrt((d ** 2).sum(-1))
    np.fill_diagonal(r, np.inf)
    nn = g.a / np.sqrt(2.0)
    assert np.isclose(r.min(), nn, rtol=1e-12)
    counts = (np.abs(r - nn) < 1e-9).sum(1)
    interior = (x[:, 0] > 0.6 * g.a) & (x[:, 0] < g.b[0] - 0.6 * g.a)
    assert np.all(counts[interior] == 12)


# --------------------------------------------------------------------------- pair law
def test_pair_energy_closed_forms():
    """Truncated-and-shifted LJ 12-6 with sigma = eps = 1 (Q6).
    Two atoms = two ordered pairs with the /2 of P:265, so U = phi(r):
    phi(1) = 4 U_shift (zero crossing at sigma), phi(2^(1/6)) = -1 + 4 U_shift
    (well depth eps at the minimum), phi(rc) = 0 (shift), beyond rc nothing."""
    us = (1 / RC) ** 6 - (1 / RC) ** 12
    assert abs(us - 0.004079222784) < 1e-15
    _, U, _ = oracle.forces(_pair(1.0), BIG, RC)
    assert abs(U - 4 * us) < 1e-14
    _, U, _ = oracle.forces(_pair(2 ** (1 / 6)), BIG, RC)
    assert abs(U - (-1 + 4 * us)) < 1e-14
    _, U, _ = oracle.forces(_pair(RC), BIG, RC)
    assert abs(U) < 1e-15
    F, U, V = oracle.forces(_pair(RC * (1 + 1e-12)), BIG, RC)
    assert U == 0.0 and V == 0.0 and np.all(F == 0.0)


def test_force_is_minus_energy_gradient():
    """F_i = -dU/dr_i by central finite differences of the oracle's own U, on a
    3-atom cluster and a random 24-atom periodic box.  Catches a wrong factor
    (24 vs 4, /r^2), a wrong sign of r_ij, or a dropped term in F_abs."""
    rng_xyz = [
        (np.array([[20.0, 20.0, 20.0], [21.1, 20.0, 20.0], [20.0, 21.2, 20.0]]), BIG),
        (inputs.random_points(24, [7.6, 7.7, 7.8], seed=3, min_sep=0.9), np.array([7.6, 7.7, 7.8])),
    ]
    h = 1e-6
    for xyz, box in rng_xyz:
        F, _, _ = oracle.forces(xyz, box, RC)
        for i in range(min(len(xyz), 8)):
            for d in range(3):
                xp = xyz.copy(); xp[i, d] += h
                xm = xyz.copy(); xm[i, d] -= h
                up = oracle.forces(xp, box, RC)[1]
                um = oracle.forces(xm, box, RC)[1]
                num = -(up - um) / (2 * h)
                assert abs(num - F[i, d]) < 2e-6 * max(1.0, abs(F[i, d])), (i, d, num, F[i, d])


def test_force_zero_at_minimum_and_jump_at_cutoff():
    """LJ minimum at 2^(1/6) sigma: F = 0 (north star pin).  At r = rc the pair is
    included (r^2 <= rc^2): |F| = 24(2 rc^-13 - rc^-7), attractive."""
    F, _, _ = oracle.forces(_pair(2 ** (1 / 6)), BIG, RC)
    assert np.all(np.abs(F) < 1e-13)
    F, _, _ = oracle.forces(_pair(RC), BIG, RC)
    mag = 24 * (2 * RC ** -13 - RC ** -7)
    assert abs(abs(F[0, 0]) - abs(mag)) < 1e-15
    assert F[0, 0] > 0  # atom 0 is left of atom 1: attraction pulls it to +x
    F, _, _ = oracle.forces(_pair(1.0), BIG, RC)
    assert abs(F[0, 0] + 24.0) < 1e-12 and abs(F[1, 0] - 24.0) < 1e-12  # repulsive, |F| = 24


def test_virial_identity():
    """Algorithm 1's V (per ordered pair (2 r^-12 - r^-6)/2) satisfies
    sum_i r_i . F_i = 24 V for an isolated cluster (no images).  Catches a wrong
    V factor or sign; single pair at r = 1 gives V = 1."""
    _, _, V = oracle.forces(_pair(1.0), BIG, RC)
    assert abs(V - 1.0) < 1e-14
    xyz = inputs.random_points(30, [6.0, 6.0, 6.0], seed=5, min_sep=0.9) + 17.0
    F, U, V = oracle.forces(xyz, BIG, RC)
    assert abs((xyz * F).sum() - 24.0 * V) < 1e-10 * max(1.0, abs(24 * V))


def test_newton_third_law():
    """Sum of F_new is zero: ordered pairs are antisymmetric and the walls exert no
    force (north star pin).  Random periodic box + the C1 lattice."""
    box = np.array([9.0, 8.0, 7.7])
    xyz = inputs.random_points(60, box, seed=11, min_sep=0.9)
    F, _, _ = oracle.forces(xyz, box, RC)
    frms = np.sqrt((F ** 2).mean())
    assert np.all(np.abs(F.sum(0)) < 1e-12 * len(xyz) * frms)


def test_minimum_image_equals_explicit_image_sum():
    """Q1: minimum image in y/z equals the explicit sum over the 3x3 images
    (n_y, n_z in {-1,0,1}) because b_y, b_z >= 2 rc.  The image sum is computed by
    the oracle itself on the tiled system in a box three times larger, so only
    the periodic bookkeeping differs.  Catches rint/floor or axis mistakes."""
    box = np.array([8.0, 7.6, 8.3])
    xyz = inputs.random_points(40, box, seed=21, min_sep=0.9)
    F, U, _ = oracle.forces(xyz, box, RC, per_atom=False)
    tiles = []
    for ny in (0, -1, 1):
        for nz in (0, -1, 1):
            tiles.append(xyz + np.array([0.0, (ny + 1) * box[1], (nz + 1) * box[2]]))
    big = np.concatenate(tiles)
    big_box = np.array([box[0], 3 * box[1], 3 * box[2]])
    Fb, _, _, Ub, _ = oracle.forces(big, big_box, RC, per_atom=True)
    n = len(xyz)
    assert np.allclose(Fb[:n], F, rtol=1e-12, atol=1e-12)
    assert abs(Ub[:n].sum() - U) < 1e-11 * abs(U)


def test_fcc_shell_sums():
    """Interior atom of the perfect lattice: neighbour count and per-atom energy
    equal the closed-form FCC shell sums (golden/fcc_shells.txt): 54 neighbours at
    rho=0.8, rc=2.5 and U_i = -5.92419044138561 (SURVEY §8(c) pin 3); F_i = 0."""
    shells = [(int(a), int(b)) for a, b in _golden("fcc_shells.txt")]
    for rho, rc, want_n, want_u in [(0.8, 2.5, 54, -5.92419044138561), (0.5, 2.5, 42, -2.68810901428186),
                                    (0.8, 4.0, 200, -6.55726869576326)]:
        nx = 12 if rc < 3 else 14
        g = oracle.geometry(nx, 8 if rc < 3 else 9, 8 if rc < 3 else 9, rho, rc, 1, 1)
        x = oracle.lattice(nx, 8 if rc < 3 else 9, 8 if rc < 3 else 9, g.a)
        F, _, _, Ui, _ = oracle.forces(x, g.b, rc, per_atom=True)
        center = np.argmin(np.abs(x[:, 0] - g.b[0] / 2) + np.abs(x[:, 1] - g.b[1] / 2) + np.abs(x[:, 2] - g.b[2] / 2))
        assert x[center, 0] > rc + 1 and x[center, 0] < g.b[0] - rc - 1
        us = (1 / rc) ** 6 - (1 / rc) ** 12
        n_in, u = 0, 0.0
        for k, m in shells:
            r2 = k * g.a * g.a / 2
            if r2 <= rc * rc:
                n_in += m
                u += m * 2 * (r2 ** -6 - r2 ** -3 + us)
        assert n_in == want_n
        assert abs(u - want_u) < 1e-12 * abs(want_u)
        assert abs(Ui[center] - u) < 1e-12 * abs(u)
        assert np.all(np.abs(F[center]) < 1e-12)


# --------------------------------------------------------------------------- integrator
def _small_state(seed=11289, nx=5, T0=1.0):
    g = oracle.geometry(nx, 5, 5, 0.8, RC, 0, 1)
    x = oracle.lattice(nx, 5, 5, g.a)
    v = oracle.velocities(len(x), seed, T0)
    return g, x, v


def test_free_flight_and_first_kick():
    """Algorithm 1 with no neighbours (one atom): r_{n+1} = r_n + v dt exactly in
    exact arithmetic and v constant; KE recorded after the kick."""
    xyz = np.array([[20.0, 20.0, 20.0]])
    v = np.array([[0.3, -0.2, 0.1]])
    x1, v1, F1, e = oracle.run(xyz, v, np.zeros((1, 3)), BIG, RC, 0.002, 10)
    assert np.allclose(x1, xyz + 10 * 0.002 * v, rtol=0, atol=1e-13)
    assert np.all(v1 == v)
    assert np.allclose(e[:, 1], 0.5 * (v ** 2).sum())


def test_two_body_kick_and_drift_first_step():
    """One Algorithm 1 iteration from F_new = F_old = 0 (Q7) for a pair at r = 1:
    F_new = -/+24 x; v += (F_new + 0) dt/2; r += v dt + F_new dt^2/2."""
    dt = 0.002
    xyz = _pair(1.0)
    v = np.zeros((2, 3))
    x1, v1, F1, e = oracle.run(xyz, v, np.zeros((2, 3)), BIG, RC, dt, 1)
    assert abs(v1[0, 0] - (-24.0 * dt / 2)) < 1e-15
    assert abs(x1[0, 0] - (20.0 + v1[0, 0] * dt + (-24.0) * 0.5 * dt * dt)) < 1e-14
    assert abs(e[0, 0] - 4 * ((1 / RC) ** 6 - (1 / RC) ** 12)) < 1e-14


@pytest.mark.slow
def test_nve_energy_conservation_and_dt2_scaling():
    """North star: |dE/E| < 1e-4 over 1000 NVE steps at dt = 0.0018 (Q8, Q19),
    and the VV error amplitude scales as dt^2: doubling dt multiplies max |dE| by ~4
    (SURVEY §8(c) pin 6 measured 4.005).  Catches a dropped dt^2/2 term or a
    wrong kick (first-order integrators scale as dt)."""
    g, x, v = _small_state()
    _, _, _, e1 = oracle.run(x, v, np.zeros_like(x), g.b, RC, 0.0018, 1000)
    E = e1[:, 3]
    drift1 = np.max(np.abs(E - E[0])) / abs(E[0])
    assert drift1 < 1e-4
    _, _, _, e2 = oracle.run(x, v, np.zeros_like(x), g.b, RC, 0.0036, 500)
    E2 = e2[:, 3]
    drift2 = np.max(np.abs(E2 - E2[0])) / abs(E2[0])
    ratio = drift2 / drift1
    assert 3.0 < ratio < 5.5, ratio


def test_time_reversibility_through_walls():
    """Velocity Verlet is time reversible; with the mirror read as Q2 (fold
    r, negate v_x and F_new,x) the map stays reversible through wall hits.  Forward
    100 steps with edge atoms driven into both walls, reverse, and return to r0
    within 1e-10 (SURVEY §8(c) pin 5).  Catches a mirror that forgets F_x or an
    asymmetric kick."""
    dt = 0.0018
    g = oracle.geometry(6, 4, 4, 0.8, RC, 1, 1)
    x0 = oracle.lattice(6, 4, 4, g.a)
    v0 = oracle.velocities(len(x0), 5, 1.0)
    left = x0[:, 0] < 0.5 * g.a
    right = x0[:, 0] > g.b[0] - 0.5 * g.a
    v0[left, 0] = -8.0
    v0[right, 0] = 8.0
    n = 100
    xn, vprev, Fprev, _ = oracle.run(x0, v0, np.zeros_like(x0), g.b, RC, dt, n)
    # map Algorithm 1's loop state (r_n, v_{n-1}, F_{n-1}) to standard VV (r_n, v_n)
    Fn, _, _ = oracle.forces(xn, g.b, RC)
    vn = vprev + (Fprev + Fn) * 0.5 * dt
    # re-enter with the Q7 convention: F_new = 0, v_entry = -v_n - F_n dt/2
    x_back, _, _, _ = oracle.run(xn, -vn - Fn * 0.5 * dt, np.zeros_like(x0), g.b, RC, dt, n)
    d = x_back - x0
    d[:, 1:] -= g.b[1:] * np.round(d[:, 1:] / g.b[1:])
    assert np.max(np.abs(d)) < 1e-10
    # sanity: the walls were hit (positions folded at least once)
    assert np.any(np.abs(xn[left | right, 0] - x0[left | right, 0]) > 0.4)


def test_thread_count_does_not_change_results():
    """The OpenMP split over i sums per-atom partials in id order: bitwise equal
    results for 1 and N threads (needed to time the oracle on all cores)."""
    g, x, v = _small_state()
    a = oracle.run(x, v, np.zeros_like(x), g.b, RC, 0.0018, 3, nthreads=1)
    b = oracle.run(x, v, np.zeros_like(x), g.b, RC, 0.0018, 3, nthreads=4)
    for p, q in zip(a, b):
        assert np.array_equal(p, q)


# --------------------------------------------------------------------------- binning
def test_binning_closed_forms():
    """cell = clamp(floor(r/l), 0, n-1) with IEEE division (Q4), slice =
    cell_x / c.  Boundaries exactly on a cell edge go up; b itself clamps down."""
    l = np.array([2.5, 2.6, 2.7])
    cells = np.array([8, 4, 4], dtype=np.int32)
    xyz = np.array([[0.0, 0.0, 0.0], [2.5, 2.6, 2.7], [2.4999999, 10.4, 10.8], [20.0, 5.2, 1.0],
                    [-1e-300, 10.39, 5.4]])
    cx, sl = oracle.bin_atoms(xyz, l, cells, c=2)
    assert cx.tolist() == [[0, 0, 0], [1, 1, 1], [0, 3, 3], [7, 2, 0], [0, 3, 2]]
    assert sl.tolist() == [0, 0, 0, 3, 0]


def test_eq1_nmax():
    """Eq. (1): N_max = N_S / (2 + N_wGPU (O_in + O_out)), floor (Q17);
    N_S/4 for one worker."""
    assert oracle.nmax(100, 1) == 25
    assert oracle.nmax(10, 1, 0, 0) == 5
    assert oracle.nmax(64, 2) == 10
    assert oracle.nmax(109, 1) == 27


# --------------------------------------------------------------------------- NVT (NEXT-1)
def _nvt_state(seed=3, T0=1.0):
    """N = 500 (5^3 FCC cells) at rho = 0.5, the SPEC's thermostat system,
    jittered, with Gaussian velocities at T0."""
    g = oracle.geometry(5, 5, 5, 0.5, RC)
    x = inputs.jitter(oracle.lattice(5, 5, 5, g.a), g.b, 0.2, seed)
    v = inputs.gaussian_velocities(len(x), T0, seed)
    return g, x, v


def test_nvt_every_slice_at_target_after_scaling():
    """P:314-316 (md_thermo_a/b compute the scale factor; md_v3b scales), reading Q23:
    after one step every slice's kinetic temperature sum v.v / (3 n_j) -- recomputed
    here from the returned velocities, grouped by the binning of the INPUT positions --
    equals T_target.  Catches lambda without the sqrt, a KE factor slip, global instead
    of per-slice scaling, or membership taken after the drift."""
    g, x, v = _nvt_state()
    _, sl = oracle.bin_atoms(x, g.l, g.cells, 1)
    assert len(np.unique(sl)) == g.n_slices
    _, v1, _, e, rec = oracle.run_ex(x, v, np.zeros_like(x), g.b, RC, 0.0018, 1, g, T_target=1.5)
    for j in range(g.n_slices):
        m = sl == j
        Tj = (v1[m] ** 2).sum() / (3 * m.sum())
        assert abs(Tj - 1.5) < 1e-12, (j, Tj)
    # the recorded KE is the post-kick, pre-scale value: not at T_target
    assert abs(2 * e[0, 1] / (3 * len(x)) - 1.5) > 0.05


def test_nvt_off_equals_nve_and_slice_records_sum_to_totals():
    """run_ex without a thermostat is Algorithm 1 exactly (bitwise equal to run), and
    the per-slice records {n, U, V, KE} sum to the domain totals every step (x-resolved
    results)."""
    g, x, v = _nvt_state(seed=4)
    a = oracle.run(x, v, np.zeros_like(x), g.b, RC, 0.0018, 5)
    b = oracle.run_ex(x, v, np.zeros_like(x), g.b, RC, 0.0018, 5, g)
    for p, q in zip(a, b[:4]):
        assert np.array_equal(p, q)
    rec, e = b[4], b[3]
    assert np.all(rec[:, :, 0].sum(1) == len(x))
    assert np.allclose(rec[:, :, 1].sum(1), e[:, 0], rtol=1e-12)
    assert np.allclose(rec[:, :, 2].sum(1), e[:, 2], rtol=1e-12)
    assert np.allclose(rec[:, :, 3].sum(1), e[:, 1], rtol=1e-12)


def test_nvt_long_run_mean_temperature():
    """SPEC S:322 / S:492 anchored on P:322 ("temperature of k_B T / eps = 1.5"): from
    the rho = 0.5 lattice with velocities at T0 = 1.0, the time-averaged kinetic
    temperature over steps 500-1500 is within 1 % of T_target = 1.5, while the NVE run
    from the same start is not (so the thermostat, not the start, sets it)."""
    g = oracle.geometry(5, 5, 5, 0.5, RC)
    x = oracle.lattice(5, 5, 5, g.a)
    v = oracle.velocities(len(x), 7, 1.0)
    *_, e_nvt, _ = oracle.run_ex(x, v, np.zeros_like(x), g.b, RC, 0.0018, 1500, g, T_target=1.5)
    T = 2 * e_nvt[500:, 1] / (3 * len(x))
    assert abs(T.mean() / 1.5 - 1) < 0.01, T.mean()
    _, _, _, e_nve = oracle.run(x, v, np.zeros_like(x), g.b, RC, 0.0018, 1500)
    T0 = 2 * e_nve[500:, 1] / (3 * len(x))
    assert abs(T0.mean() / 1.5 - 1) > 0.05


def test_configurational_pressure_is_minus_dU_dVol():
    """Pressure from Algorithm 1's virial accumulator: for a static
    configuration p = -dU/dVol under homogeneous scaling of positions and box (y/z
    periodic, x walls: U depends only on pair distances), by central differences of
    the oracle's U alone.  Pins oracle.pressure's 24 V / (3 Vol) (a wrong factor 8 vs
    24, or V vs 2V, fails by >= 2x)."""
    box = np.array([9.0, 8.0, 7.7])
    x = inputs.random_points(60, box, seed=12, min_sep=0.95)
    _, U, V = oracle.forces(x, box, RC)
    vol = box.prod()
    h = 1e-6
    up = oracle.forces(x * (1 + h), box * (1 + h), RC)[1]
    um = oracle.forces(x * (1 - h), box * (1 - h), RC)[1]
    p_fd = -((up - um) / (2 * h)) / (3 * vol)
    p = oracle.pressure(0.0, V, len(x), vol)
    assert abs(p - p_fd) < 1e-6 * max(1.0, abs(p_fd)), (p, p_fd)
    # ideal-gas limit: no pair within rc -> p = rho T
    assert abs(oracle.pressure(3.0, 0.0, 10, 5.0) - (10 / 5.0) * (2 * 3.0 / 30)) < 1e-15


# --------------------------------------------------------------------------- worked examples
def _three_atom_examples():
    ex, cur = [], None
    for row in _golden("three_atom.txt"):
        if row[0] == "example":
            cur = {"name": row[1], "F": np.zeros((3, 3))}
            ex.append(cur)
        elif row[0] == "pos":
            cur["pos"] = np.array([float(v) for v in row[1:]]).reshape(3, 3)
        elif row[0] in ("F0", "F1", "F2"):
            cur["F"][int(row[0][1])] = [float(v) for v in row[1:]]
        else:
            cur[row[0]] = float(row[1])
    return ex


def _exact_three_body(pos, rc):
    """Exact rational arithmetic of the textbook LJ cluster (Fractions of the fp64
    inputs): U = sum_{i<j} 4 (s^6 - s^3 + U_shift) with s = 1/r^2, forces from the
    analytic gradient dU/d(r^2) = 4 (-6 s^7 + 3 s^4), i.e. F_i = -sum_j 2 r_ij dU/d(r^2).
    Only even powers of r occur, so every value is rational and exact."""
    from fractions import Fraction as Fr
    P = [[Fr(v) for v in p] for p in pos]
    rc2 = Fr(rc) ** 2
    us = (1 / rc2) ** 3 - (1 / rc2) ** 6
    F = [[Fr(0)] * 3 for _ in range(3)]
    U = Fr(0)
    V = Fr(0)
    for i in range(3):
        for j in range(i + 1, 3):
            d = [P[i][k] - P[j][k] for k in range(3)]
            r2 = sum(x * x for x in d)
            if r2 > rc2:
                continue
            s = 1 / r2
            U += 4 * (s ** 6 - s ** 3 + us)
            V += 2 * s ** 6 - s ** 3
            dudr2 = 4 * (-6 * s ** 7 + 3 * s ** 4)
            for k in range(3):
                F[i][k] -= 2 * d[k] * dudr2
                F[j][k] += 2 * d[k] * dudr2
    return np.array([[float(x) for x in f] for f in F]), float(U), float(V)


@pytest.mark.parametrize("ex", _three_atom_examples(), ids=lambda e: e["name"])
def test_three_atom_worked_examples(ex):
    """SURVEY §8(c) pin 2 (north star: 'two- and three-atom worked examples'):
    collinear, L-shape and generic triples, golden values to 1e-14 relative.  The
    golden numbers are first checked against exact rational arithmetic of the
    textbook potential's gradient (so a typo in the file fails too), then the oracle
    against the golden numbers.  Catches a dropped pair, a wrong r_ij sign or index,
    a transposed component, the /2 of P:265/P:267 or a missing U_shift."""
    Fx, Ux, Vx = _exact_three_body(ex["pos"], RC)
    scale = max(1.0, np.abs(ex["F"]).max())
    assert np.abs(Fx - ex["F"]).max() <= 1e-14 * scale
    assert abs(Ux - ex["U"]) <= 1e-14 * abs(ex["U"])
    assert abs(Vx - ex["V"]) <= 1e-14 * max(1.0, abs(ex["V"]))
    F, U, V = oracle.forces(ex["pos"], BIG, RC)
    assert np.abs(F - ex["F"]).max() <= 1e-14 * scale
    assert abs(U - ex["U"]) <= 1e-14 * abs(ex["U"])
    assert abs(V - ex["V"]) <= 1e-14 * max(1.0, abs(ex["V"]))


def test_forces_subset_equals_full_rows():
    """oracle_forces_subset (the sampled reference of the full-size C2/C4 parity) on a
    shuffled index set with repeats equals the matching rows of the full all-pairs
    oracle_forces (pinned above), forces and per-atom U bit for bit, on a random box
    with walls and y/z images.  Catches an idx[k] <-> k mix-up, a wrong output row,
    a missing minimum image or a dropped self-exclusion."""
    box = np.array([11.0, 8.1, 7.9])
    xyz = inputs.random_points(180, box, seed=31, min_sep=0.88)
    F, U, V, Ui, Vi = oracle.forces(xyz, box, RC, per_atom=True)
    rng = np.random.default_rng(4)
    idx = np.concatenate([rng.permutation(180)[:70], [5, 5, 179, 0]])
    Fs, Us = oracle.forces_subset(xyz, box, RC, idx)
    assert np.array_equal(Fs, F[idx])
    assert np.array_equal(Us, Ui[idx])
    assert Fs.shape == (len(idx), 3)
