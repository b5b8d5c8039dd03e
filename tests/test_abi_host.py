"""CPU-side tests of the C-ABI library (no GPU needed): the library loads and
exports every symbol include/dsea.h declares; the host-only entry points
(geometry, initial state, stage schedule) agree with the oracle and the paper."""
import os
import re

import numpy as np
import pytest

import oracle
from paper_2507_11289_b200 import CONFIGS
from paper_2507_11289_b200 import dsea as D

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "dsea.h")).read()
    declared = set(re.findall(r"^\s*(?:dsea_status|void|const char \*)\s*(dsea_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 19
    bound = {name for name, _, _ in D.SIGNATURES}
    assert declared == bound, declared ^ bound
    for name in declared:
        assert hasattr(D.lib, name)


def test_library_exports_every_grid_symbol():
    """include/dsea_grid.h (the stencil workload): every declaration is exported by
    libdsea.so and bound, under the same name, by paper_2507_11289_b200.grid."""
    from paper_2507_11289_b200 import grid as G
    hdr = open(os.path.join(ROOT, "include", "dsea_grid.h")).read()
    declared = set(re.findall(r"^\s*(?:dsea_status|void|const char \*)\s*(dsea_grid_\w+)\s*\(", hdr, re.M))
    assert len(declared) == 12
    assert declared == {name for name, _, _ in G.SIGNATURES}
    for name in declared:
        assert hasattr(D.lib, name)


@pytest.mark.parametrize("kw", [dict(nx=10, n_slices=4), dict(r=0.2), dict(r=0.0), dict(ny=2), dict(n_slices=2),
                                dict(rank=2, n_gpus=2), dict(workers_per_gpu=0), dict(mode=1, n_gpus=2),
                                dict(slices_per_stage=13)])
def test_grid_create_rejects_bad_parameters(kw):
    """Parameter validation happens on the host before any device call (DSEA_EINVAL);
    valid parameters on a machine without a GPU give DSEA_ECUDA (no CPU fallback)."""
    from paper_2507_11289_b200 import grid as G
    p = dict(nx=12, ny=4, nz=5, n_slices=12, r=0.1)
    p.update(kw)
    with pytest.raises(D.DseaError) as e:
        G.dsea_grid_create(**p)
    assert e.value.status == D.DSEA_EINVAL


def test_grid_create_without_gpu_is_ecuda():
    import torch
    from paper_2507_11289_b200 import grid as G
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(D.DseaError) as e:
        G.dsea_grid_create(12, 4, 5, 12, 0.1)
    assert e.value.status == D.DSEA_ECUDA


@pytest.mark.parametrize("name", ["C1", "P8", "C2", "C3", "C4", "C5b", "C5f"])
def test_geometry_matches_oracle(name):
    """dsea_geometry_compute (Q3) equals the oracle's geometry bit for bit."""
    c = CONFIGS[name]
    st, g = D.dsea_geometry_compute(c.nx, c.ny, c.nz, c.rho, c.rc, c.n_slices, c.cells_per_slice_x)
    o = oracle.geometry(c.nx, c.ny, c.nz, c.rho, c.rc, c.n_slices, c.cells_per_slice_x)
    assert st == 0 and o.feasible
    assert list(g.b) == list(o.b) and list(g.l) == list(o.l)
    assert list(g.cells) == list(o.cells) and g.n_slices == o.n_slices and g.n_atoms == o.n_atoms
    assert g.w == o.w and g.a == o.a and g.u_shift == o.ushift
    assert g.slot_capacity >= 1.25 * g.n_atoms / g.n_slices and g.slot_capacity % 32 == 0


def test_geometry_rejections():
    # slices thinner than rc (north star: keep O_in = O_out = 1)
    st, _ = D.dsea_geometry_compute(10, 10, 10, 0.8, 2.5, n_slices=8)
    assert st == D.DSEA_EGEOM
    # fewer than 3 cells in y
    st, _ = D.dsea_geometry_compute(20, 2, 5, 0.8, 2.5, n_slices=4)
    assert st == D.DSEA_EGEOM
    st, _ = D.dsea_geometry_compute(20, 5, 5, 0.8, 2.5, n_slices=4, cells_per_slice_x=0)
    assert st == D.DSEA_EINVAL


@pytest.mark.parametrize("name,seed", [("C1", 11289), ("P8", 3), ("C1", 1)])
def test_initial_state_bit_exact_vs_oracle(name, seed):
    """Parity 1 (host, no GPU): dsea_init's FCC lattice (Q10) and velocities
    (Q9) are bit-identical to the oracle's independent generator."""
    c = CONFIGS[name]
    ctx = D.dsea_init(c.nx, c.ny, c.nz, c.rho, c.rc, c.dt, 1.0, seed)
    try:
        x = D.dsea_get_positions(ctx, c.n_atoms)
        v = D.dsea_get_velocities(ctx, c.n_atoms)
        f = D.dsea_get_forces(ctx, c.n_atoms)
    finally:
        D.dsea_destroy(ctx)
    g = oracle.geometry(c.nx, c.ny, c.nz, c.rho, c.rc, c.n_slices, 1)
    assert np.array_equal(x, oracle.lattice(c.nx, c.ny, c.nz, g.a))
    assert np.array_equal(v, oracle.velocities(c.n_atoms, seed, 1.0))
    assert not f.any()


def test_init_rejects_bad_box():
    with pytest.raises(D.DseaError):
        D.dsea_init(0, 5, 5, 0.8, 2.5)
    with pytest.raises(D.DseaError):
        D.dsea_init(5, 5, 5, -0.8, 2.5)
    with pytest.raises(D.DseaError):
        D.dsea_init(5, 5, 5, 0.8, 2.5, dt=0.0)


def _table1():
    rows = []
    for line in open(os.path.join(GOLDEN, "table1.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        rows.append(line.split())
    return rows


def test_schedule_reproduces_table1():
    """Table 1 (§3.3): one worker, one GPU, O_in = O_out = 1, N_S = 6.
    Compare receive, worker and send columns and the derived partial column."""
    ns = 6
    rows = D.dsea_schedule(ns, 1, 0, 1, 1)
    by_stage = {}
    for st, recv, w, proc, binned, send, cyc, t in rows:
        e = by_stage.setdefault(int(st), {"recv": "-", "proc": "-", "send": "-"})
        if recv > 0:
            e["recv"] = str(recv)
        if w >= 0 and proc > 0:
            e["proc"] = str(proc)
        if w >= 0 and send > 0:
            e["send"] = str(send)
    done = set()
    for stage, recv, proc, partial, send in _table1():
        e = by_stage.get(int(stage), {"recv": "-", "proc": "-", "send": "-"})
        assert e["recv"] == recv, (stage, e)
        assert e["proc"] == proc, (stage, e)
        assert e["send"] == send, (stage, e)
        # partial = slices with a contribution that are not yet final
        if proc != "-":
            p = int(proc)
            if send != "-":
                done.add(int(send))
            part = [s for s in (p, p + 1) if 1 <= s <= ns and s not in done]
            assert ",".join(map(str, part)) == partial, (stage, part, partial)
    assert max(by_stage) == ns + 3  # last send in stage N_S + 3


@pytest.mark.parametrize("ns,ng,W,cycles", [(16, 2, 1, 2), (32, 8, 1, 3), (24, 2, 3, 2), (12, 1, 3, 3),
                                           (109, 4, 2, 2)])
def test_ring_schedule_invariants(ns, ng, W, cycles):
    """The generalised schedule: every (slice, timestep) unit is processed exactly
    once over the ring; rank g sends exactly the items rank g+1 receives, in order
    (P:117-120); a super-cycle advances N_w = N_GPU*W timesteps; worker w
    processes slice m in the same stage as worker w-1 processes m+2, right after it
    (workers run sequentially within a stage)."""
    units = set()
    sends, recvs = {}, {}
    for g in range(ng):
        rows = D.dsea_schedule(ns, ng, g, W, cycles)
        sends[g] = [int(r[5]) for r in rows if r[5] > 0 and r[2] == W - 1]
        recvs[g] = [int(r[1]) for r in rows if r[1] > 0]
        proc_stage = {}
        for st, recv, w, proc, binned, send, cyc, t in rows:
            if w >= 0 and proc > 0:
                assert t == cyc * ng * W + g * W + w
                key = (proc, t)
                assert key not in units
                units.add(key)
                proc_stage[(w, cyc, proc)] = st
        for (w, cyc, proc), st in proc_stage.items():
            if w > 0 and (w - 1, cyc, proc + 2) in proc_stage:
                assert st == proc_stage[(w - 1, cyc, proc + 2)]
    assert units == {(j, t) for j in range(1, ns + 1) for t in range(cycles * ng * W)}
    if ng > 1:
        for g in range(ng):
            nxt = (g + 1) % ng
            # items flow in (cycle, slice) order; rank 0's first cycle is resident
            got = recvs[nxt][ns:] if nxt == 0 else recvs[nxt]
            assert sends[g] == got
            assert len(sends[g]) == cycles * ns


def test_eq1_nmax_reported():
    """Eq. (1) as reported by the library: N_S / (2 + 2W)."""
    for ns, W in [(100, 1), (64, 2), (109, 1), (256, 15)]:
        st, g = D.dsea_geometry_compute(4 * ns // 3 + 10, 5, 5, 0.8, 2.5, n_slices=ns, workers_per_gpu=W)
        assert g.n_max == oracle.nmax(ns, W)


def test_thermo_compute_matches_oracle_pressure():
    """dsea_thermo_compute (host-only ABI call; NEXT-1 observables, Q24) against the
    oracle's independent pressure definition and the plain T, u, e formulas."""
    rng = np.random.default_rng(3)
    rec = np.zeros(7, dtype=D._ENERGY_DT)
    rec["step"] = np.arange(7) + 40
    rec["U"] = -5.0 * 1000 + rng.random(7)
    rec["KE"] = 1500.0 + rng.random(7)
    rec["V"] = -900.0 + rng.random(7)
    n, vol = 1000, 1250.0
    t = D.dsea_thermo_compute(rec, n, vol)
    assert np.array_equal(t["step"], rec["step"])
    assert np.allclose(t["p"], oracle.pressure(rec["KE"], rec["V"], n, vol), rtol=1e-14)
    assert np.allclose(t["T"], 2 * rec["KE"] / (3 * n), rtol=1e-15)
    assert np.allclose(t["u"], rec["U"] / n, rtol=1e-15)
    assert np.allclose(t["e"], (rec["U"] + rec["KE"]) / n, rtol=1e-15)
    with pytest.raises(D.DseaError):
        D.dsea_thermo_compute(rec, 0, vol)


def test_xprofile_compute_matches_oracle_pressure():
    """dsea_xprofile_compute: per-slice averages and pressure (slice volume w b_y b_z)
    against the oracle's pressure of the averaged sums; empty slices report zeros."""
    st, g = D.dsea_geometry_compute(20, 10, 5, 0.8, 2.5, n_slices=8)
    assert st == 0
    raw = np.zeros(8, dtype=D._PROFILE_DT)
    raw["samples"] = 10
    raw["n_sum"] = 500.0 * 10
    raw["n_sum"][3] = 0.0
    raw["U_sum"] = -2900.0 * 10
    raw["V_sum"] = -480.0 * 10
    raw["KE_sum"] = 360.0 * 10
    raw["U_sum"][3] = raw["V_sum"][3] = raw["KE_sum"][3] = 0.0
    x = D.dsea_xprofile_compute(raw, g)
    vol = g.w * g.b[1] * g.b[2]
    ok = np.arange(8) != 3
    assert np.allclose(x["p"], oracle.pressure(raw["KE_sum"] / 10, raw["V_sum"] / 10, raw["n_sum"] / 10, vol),
                       rtol=1e-14)
    assert np.allclose(x["x"], (np.arange(8) + 0.5) * g.w)
    assert np.allclose(x["u"][ok], -2900.0 / 500.0) and x["u"][3] == 0.0 and x["T"][3] == 0.0
    assert np.allclose(x["rho"], raw["n_sum"] / 10 / vol)


def test_next3_billion_atom_geometry_fits_four_b200s():
    """NEXT-3 (10^9 molecules, the N_i = 630 cube): the paper's slicing rule
    gives 430 slices of 2.33e6 atoms; geometry equals the oracle's; the input buffer of
    N_S slots (76 B of carried state per slot atom, ~95 GB) plus slot pools fits one
    180 GB B200 -- measured 101-102 GB per GPU (profiles/r02/next3_1e9/)."""
    st, g = D.dsea_geometry_compute(630, 630, 630, 0.8, 2.5)
    o = oracle.geometry(630, 630, 630, 0.8, 2.5, 0, 1)
    assert st == 0 and o.feasible
    assert g.n_atoms == 1_000_188_000 == o.n_atoms
    assert g.n_slices == o.n_slices == 430
    assert g.slot_capacity >= 1.25 * g.n_atoms / g.n_slices and g.slot_capacity % 32 == 0
    input_buffer = g.n_slices * g.slot_capacity * 76
    assert 90e9 < input_buffer < 100e9
    # Eq. (1): N_max = N_S / (2 + 2W) = 107 GPUs at W = 1 -- a ring of 4 is far from the plateau
    assert g.n_max == 430 // 4
