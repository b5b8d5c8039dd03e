"""Thin ctypes binding of libdsea.so (include/dsea.h).  Argument marshalling only:
every step of the hot path runs in the library's sm_100a kernels.  There is no
CPU fallback -- if the library cannot be loaded, importing this module raises.

Functions carry the C names (dsea_init, dsea_slice, ...); `Engine` is a small
convenience wrapper over them used by the tests and bench.py.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdsea.so")

# status codes (dsea.h)
DSEA_OK = 0
DSEA_EINVAL = -1
DSEA_EGEOM = -2
DSEA_ESTATE = -3
DSEA_ECAPACITY = -4
DSEA_EUNSTABLE = -5
DSEA_ECUDA = -6
DSEA_ENOMEM = -7
DSEA_EPEER = -8
STATUS_NAMES = {0: "DSEA_OK", -1: "DSEA_EINVAL", -2: "DSEA_EGEOM", -3: "DSEA_ESTATE",
                -4: "DSEA_ECAPACITY", -5: "DSEA_EUNSTABLE", -6: "DSEA_ECUDA", -7: "DSEA_ENOMEM",
                -8: "DSEA_EPEER"}

DSEA_MODE_AUTO = 0
DSEA_MODE_FUSED = 1
DSEA_MODE_STAGED = 2

NCCL_ID_BYTES = 128


class dsea_box_params(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("rho", ctypes.c_double), ("rc", ctypes.c_double), ("dt", ctypes.c_double),
                ("T0", ctypes.c_double), ("seed", ctypes.c_uint64)]


class dsea_slice_params(ctypes.Structure):
    _fields_ = [("n_slices", ctypes.c_int32), ("cells_per_slice_x", ctypes.c_int32),
                ("n_gpus", ctypes.c_int32), ("rank", ctypes.c_int32), ("device", ctypes.c_int32),
                ("workers_per_gpu", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("slices_per_stage", ctypes.c_int32), ("capacity_factor", ctypes.c_double)]


class dsea_geometry(ctypes.Structure):
    _fields_ = [("b", ctypes.c_double * 3), ("l", ctypes.c_double * 3), ("w", ctypes.c_double),
                ("a", ctypes.c_double), ("u_shift", ctypes.c_double), ("cells", ctypes.c_int32 * 3),
                ("n_slices", ctypes.c_int32), ("n_max", ctypes.c_int32),
                ("slot_capacity", ctypes.c_int32), ("n_atoms", ctypes.c_int64)]


class dsea_energy(ctypes.Structure):
    _fields_ = [("step", ctypes.c_int64), ("U", ctypes.c_double), ("KE", ctypes.c_double),
                ("V", ctypes.c_double)]


class dsea_profile(ctypes.Structure):
    _fields_ = [("samples", ctypes.c_int64), ("n_sum", ctypes.c_double), ("U_sum", ctypes.c_double),
                ("V_sum", ctypes.c_double), ("KE_sum", ctypes.c_double)]


class dsea_thermo(ctypes.Structure):
    _fields_ = [("step", ctypes.c_int64), ("T", ctypes.c_double), ("p", ctypes.c_double),
                ("u", ctypes.c_double), ("e", ctypes.c_double)]


class dsea_xprofile(ctypes.Structure):
    _fields_ = [("x", ctypes.c_double), ("n", ctypes.c_double), ("rho", ctypes.c_double),
                ("u", ctypes.c_double), ("T", ctypes.c_double), ("p", ctypes.c_double),
                ("samples", ctypes.c_int64)]


class dsea_stats(ctypes.Structure):
    _fields_ = [("kernel_launches", ctypes.c_int64), ("force_launches", ctypes.c_int64),
                ("atom_steps", ctypes.c_int64), ("force_ms", ctypes.c_double),
                ("bin_ms", ctypes.c_double), ("hop_ms", ctypes.c_double),
                ("hop_bytes", ctypes.c_int64), ("force_pairs", ctypes.c_int64)]


_c = ctypes.c_void_p
_st = ctypes.c_int
_pd = ctypes.POINTER(ctypes.c_double)
_pi32 = ctypes.POINTER(ctypes.c_int32)
_pi64 = ctypes.POINTER(ctypes.c_int64)

# (name, restype, argtypes) -- every symbol declared in include/dsea.h
SIGNATURES = [
    ("dsea_init", _st, [ctypes.POINTER(dsea_box_params), ctypes.POINTER(_c)]),
    ("dsea_slice", _st, [_c, ctypes.POINTER(dsea_slice_params)]),
    ("dsea_ring_connect", _st, [_c, ctypes.c_void_p, ctypes.c_int32]),
    ("dsea_ring_unique_id", _st, [ctypes.c_void_p, ctypes.c_size_t]),
    ("dsea_ring_export", _st, [_c, ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    ("dsea_ring_connect_peer", _st, [_c, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32]),
    ("dsea_ring_disconnect", _st, [_c]),
    ("dsea_step", _st, [_c, ctypes.c_int64]),
    ("dsea_destroy", None, [_c]),
    ("dsea_last_error", ctypes.c_char_p, [_c]),
    ("dsea_get_geometry", _st, [_c, ctypes.POINTER(dsea_geometry)]),
    ("dsea_get_positions", _st, [_c, _pd, ctypes.c_int64]),
    ("dsea_get_velocities", _st, [_c, _pd, ctypes.c_int64]),
    ("dsea_get_forces", _st, [_c, _pd, ctypes.c_int64]),
    ("dsea_get_cells", _st, [_c, _pi32, _pi32, ctypes.c_int64]),
    ("dsea_get_energies", _st, [_c, ctypes.POINTER(dsea_energy), ctypes.c_int64, _pi64]),
    ("dsea_get_slice", _st, [_c, ctypes.c_int32, _pd, _pd, _pd, _pi32, ctypes.c_int64, _pi64]),
    ("dsea_set_state", _st, [_c, _pd, _pd, _pd, ctypes.c_int64]),
    ("dsea_set_thermostat", _st, [_c, ctypes.c_int32, ctypes.c_double]),
    ("dsea_get_profiles", _st, [_c, ctypes.POINTER(dsea_profile), ctypes.c_int32]),
    ("dsea_reset_profiles", _st, [_c]),
    ("dsea_thermo_compute", _st, [ctypes.POINTER(dsea_energy), ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                  ctypes.POINTER(dsea_thermo)]),
    ("dsea_xprofile_compute", _st, [ctypes.POINTER(dsea_profile), ctypes.c_int32, ctypes.POINTER(dsea_geometry),
                                    ctypes.POINTER(dsea_xprofile)]),
    ("dsea_set_timing", _st, [_c, ctypes.c_int32]),
    ("dsea_get_stats", _st, [_c, ctypes.POINTER(dsea_stats)]),
    ("dsea_reset_stats", _st, [_c]),
    ("dsea_geometry_compute", _st, [ctypes.POINTER(dsea_box_params),
                                    ctypes.POINTER(dsea_slice_params), ctypes.POINTER(dsea_geometry)]),
    ("dsea_schedule", _st, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                            ctypes.c_int32, _pi32, ctypes.c_int64, _pi64]),
    ("dsea_plan_ops", _st, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                            ctypes.c_int32, _pi32, ctypes.c_int64, _pi64]),
]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2507_11289_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    for name, res, args in SIGNATURES:
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


class DseaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _check(ctx, st):
    if st != 0:
        msg = lib.dsea_last_error(ctx).decode() if ctx else ""
        raise DseaError(st, msg)


def _pd_of(a):
    return a.ctypes.data_as(_pd)


# ---- same-name functional layer ---------------------------------------------------
def dsea_init(nx, ny, nz, rho, rc, dt=0.0018, T0=1.0, seed=11289):
    box = dsea_box_params(nx, ny, nz, rho, rc, dt, T0, seed)
    ctx = ctypes.c_void_p()
    st = lib.dsea_init(ctypes.byref(box), ctypes.byref(ctx))
    if st != 0:
        raise DseaError(st, "dsea_init rejected the box parameters")
    return ctx


def dsea_slice(ctx, n_slices=0, cells_per_slice_x=1, n_gpus=1, rank=0, device=0,
               workers_per_gpu=1, mode=DSEA_MODE_AUTO, capacity_factor=0.0, slices_per_stage=0):
    sp = dsea_slice_params(n_slices, cells_per_slice_x, n_gpus, rank, device, workers_per_gpu,
                           mode, slices_per_stage, capacity_factor)
    _check(ctx, lib.dsea_slice(ctx, ctypes.byref(sp)))


def dsea_ring_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(NCCL_ID_BYTES)
    st = lib.dsea_ring_unique_id(buf, NCCL_ID_BYTES)
    if st != 0:
        raise DseaError(st, "ncclGetUniqueId failed")
    return buf.raw


def dsea_ring_connect(ctx, ids: bytes, n_ids: int):
    buf = ctypes.create_string_buffer(ids, len(ids))
    _check(ctx, lib.dsea_ring_connect(ctx, buf, n_ids))


def dsea_ring_export(ctx) -> bytes:
    n = ctypes.c_size_t()
    _check(ctx, lib.dsea_ring_export(ctx, None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value)
    _check(ctx, lib.dsea_ring_export(ctx, buf, n.value, ctypes.byref(n)))
    return buf.raw


def dsea_ring_connect_peer(ctx, blobs: list):
    data = b"".join(blobs)
    buf = ctypes.create_string_buffer(data, len(data))
    _check(ctx, lib.dsea_ring_connect_peer(ctx, buf, len(blobs[0]), len(blobs)))


def ring_connect(ctx, rank: int, world: int, backend: str = "peer"):
    """Connect one rank of a ring over torch.distributed (plumbing only): "peer" maps
    the neighbours' slot buffers over NVLink (CUDA IPC); "nccl" opens NCCL p2p links."""
    import torch.distributed as dist
    if world == 1:
        return
    if backend == "peer":
        blobs = [None] * world
        dist.all_gather_object(blobs, dsea_ring_export(ctx))
        dsea_ring_connect_peer(ctx, blobs)
    else:
        ids = [b"".join(dsea_ring_unique_id() for _ in range(world))] if rank == 0 else [None]
        dist.broadcast_object_list(ids, src=0)
        dsea_ring_connect(ctx, ids[0], world)
    dist.barrier()


def dsea_ring_disconnect(ctx):
    _check(ctx, lib.dsea_ring_disconnect(ctx))


def ring_disconnect(ctx, world: int):
    """Collective teardown: close mappings everywhere, barrier, then callers may destroy."""
    import torch.distributed as dist
    if world == 1:
        return
    dsea_ring_disconnect(ctx)
    dist.barrier()


def dsea_step(ctx, n_steps: int):
    _check(ctx, lib.dsea_step(ctx, int(n_steps)))


def dsea_destroy(ctx):
    lib.dsea_destroy(ctx)


def dsea_last_error(ctx) -> str:
    return lib.dsea_last_error(ctx).decode()


def dsea_get_geometry(ctx) -> dsea_geometry:
    g = dsea_geometry()
    _check(ctx, lib.dsea_get_geometry(ctx, ctypes.byref(g)))
    return g


def _n_atoms(ctx):
    return dsea_get_geometry(ctx).n_atoms


def dsea_get_positions(ctx, n_atoms, out=None):
    out = np.empty((n_atoms, 3)) if out is None else out
    _check(ctx, lib.dsea_get_positions(ctx, _pd_of(out), n_atoms))
    return out


def dsea_get_velocities(ctx, n_atoms, out=None):
    out = np.empty((n_atoms, 3)) if out is None else out
    _check(ctx, lib.dsea_get_velocities(ctx, _pd_of(out), n_atoms))
    return out


def dsea_get_forces(ctx, n_atoms, out=None):
    out = np.empty((n_atoms, 3)) if out is None else out
    _check(ctx, lib.dsea_get_forces(ctx, _pd_of(out), n_atoms))
    return out


def dsea_get_cells(ctx, n_atoms):
    cells = np.empty((n_atoms, 3), dtype=np.int32)
    sl = np.empty(n_atoms, dtype=np.int32)
    _check(ctx, lib.dsea_get_cells(ctx, cells.ctypes.data_as(_pi32), sl.ctypes.data_as(_pi32), n_atoms))
    return cells, sl


_ENERGY_DT = np.dtype([("step", np.int64), ("U", np.float64), ("KE", np.float64), ("V", np.float64)])


def dsea_get_energy_records(ctx):
    """The raw dsea_energy records (structured array: step, U, KE, V) of this rank."""
    n = ctypes.c_int64()
    cap = 4096
    while True:
        rec = np.zeros(cap, dtype=_ENERGY_DT)
        _check(ctx, lib.dsea_get_energies(ctx, rec.ctypes.data_as(ctypes.POINTER(dsea_energy)), cap,
                                          ctypes.byref(n)))
        if n.value < cap:
            return rec[:n.value]
        cap *= 4


_THERMO_DT = np.dtype([("step", np.int64), ("T", np.float64), ("p", np.float64), ("u", np.float64),
                       ("e", np.float64)])
_XPROF_DT = np.dtype([("x", np.float64), ("n", np.float64), ("rho", np.float64), ("u", np.float64),
                      ("T", np.float64), ("p", np.float64), ("samples", np.int64)])


def dsea_thermo_compute(records, n_atoms, volume):
    """Per-timestep T, p, u, e of dsea_energy records (the library's dsea_thermo_compute);
    returns a dict of arrays."""
    rec = np.ascontiguousarray(records, dtype=_ENERGY_DT)
    out = np.zeros(rec.shape[0], dtype=_THERMO_DT)
    _check(None, lib.dsea_thermo_compute(rec.ctypes.data_as(ctypes.POINTER(dsea_energy)), rec.shape[0],
                                         int(n_atoms), float(volume),
                                         out.ctypes.data_as(ctypes.POINTER(dsea_thermo))))
    return {k: out[k].copy() for k in _THERMO_DT.names}


def dsea_xprofile_compute(raw, geo):
    """Per-slice time averages (the library's dsea_xprofile_compute) of raw per-slice
    sums for geometry geo (a dsea_geometry); returns a dict of arrays."""
    rec = np.ascontiguousarray(raw, dtype=_PROFILE_DT)
    out = np.zeros(rec.shape[0], dtype=_XPROF_DT)
    _check(None, lib.dsea_xprofile_compute(rec.ctypes.data_as(ctypes.POINTER(dsea_profile)), rec.shape[0],
                                           ctypes.byref(geo), out.ctypes.data_as(ctypes.POINTER(dsea_xprofile))))
    return {k: out[k].copy() for k in _XPROF_DT.names}


def dsea_get_energies(ctx):
    """(steps[n], [n, 4] = {U, KE, V, E = U + KE}) of every timestep this rank computed."""
    n = ctypes.c_int64()
    cap = 4096
    while True:   # the C call writes min(cap, available): grow until it comes back short
        rec = np.zeros(cap, dtype=_ENERGY_DT)
        _check(ctx, lib.dsea_get_energies(ctx, rec.ctypes.data_as(ctypes.POINTER(dsea_energy)), cap,
                                          ctypes.byref(n)))
        if n.value < cap:
            break
        cap *= 4
    rec = rec[:n.value]
    arr = np.stack([rec["U"], rec["KE"], rec["V"], rec["U"] + rec["KE"]], axis=1) if n.value else np.zeros((0, 4))
    return rec["step"].copy(), arr


def dsea_get_slice(ctx, j):
    """The atoms of slice j in slot order: dict of xyz [n, 3], v [n, 3], f [n, 3], id [n]."""
    n = ctypes.c_int64()
    _check(ctx, lib.dsea_get_slice(ctx, int(j), None, None, None, None, 0, ctypes.byref(n)))
    k = n.value
    xyz, v, f = np.zeros((k, 3)), np.zeros((k, 3)), np.zeros((k, 3))
    ids = np.zeros(k, dtype=np.int32)
    _check(ctx, lib.dsea_get_slice(ctx, int(j), _pd_of(xyz), _pd_of(v), _pd_of(f), ids.ctypes.data_as(_pi32), k,
                                   ctypes.byref(n)))
    return {"xyz": xyz, "v": v, "f": f, "id": ids}


def dsea_set_thermostat(ctx, T_target):
    """NVT per-slice isokinetic thermostat at T_target (None/0 -> off), Q23."""
    on = T_target is not None and T_target != 0
    _check(ctx, lib.dsea_set_thermostat(ctx, 1 if on else 0, float(T_target) if on else 0.0))


_PROFILE_DT = np.dtype([("samples", np.int64), ("n_sum", np.float64), ("U_sum", np.float64),
                        ("V_sum", np.float64), ("KE_sum", np.float64)])


def dsea_get_profiles(ctx, n_slices):
    rec = np.zeros(n_slices, dtype=_PROFILE_DT)
    _check(ctx, lib.dsea_get_profiles(ctx, rec.ctypes.data_as(ctypes.POINTER(dsea_profile)), n_slices))
    return rec


def dsea_reset_profiles(ctx):
    _check(ctx, lib.dsea_reset_profiles(ctx))


def dsea_set_state(ctx, xyz, vxyz, fxyz=None):
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    vxyz = np.ascontiguousarray(vxyz, dtype=np.float64)
    f = None if fxyz is None else np.ascontiguousarray(fxyz, dtype=np.float64)
    _check(ctx, lib.dsea_set_state(ctx, _pd_of(xyz), _pd_of(vxyz), None if f is None else _pd_of(f),
                                   xyz.shape[0]))


def dsea_set_timing(ctx, enable: bool):
    _check(ctx, lib.dsea_set_timing(ctx, 1 if enable else 0))


def dsea_get_stats(ctx) -> dsea_stats:
    s = dsea_stats()
    _check(ctx, lib.dsea_get_stats(ctx, ctypes.byref(s)))
    return s


def dsea_reset_stats(ctx):
    _check(ctx, lib.dsea_reset_stats(ctx))


def dsea_geometry_compute(nx, ny, nz, rho, rc, n_slices=0, cells_per_slice_x=1, workers_per_gpu=1,
                          capacity_factor=0.0):
    box = dsea_box_params(nx, ny, nz, rho, rc, 0.0018, 1.0, 0)
    sp = dsea_slice_params(n_slices, cells_per_slice_x, 1, 0, 0, workers_per_gpu, 0, 1, capacity_factor)
    g = dsea_geometry()
    st = lib.dsea_geometry_compute(ctypes.byref(box), ctypes.byref(sp), ctypes.byref(g))
    return st, g


def dsea_schedule(n_slices, n_gpus, rank, workers_per_gpu, n_cycles):
    n = ctypes.c_int64()
    _check(None, lib.dsea_schedule(n_slices, n_gpus, rank, workers_per_gpu, n_cycles, None, 0,
                                   ctypes.byref(n)))
    rows = np.zeros((n.value, 8), dtype=np.int32)
    _check(None, lib.dsea_schedule(n_slices, n_gpus, rank, workers_per_gpu, n_cycles,
                                   rows.ctypes.data_as(_pi32), n.value, ctypes.byref(n)))
    return rows


# ---- convenience wrapper ----------------------------------------------------------
@dataclass
class Box:
    nx: int
    ny: int
    nz: int
    rho: float = 0.8
    rc: float = 2.5
    dt: float = 0.0018
    T0: float = 1.0
    seed: int = 11289


class Engine:
    """One context = one GPU.  For a ring, one Engine per process (rank)."""

    def __init__(self, box: Box):
        self.box = box
        self.ctx = dsea_init(box.nx, box.ny, box.nz, box.rho, box.rc, box.dt, box.T0, box.seed)
        self.n_atoms = 4 * box.nx * box.ny * box.nz

    def slice(self, **kw):
        dsea_slice(self.ctx, **kw)
        return self

    @property
    def geometry(self):
        return dsea_get_geometry(self.ctx)

    def step(self, n):
        dsea_step(self.ctx, n)

    def positions(self):
        return dsea_get_positions(self.ctx, self.n_atoms)

    def velocities(self):
        return dsea_get_velocities(self.ctx, self.n_atoms)

    def forces(self):
        return dsea_get_forces(self.ctx, self.n_atoms)

    def cells(self):
        return dsea_get_cells(self.ctx, self.n_atoms)

    def energies(self):
        return dsea_get_energies(self.ctx)

    def _energy_records(self):
        return dsea_get_energy_records(self.ctx)

    def _geometry_struct(self):
        return dsea_get_geometry(self.ctx)

    def set_state(self, xyz, v, f=None):
        dsea_set_state(self.ctx, xyz, v, f)

    def set_thermostat(self, T_target):
        dsea_set_thermostat(self.ctx, T_target)

    def thermo(self):
        """Per-timestep T, p, u, e (dsea_thermo_compute: p = rho T + 24 V / (3 Vol), Alg. 1's
        V; reading Q24) as a dict of arrays keyed by name."""
        g = self.geometry
        return dsea_thermo_compute(self._energy_records(), self.n_atoms, g.b[0] * g.b[1] * g.b[2])

    def pressure(self):
        """Per-timestep virial pressure p = rho T + 24 V / (3 Vol), T = 2 KE / (3 N)."""
        return self.thermo()["p"]

    def raw_profiles(self):
        return dsea_get_profiles(self.ctx, self.geometry.n_slices)

    def profiles(self, raw=None):
        """x-resolved time averages per slice (Q24) from dsea_xprofile_compute:
        slice centre x, atom count n, density rho, potential energy per atom u,
        temperature T, pressure p.  raw: per-slice sums (e.g. summed over ring ranks)."""
        return dsea_xprofile_compute(self.raw_profiles() if raw is None else raw, self._geometry_struct())

    def reset_profiles(self):
        dsea_reset_profiles(self.ctx)

    def stats(self):
        return dsea_get_stats(self.ctx)

    def close(self):
        if self.ctx:
            dsea_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


OP_RECV, OP_FORCE, OP_PASS, OP_BIN, OP_SEND = range(5)


def dsea_plan_ops(n_slices, n_gpus, rank, workers_per_gpu, n_steps, slices_per_stage=1):
    """Stream-ordered ops of one rank: [n, 7] = kind, stage, worker, slice, count, cycle, t_rel."""
    n = ctypes.c_int64()
    _check(None, lib.dsea_plan_ops(n_slices, n_gpus, rank, workers_per_gpu, n_steps, slices_per_stage,
                                   None, 0, ctypes.byref(n)))
    rows = np.zeros((n.value, 7), dtype=np.int32)
    _check(None, lib.dsea_plan_ops(n_slices, n_gpus, rank, workers_per_gpu, n_steps, slices_per_stage,
                                   rows.ctypes.data_as(_pi32), n.value, ctypes.byref(n)))
    return rows
