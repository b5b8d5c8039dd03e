"""ctypes wrapper of oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY.

The oracle is the plain O(N^2) CPU implementation of Algorithm 1 of arXiv
2507.11289 with the boundary readings of DESIGN.md §3.
Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package.  The product path
(paper_2507_11289_b200) never imports it.

All per-atom arrays are float64 numpy arrays of shape (N, 3), ordered by atom id.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_d = ctypes.c_double
_i = ctypes.c_int
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_pd = ctypes.POINTER(ctypes.c_double)
_pi32 = ctypes.POINTER(ctypes.c_int32)
_pi64 = ctypes.POINTER(ctypes.c_int64)
_pu64 = ctypes.POINTER(ctypes.c_uint64)


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2 -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
               "-shared", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.oracle_geometry.argtypes = [_i, _i, _i, _d, _d, _i, _i, _pd]
        L.oracle_geometry.restype = _i
        L.oracle_lattice.argtypes = [_i, _i, _i, _d, _pd]
        L.oracle_lattice.restype = None
        L.oracle_splitmix64_next.argtypes = [_pu64]
        L.oracle_splitmix64_next.restype = _u64
        L.oracle_normal.argtypes = [_pu64]
        L.oracle_normal.restype = _d
        L.oracle_velocities.argtypes = [_i64, _u64, _d, _pd]
        L.oracle_velocities.restype = None
        L.oracle_forces.argtypes = [_i64, _pd, _pd, _d, _pd, _pd, _pd, _pd, _pd, _i]
        L.oracle_forces.restype = None
        L.oracle_forces_subset.argtypes = [_i64, _pd, _pd, _d, _i64, _pi64, _pd, _pd, _i]
        L.oracle_forces_subset.restype = None
        L.oracle_run.argtypes = [_i64, _pd, _pd, _pd, _pd, _d, _d, _i64, _pd, _i]
        L.oracle_run_ex.argtypes = [_i64, _pd, _pd, _pd, _pd, _d, _d, _i64, _pd, _i, _d, _pd, _pi32,
                                    _i, _i, _pd]
        L.oracle_run.restype = _i
        L.oracle_run_ex.restype = _i
        L.oracle_bin.argtypes = [_i64, _pd, _pd, _pi32, _i, _pi32, _pi32]
        L.oracle_bin.restype = None
        L.oracle_nmax.argtypes = [_i, _i, _i, _i]
        L.oracle_nmax.restype = _i
        L.oracle_num_threads.argtypes = []
        L.oracle_num_threads.restype = _i
        _lib = L
    return _lib


def _p(a: np.ndarray, t=_pd):
    return a.ctypes.data_as(t)


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


@dataclass
class Geometry:
    b: np.ndarray        # box edges (3,)
    l: np.ndarray        # cell edges (3,)
    w: float             # slice width
    a: float             # FCC lattice constant
    ushift: float
    cells: np.ndarray    # int32 (3,)
    n_slices: int
    n_atoms: int
    feasible: bool


def geometry(nx, ny, nz, rho, rc, n_slices=0, c=1) -> Geometry:
    out = np.zeros(16)
    rv = lib().oracle_geometry(nx, ny, nz, rho, rc, n_slices, c, _p(out))
    return Geometry(b=out[0:3].copy(), l=out[3:6].copy(), w=float(out[6]), a=float(out[7]),
                    ushift=float(out[8]), cells=out[9:12].astype(np.int32), n_slices=int(out[12]),
                    n_atoms=int(out[13]), feasible=(rv == 0))


def lattice(nx, ny, nz, a) -> np.ndarray:
    n = 4 * nx * ny * nz
    xyz = np.zeros((n, 3))
    lib().oracle_lattice(nx, ny, nz, a, _p(xyz))
    return xyz


def splitmix64(seed: int, count: int) -> list[int]:
    st = ctypes.c_uint64(seed)
    return [int(lib().oracle_splitmix64_next(ctypes.byref(st))) for _ in range(count)]


def normals(seed: int, count: int) -> np.ndarray:
    st = ctypes.c_uint64(seed)
    return np.array([lib().oracle_normal(ctypes.byref(st)) for _ in range(count)])


def velocities(n, seed, T0) -> np.ndarray:
    v = np.zeros((n, 3))
    lib().oracle_velocities(n, seed, T0, _p(v))
    return v


def forces(xyz, box, rc, nthreads=None, per_atom=False):
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    box = np.ascontiguousarray(box, dtype=np.float64)
    n = xyz.shape[0]
    F = np.zeros((n, 3))
    U = ctypes.c_double()
    V = ctypes.c_double()
    Ui = np.zeros(n) if per_atom else None
    Vi = np.zeros(n) if per_atom else None
    lib().oracle_forces(n, _p(xyz), _p(box), rc, _p(F), ctypes.byref(U), ctypes.byref(V),
                        _p(Ui) if per_atom else None, _p(Vi) if per_atom else None,
                        nthreads or default_threads())
    if per_atom:
        return F, U.value, V.value, Ui, Vi
    return F, U.value, V.value


def forces_subset(xyz, box, rc, idx, nthreads=None):
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    box = np.ascontiguousarray(box, dtype=np.float64)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    F = np.zeros((idx.shape[0], 3))
    Ui = np.zeros(idx.shape[0])
    lib().oracle_forces_subset(xyz.shape[0], _p(xyz), _p(box), rc, idx.shape[0], _p(idx, _pi64),
                               _p(F), _p(Ui), nthreads or default_threads())
    return F, Ui


def run(xyz, v, F, box, rc, dt, nsteps, nthreads=None):
    """Advance (xyz, v, F) in place-copies by nsteps; returns (xyz, v, F, energies[nsteps,4])."""
    xyz = np.array(xyz, dtype=np.float64, order="C")
    v = np.array(v, dtype=np.float64, order="C")
    F = np.array(F, dtype=np.float64, order="C")
    box = np.ascontiguousarray(box, dtype=np.float64)
    e = np.zeros((max(nsteps, 0), 4))
    rv = lib().oracle_run(xyz.shape[0], _p(xyz), _p(v), _p(F), _p(box), rc, dt, nsteps, _p(e),
                          nthreads or default_threads())
    if rv != 0:
        raise MemoryError("oracle_run failed")
    return xyz, v, F, e


def run_ex(xyz, v, F, box, rc, dt, nsteps, geom, T_target=None, nthreads=None):
    """Algorithm 1 with the optional per-slice NVT thermostat (reading Q23)
    and per-slice records.  geom: oracle.geometry(...) of the same box.  Returns
    (xyz, v, F, energies[nsteps, 4], slice_rec[nsteps, n_slices, 4] = {n, U, V, KE})."""
    xyz = np.array(xyz, dtype=np.float64, order="C")
    v = np.array(v, dtype=np.float64, order="C")
    F = np.array(F, dtype=np.float64, order="C")
    box = np.ascontiguousarray(box, dtype=np.float64)
    l = np.ascontiguousarray(geom.l, dtype=np.float64)
    cells = np.ascontiguousarray(geom.cells, dtype=np.int32)
    ns = int(geom.n_slices)
    e = np.zeros((max(nsteps, 0), 4))
    rec = np.zeros((max(nsteps, 0), ns, 4))
    rv = lib().oracle_run_ex(xyz.shape[0], _p(xyz), _p(v), _p(F), _p(box), rc, dt, nsteps, _p(e),
                             nthreads or default_threads(), -1.0 if T_target is None else float(T_target),
                             _p(l), _p(cells, _pi32), int(geom.cells[0]) // ns, ns, _p(rec))
    if rv != 0:
        raise RuntimeError(f"oracle_run_ex failed ({rv})")
    return xyz, v, F, e, rec


def pressure(KE, V, n_atoms, volume):
    """Virial pressure from Algorithm 1's accumulators ("virial V (for pressure
    calculation)"): p = rho T + W / (3 Vol) with T = 2 KE / (3 N) and the virial
    W = sum_{i<j} r_ij . F_ij = 24 V (Alg. 1 accumulates (2 r^-12 - r^-6) / 2 per
    ordered pair, i.e. W / 24).  Works elementwise on arrays (x-resolved profiles:
    per-slice KE, V, n and the slice volume)."""
    KE = np.asarray(KE, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    n = np.asarray(n_atoms, dtype=np.float64)
    T = np.divide(2.0 * KE, 3.0 * n, out=np.zeros_like(KE * n), where=n > 0)
    return (n / volume) * T + 24.0 * V / (3.0 * volume)


def bin_atoms(xyz, l, cells, c=1):
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    l = np.ascontiguousarray(l, dtype=np.float64)
    cells = np.ascontiguousarray(cells, dtype=np.int32)
    n = xyz.shape[0]
    cx = np.zeros((n, 3), dtype=np.int32)
    sl = np.zeros(n, dtype=np.int32)
    lib().oracle_bin(n, _p(xyz), _p(l), _p(cells, _pi32), c, _p(cx, _pi32), _p(sl, _pi32))
    return cx, sl


def nmax(n_slices, w_per_gpu, o_in=1, o_out=1) -> int:
    return int(lib().oracle_nmax(n_slices, w_per_gpu, o_in, o_out))


def num_threads() -> int:
    return int(lib().oracle_num_threads())
