"""Thin ctypes binding of the stencil workload's C ABI (include/dsea_grid.h), in
libdsea.so next to the MD engine.  Argument marshalling only: every stencil step runs
in the library's sm_100a kernel; there is no CPU fallback (importing fails loudly
without the built library).  Functions carry the C names; `Grid` is a small wrapper
used by the tests and bench.py."""
from __future__ import annotations

import ctypes

import numpy as np

from .dsea import DseaError, lib

DSEA_GRID_MODE_AUTO, DSEA_GRID_MODE_FUSED, DSEA_GRID_MODE_STAGED = 0, 1, 2


class dsea_grid_params(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("n_slices", ctypes.c_int32), ("r", ctypes.c_double),
                ("n_gpus", ctypes.c_int32), ("rank", ctypes.c_int32), ("device", ctypes.c_int32),
                ("workers_per_gpu", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("slices_per_stage", ctypes.c_int32)]


class dsea_grid_stats(ctypes.Structure):
    _fields_ = [("kernel_launches", ctypes.c_int64), ("cell_steps", ctypes.c_int64),
                ("stencil_ms", ctypes.c_double), ("stencil_launches", ctypes.c_int64),
                ("hop_bytes", ctypes.c_int64)]


_c = ctypes.c_void_p
_st = ctypes.c_int
_pd = ctypes.POINTER(ctypes.c_double)

# (name, restype, argtypes) -- every symbol declared in include/dsea_grid.h
SIGNATURES = [
    ("dsea_grid_create", _st, [ctypes.POINTER(dsea_grid_params), ctypes.POINTER(_c)]),
    ("dsea_grid_set_field", _st, [_c, _pd, ctypes.c_int64]),
    ("dsea_grid_get_field", _st, [_c, _pd, ctypes.c_int64]),
    ("dsea_grid_ring_export", _st, [_c, ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    ("dsea_grid_ring_connect_peer", _st, [_c, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32]),
    ("dsea_grid_ring_disconnect", _st, [_c]),
    ("dsea_grid_step", _st, [_c, ctypes.c_int64]),
    ("dsea_grid_set_timing", _st, [_c, ctypes.c_int32]),
    ("dsea_grid_get_stats", _st, [_c, ctypes.POINTER(dsea_grid_stats)]),
    ("dsea_grid_reset_stats", _st, [_c]),
    ("dsea_grid_last_error", ctypes.c_char_p, [_c]),
    ("dsea_grid_destroy", None, [_c]),
]
for _name, _res, _args in SIGNATURES:
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def _check(g, st):
    if st != 0:
        raise DseaError(st, lib.dsea_grid_last_error(g).decode() if g else "")


def dsea_grid_create(nx, ny, nz, n_slices, r, n_gpus=1, rank=0, device=0, workers_per_gpu=1,
                     mode=DSEA_GRID_MODE_AUTO, slices_per_stage=0):
    p = dsea_grid_params(nx, ny, nz, n_slices, r, n_gpus, rank, device, workers_per_gpu, mode, slices_per_stage)
    g = ctypes.c_void_p()
    st = lib.dsea_grid_create(ctypes.byref(p), ctypes.byref(g))
    if st != 0:
        raise DseaError(st, "dsea_grid_create rejected the parameters")
    return g


def dsea_grid_set_field(g, u):
    u = np.ascontiguousarray(u, dtype=np.float64)
    _check(g, lib.dsea_grid_set_field(g, u.ctypes.data_as(_pd), u.size))


def dsea_grid_get_field(g, shape):
    u = np.empty(shape, dtype=np.float64)
    _check(g, lib.dsea_grid_get_field(g, u.ctypes.data_as(_pd), u.size))
    return u


def dsea_grid_ring_export(g) -> bytes:
    n = ctypes.c_size_t()
    _check(g, lib.dsea_grid_ring_export(g, None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value)
    _check(g, lib.dsea_grid_ring_export(g, buf, n.value, ctypes.byref(n)))
    return buf.raw


def dsea_grid_ring_connect_peer(g, blobs: list):
    data = b"".join(blobs)
    buf = ctypes.create_string_buffer(data, len(data))
    _check(g, lib.dsea_grid_ring_connect_peer(g, buf, len(blobs[0]), len(blobs)))


def dsea_grid_ring_disconnect(g):
    _check(g, lib.dsea_grid_ring_disconnect(g))


def dsea_grid_step(g, n_steps: int):
    _check(g, lib.dsea_grid_step(g, int(n_steps)))


def dsea_grid_set_timing(g, enable: bool):
    _check(g, lib.dsea_grid_set_timing(g, 1 if enable else 0))


def dsea_grid_get_stats(g) -> dsea_grid_stats:
    s = dsea_grid_stats()
    _check(g, lib.dsea_grid_get_stats(g, ctypes.byref(s)))
    return s


def dsea_grid_reset_stats(g):
    _check(g, lib.dsea_grid_reset_stats(g))


def dsea_grid_destroy(g):
    lib.dsea_grid_destroy(g)


class Grid:
    """Convenience wrapper: one context (one GPU, one ring rank)."""

    def __init__(self, nx, ny, nz, n_slices, r, **kw):
        self.shape = (nx, ny, nz)
        self.g = dsea_grid_create(nx, ny, nz, n_slices, r, **kw)

    def connect(self, rank: int, world: int):
        """Peer ring over torch.distributed (plumbing only): exchange IPC blobs."""
        if world == 1:
            return
        import torch.distributed as dist
        blobs = [None] * world
        dist.all_gather_object(blobs, dsea_grid_ring_export(self.g))
        dsea_grid_ring_connect_peer(self.g, blobs)
        dist.barrier()

    def disconnect(self, world: int):
        if world == 1:
            return
        import torch.distributed as dist
        dsea_grid_ring_disconnect(self.g)
        dist.barrier()

    def set_field(self, u):
        dsea_grid_set_field(self.g, u)

    def field(self):
        return dsea_grid_get_field(self.g, self.shape)

    def step(self, n):
        dsea_grid_step(self.g, n)

    def stats(self):
        return dsea_grid_get_stats(self.g)

    def close(self):
        if self.g:
            dsea_grid_destroy(self.g)
            self.g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
