"""Seeded synthetic input generators shared by the oracle tests and the GPU parity
tests.  Holds none of the method's arithmetic (no forces, no integration, no
binning): only random numbers and simple placements, with the recipes stated in
DESIGN.md §4."""
from __future__ import annotations

import numpy as np


def random_points(n: int, box, seed: int, min_sep: float = 0.85, margin_x: float = 0.0):
    """n points uniform in [margin_x, b_x - margin_x) x [0, b_y) x [0, b_z), rejecting
    any candidate closer than min_sep (minimum image in y/z) to an accepted point."""
    rng = np.random.default_rng(seed)
    box = np.asarray(box, dtype=np.float64)
    pts = []
    tries = 0
    while len(pts) < n:
        tries += 1
        if tries > 200000:
            raise RuntimeError("cannot place points; lower min_sep")
        p = rng.random(3) * box
        p[0] = margin_x + rng.random() * (box[0] - 2 * margin_x)
        ok = True
        for q in pts:
            d = p - q
            d[1:] -= box[1:] * np.round(d[1:] / box[1:])
            if d @ d < min_sep * min_sep:
                ok = False
                break
        if ok:
            pts.append(p)
    return np.array(pts)


def jitter(xyz: np.ndarray, box, amp: float, seed: int) -> np.ndarray:
    """Displace every point by a uniform random vector in [-amp, amp)^3, then fold x
    into (0, b_x) by reflection and y/z periodically.  Used to make thermal-looking
    states from a lattice without running dynamics."""
    rng = np.random.default_rng(seed)
    box = np.asarray(box, dtype=np.float64)
    out = xyz + (rng.random(xyz.shape) * 2.0 - 1.0) * amp
    x = out[:, 0]
    x = np.where(x < 0, -x, x)
    x = np.where(x > box[0], 2 * box[0] - x, x)
    out[:, 0] = x
    out[:, 1] = np.mod(out[:, 1], box[1])
    out[:, 2] = np.mod(out[:, 2], box[2])
    return out


def gaussian_velocities(n: int, scale: float, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, 3)) * scale


def grid_field(nx: int, ny: int, nz: int, seed: int) -> np.ndarray:
    """Seeded synthetic scalar field for the stencil workload: a
    smooth part (a few random low Fourier modes, like a large-scale temperature or
    velocity component) plus uniform noise, shape (nx, ny, nz), float64."""
    rng = np.random.default_rng(seed)
    x = (np.arange(nx) + 0.5)[:, None, None] / nx
    y = np.arange(ny)[None, :, None] / ny
    z = np.arange(nz)[None, None, :] / nz
    u = np.zeros((nx, ny, nz))
    for _ in range(4):
        kx, ky, kz = rng.integers(0, 4, 3)
        ph = rng.random(2) * 2 * np.pi
        u += rng.random() * np.cos(np.pi * kx * x) * np.cos(2 * np.pi * ky * y + ph[0]) * \
            np.cos(2 * np.pi * kz * z + ph[1])
    return u + 0.25 * rng.random((nx, ny, nz))
