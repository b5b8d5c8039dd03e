"""Stencil oracle -- TEST INFRASTRUCTURE ONLY (second DSEA workload).

The paper presents DSEA as a framework for explicit short-range stencil algorithms on
sliced Cartesian grids (PAPER.md P:17-21 abstract, §3, keyword "stencil
operations"; future work "direct numerical simulation", §5) and implements only
MD.  The second workload here is the simplest explicit stencil with the paper's slice
contract: forward-time centred-space (FTCS) diffusion du/dt = alpha lap(u) on an
nx x ny x nz grid, sliced along x.  One step reads the six face neighbours, so a slice
needs one neighbour slice on each side (O_in = 1) and writes only itself
(O_out = 0).  Readings (G1-G4):

  G1  u'[x,y,z] = u + r * (s - 6 u),  r = alpha dt / h^2,  with the fixed evaluation
      order  s = ((((u[x-1] + u[x+1]) + u[y-1]) + u[y+1]) + u[z-1]) + u[z+1],
      t = 6 u,  d = s - t,  q = r d,  u' = u + q  -- every operation one IEEE double
      rounding, no fused multiply-add (the GPU path evaluates the same expression, so
      the two agree bit for bit).
  G2  y and z periodic; x (the streaming axis) is not periodic -- the first and last
      slices must not interact (requirement (3)) -- with homogeneous Neumann
      walls: the ghost plane beyond x = 0 (x = nx-1) is a copy of plane 0 (nx-1).
  G3  stable for 0 < r <= 1/6 (the maximum principle holds there).
  G4  field layout x-major, z fastest: index (x ny + y) nz + z; slice j holds planes
      [j p, (j+1) p), p = nx / n_slices.

Only tests/, __graft_entry__.smoke() and bench.py may import this module.
"""
from __future__ import annotations

import numpy as np


def ftcs_step(u: np.ndarray, r: float) -> np.ndarray:
    """One FTCS step of the whole grid, G1/G2 written out with numpy (float64)."""
    u = np.asarray(u, dtype=np.float64)
    xm = np.concatenate([u[:1], u[:-1]], axis=0)      # u[x-1], mirror ghost at x = 0
    xp = np.concatenate([u[1:], u[-1:]], axis=0)      # u[x+1], mirror ghost at x = nx-1
    ym = np.roll(u, 1, axis=1)                        # u[y-1], periodic
    yp = np.roll(u, -1, axis=1)
    zm = np.roll(u, 1, axis=2)
    zp = np.roll(u, -1, axis=2)
    s = xm + xp
    s = s + ym
    s = s + yp
    s = s + zm
    s = s + zp
    t = 6.0 * u
    d = s - t
    q = r * d
    return u + q


def run(u: np.ndarray, r: float, n_steps: int) -> np.ndarray:
    """n_steps FTCS steps (G1-G3)."""
    u = np.array(u, dtype=np.float64, copy=True)
    for _ in range(n_steps):
        u = ftcs_step(u, r)
    return u


def laplacian_matrix(nx: int, ny: int, nz: int):
    """The same operator assembled independently as a sparse matrix (test pin): the
    Kronecker sum of 1-D second differences, Neumann (mirror) in x, periodic in y, z."""
    import scipy.sparse as sp

    def d1(n, periodic):
        main = -2.0 * np.ones(n)
        off = np.ones(n - 1)
        m = sp.diags([off, main, off], [-1, 0, 1], shape=(n, n), format="lil")
        if periodic:
            m[0, n - 1] += 1.0
            m[n - 1, 0] += 1.0
        else:
            m[0, 0] += 1.0          # ghost u[-1] = u[0]
            m[n - 1, n - 1] += 1.0  # ghost u[n] = u[n-1]
        return m.tocsr()

    Ix, Iy, Iz = sp.identity(nx), sp.identity(ny), sp.identity(nz)
    return (sp.kron(sp.kron(d1(nx, False), Iy), Iz) + sp.kron(sp.kron(Ix, d1(ny, True)), Iz)
            + sp.kron(sp.kron(Ix, Iy), d1(nz, True))).tocsr()
