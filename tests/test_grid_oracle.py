"""Pins of the stencil oracle (oracle/grid.py, readings G1-G4 of DESIGN.md §13)
against what the mathematics fixes, independent of the oracle's own code: an
independently assembled sparse Laplacian (Kronecker sum of textbook 1-D second
differences), closed-form eigenmode decay, conservation, the maximum principle, the
constant field, mirror symmetry and the slice contract (O_in = 1)."""
import numpy as np
import pytest

from oracle import grid as G
from tests import inputs

SHAPES = [(12, 6, 5), (9, 8, 7), (16, 3, 4)]


@pytest.mark.parametrize("shape", SHAPES)
def test_step_equals_sparse_laplacian(shape):
    nx, ny, nz = shape
    u = inputs.grid_field(nx, ny, nz, 3)
    r = 0.15
    L = G.laplacian_matrix(nx, ny, nz)
    ref = u.ravel() + r * (L @ u.ravel())
    out = G.ftcs_step(u, r).ravel()
    assert np.abs(out - ref).max() <= 1e-14 * np.abs(u).max() * 8


@pytest.mark.parametrize("kx,ky,kz", [(1, 0, 0), (0, 1, 0), (0, 0, 2), (2, 1, 1), (3, 2, 1)])
def test_eigenmode_decay(kx, ky, kz):
    """cos(pi kx (x+1/2)/nx) (DCT-II, Neumann) x cos(2 pi ky y/ny) x cos(2 pi kz z/nz)
    is an eigenvector; one FTCS step multiplies it by 1 + r mu,
    mu = -4 [sin^2(pi kx / 2nx) + sin^2(pi ky / ny) + sin^2(pi kz / nz)]."""
    nx, ny, nz, r, n = 10, 8, 6, 0.12, 7
    x = (np.arange(nx) + 0.5)[:, None, None]
    y = np.arange(ny)[None, :, None]
    z = np.arange(nz)[None, None, :]
    u0 = np.cos(np.pi * kx * x / nx) * np.cos(2 * np.pi * ky * y / ny) * np.cos(2 * np.pi * kz * z / nz)
    mu = -4 * (np.sin(np.pi * kx / (2 * nx)) ** 2 + np.sin(np.pi * ky / ny) ** 2 + np.sin(np.pi * kz / nz) ** 2)
    out = G.run(u0, r, n)
    assert np.abs(out - (1 + r * mu) ** n * u0).max() <= 1e-13


def test_conservation_and_maximum_principle():
    u = inputs.grid_field(14, 9, 11, 5)
    for r in (0.05, 1.0 / 6.0):
        v = G.run(u, r, 20)
        assert abs(v.sum() - u.sum()) <= 1e-12 * np.abs(u).sum()
        assert v.min() >= u.min() - 1e-15 and v.max() <= u.max() + 1e-15


def test_constant_field_is_exact_fixed_point():
    u = np.ones((6, 5, 4))
    assert np.array_equal(G.run(u, 1.0 / 6.0, 5), u)


def test_mirror_symmetry_in_x_is_exact():
    u = inputs.grid_field(8, 5, 6, 2)
    u = u + u[::-1]
    v = G.run(u, 0.1, 6)
    assert np.array_equal(v, v[::-1])


def test_slice_contract_input_order_one():
    """A slice's new values depend only on itself and one plane on each side: changing
    planes two or more away from a slice leaves its update unchanged (O_in = 1)."""
    u = inputs.grid_field(12, 5, 4, 9)
    w = u.copy()
    w[:3] += 1.0
    w[9:] -= 2.0
    a, b = G.ftcs_step(u, 0.1), G.ftcs_step(w, 0.1)
    assert np.array_equal(a[4:8], b[4:8])
    assert not np.array_equal(a[3], b[3])
