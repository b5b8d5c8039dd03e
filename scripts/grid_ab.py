"""A/B timing of the stencil kernel in prebuilt copies: python scripts/grid_ab.py <pkg_parent> [cfg]"""
import os
import sys
sys.path.insert(0, os.path.abspath(sys.argv[1]))
import numpy as np  # noqa: E402
from paper_2507_11289_b200 import GRID_CONFIGS  # noqa: E402
from paper_2507_11289_b200 import grid as G  # noqa: E402
c = GRID_CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "G1"]
g = G.Grid(c.nx, c.ny, c.nz, c.n_slices, c.r)
g.set_field(np.random.default_rng(1).random((c.nx, c.ny, c.nz)))
g.step(5)
G.dsea_grid_reset_stats(g.g)
G.dsea_grid_set_timing(g.g, True)
g.step(20)
st = g.stats()
ms = st.stencil_ms / st.stencil_launches
print(f"{sys.argv[1]} {c.name}: {ms:.4f} ms/sweep, {16 * c.n_cells / ms / 1e6:.1f} GB/s")
