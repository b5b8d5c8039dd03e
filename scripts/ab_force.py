"""A/B timing of built engine variants: python scripts/ab_force.py <pkg_parent_dir> <cfg> [melt] [steps]
(<pkg_parent_dir>/paper_2507_11289_b200 holds a built libdsea.so)."""
import os
import sys
sys.path.insert(0, os.path.abspath(sys.argv[1]))
from paper_2507_11289_b200 import CONFIGS  # noqa: E402
from paper_2507_11289_b200 import dsea as D  # noqa: E402
cfg = CONFIGS[sys.argv[2]]
melt = int(sys.argv[3]) if len(sys.argv) > 3 else 200
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
e = D.Engine(D.Box(cfg.nx, cfg.ny, cfg.nz, cfg.rho, cfg.rc, cfg.dt, cfg.T0, cfg.seed))
e.slice(n_slices=cfg.n_slices, cells_per_slice_x=cfg.cells_per_slice_x)
e.step(melt)
D.dsea_reset_stats(e.ctx)
D.dsea_set_timing(e.ctx, True)
e.step(steps)
st = e.stats()
print(f"{sys.argv[1]} {cfg.name} melt {melt}: force {st.force_ms / steps:.3f} ms/launch, "
      f"bin {st.bin_ms / steps:.3f} ms/step")
