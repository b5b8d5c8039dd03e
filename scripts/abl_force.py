"""Force-kernel timing of an ablated build (results are wrong by design; errors ignored):
python scripts/abl_force.py <pkg_parent_dir> <cfg> [steps]"""
import os
import sys
sys.path.insert(0, os.path.abspath(sys.argv[1]))
from paper_2507_11289_b200 import CONFIGS  # noqa: E402
from paper_2507_11289_b200 import dsea as D  # noqa: E402
cfg = CONFIGS[sys.argv[2]]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
e = D.Engine(D.Box(cfg.nx, cfg.ny, cfg.nz, cfg.rho, cfg.rc, cfg.dt, cfg.T0, cfg.seed))
e.slice(n_slices=cfg.n_slices, cells_per_slice_x=cfg.cells_per_slice_x)
D.dsea_set_timing(e.ctx, True)
ms = []
for s in range(steps):
    D.dsea_reset_stats(e.ctx)
    try:
        e.step(1)
    except Exception as ex:  # noqa: BLE001
        pass
    ms.append(e.stats().force_ms)
print(f"{sys.argv[1]} {cfg.name}: force ms per launch {' '.join(f'{m:.3f}' for m in ms)}")
