"""Short run for ncu: C2 or C4 fused, a few steps after a short melt."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11289_b200 import CONFIGS
from paper_2507_11289_b200 import dsea as D
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
e = D.Engine(D.Box(cfg.nx, cfg.ny, cfg.nz, cfg.rho, cfg.rc, cfg.dt, cfg.T0, cfg.seed))
mode = int(os.environ.get("PROF_MODE", "0")); B = int(os.environ.get("PROF_B", "0"))
e.slice(n_slices=cfg.n_slices, cells_per_slice_x=cfg.cells_per_slice_x, mode=mode, slices_per_stage=B)
D.dsea_set_timing(e.ctx, True)
e.step(steps)
st = e.stats()
print(f"{cfg.name}: {steps} steps, force {st.force_ms/steps:.3f} ms/launch, bin {st.bin_ms/steps:.3f} ms/step, "
      f"pairs/atom {st.force_pairs/cfg.n_atoms:.2f}")
