"""Determinism probe: same engine config run twice; bitwise compare (env DSEA_MAXH etc.)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_11289_b200 import CONFIGS
from paper_2507_11289_b200 import dsea as D


def run(cfg, steps, **kw):
    c = CONFIGS[cfg]
    e = D.Engine(D.Box(c.nx, c.ny, c.nz, c.rho, c.rc, c.dt, c.T0, c.seed))
    e.slice(n_slices=c.n_slices, cells_per_slice_x=c.cells_per_slice_x, **kw)
    e.step(steps)
    r = e.velocities(), e.forces()
    e.close()
    return r


cfg = sys.argv[1] if len(sys.argv) > 1 else "P8"
for name, kw in [("fused", {}), ("staged", dict(workers_per_gpu=1, mode=D.DSEA_MODE_STAGED, slices_per_stage=1))]:
    a = run(cfg, 7, **kw)
    b = run(cfg, 7, **kw)
    print(name, "rerun equal:", np.array_equal(a[0], b[0]), np.array_equal(a[1], b[1]),
          "nbad", int((a[1] != b[1]).any(1).sum()))
    if name == "fused":
        f = a
    else:
        print("fused vs staged forces: nbad", int((a[1] != f[1]).any(1).sum()), "maxdiff", np.abs(a[1] - f[1]).max())
