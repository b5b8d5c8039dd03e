"""B200-native DSEAmd: the data-parallel hot path of arXiv 2507.11289 (cyclic data
streaming of cell-binned slices through a ring of GPUs, applied to Lennard-Jones
MD) as sm_100a CUDA kernels behind the C ABI of include/dsea.h.

`paper_2507_11289_b200.dsea` is the ctypes binding (same names as the C calls);
importing it fails loudly when libdsea.so has not been built -- there is no CPU
fallback on the product path."""
from .configs import CONFIGS, GRID_CONFIGS, Config, GridConfig  # noqa: F401
