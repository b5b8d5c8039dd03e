"""BASELINE.json configurations as concrete synthetic workloads (
DESIGN.md §4).  Pure data: FCC cells per axis, density, cutoff, slicing.

Reading Q3: the BASELINE slice counts are honoured at rho = 0.8, rc = 2.5 by
elongating the box along x ("slices ... perpendicular to the longest axis",
P:72 §3); C4 is the paper's cube with the paper's slice rule."""
from dataclasses import dataclass


@dataclass(frozen=True)
class Config:
    name: str
    nx: int
    ny: int
    nz: int
    n_slices: int          # 0 -> paper rule floor(b_x / (c rc))
    rho: float = 0.8
    rc: float = 2.5
    cells_per_slice_x: int = 1
    T0: float = 1.0
    dt: float = 0.0018
    seed: int = 11289
    note: str = ""

    @property
    def n_atoms(self) -> int:
        return 4 * self.nx * self.ny * self.nz


CONFIGS = {
    "C1": Config("C1", 20, 10, 5, 8, note="4,000 atoms, 8 slices, 100 NVE steps, 1 GPU, oracle parity"),
    "P8": Config("P8", 48, 5, 5, 32, note="4,800 atoms, 32 slices: 8-GPU ring at oracle size"),
    "C2": Config("C2", 100, 32, 20, 64, note="256,000 atoms, 64 slices, 1 B200"),
    "C3": Config("C3", 400, 40, 32, 256, note="2,048,000 atoms, 256 slices, 8-GPU ring"),
    "C4": Config("C4", 160, 160, 160, 0, note="16,384,000-atom cube, 109 slices (paper rule), "
                 "strong scaling 1/2/4/8 GPUs"),
    "S12": Config("S12", 18, 64, 64, 12, note="294,912 atoms, 12 slices: Eq. (1) N_max = 3 (W=1), 2 (W=2); "
                  "NEXT-2 scaling study"),
    "S24": Config("S24", 36, 64, 64, 24, note="589,824 atoms, 24 slices: N_max = 6 (W=1), 4 (W=2), 3 (W=3)"),
    "C5a": Config("C5a", 400, 40, 32, 273, note="C3 box, rc 2.5, 1 cell/slice"),
    "C5b": Config("C5b", 400, 40, 32, 136, cells_per_slice_x=2, note="C3 box, rc 2.5, 2 cells/slice"),
    "C5c": Config("C5c", 400, 40, 32, 91, cells_per_slice_x=3, note="C3 box, rc 2.5, 3 cells/slice"),
    "C5d": Config("C5d", 400, 40, 32, 170, rc=4.0, note="C3 box, rc 4.0, 1 cell/slice"),
    "C5e": Config("C5e", 400, 40, 32, 85, rc=4.0, cells_per_slice_x=2, note="C3 box, rc 4.0, 2 cells/slice"),
    "C5f": Config("C5f", 400, 40, 32, 56, rc=4.0, cells_per_slice_x=3, note="C3 box, rc 4.0, 3 cells/slice"),
}


@dataclass(frozen=True)
class GridConfig:
    """Stencil workload (include/dsea_grid.h): nx x ny x nz cells,
    sliced along x into n_slices slices of nx / n_slices planes, FTCS number r."""
    name: str
    nx: int
    ny: int
    nz: int
    n_slices: int
    r: float = 0.1
    seed: int = 11289
    note: str = ""

    @property
    def n_cells(self) -> int:
        return self.nx * self.ny * self.nz


GRID_CONFIGS = {
    "G0": GridConfig("G0", 48, 12, 10, 12, note="oracle-size parity: 12 slices of 4 planes, ragged tiles"),
    "G8": GridConfig("G8", 64, 9, 40, 32, note="ring parity at 2-8 GPUs: 32 slices of 2 planes"),
    "G1": GridConfig("G1", 512, 512, 512, 128, note="bench: 134M cells (1.07 GB per field), 128 slices "
                     "of 4 planes (8 MB each); parallel-in-time ring at 1/2/4/8 GPUs"),
}
