// dsea_internal.h -- layouts and kernel entry points shared by the host runtime
// (dsea_host.cpp) and the sm_100a kernels (dsea_kernels.cu).  Not part of the ABI.
//
// HBM layout.  A *buffer* holds one slot per slice, slot j at
// base + j*slot_bytes, each slot one contiguous block so that a ring hop is a
// single transfer (§3.1):
//   int32  cell_start[ncell+1]     cell prefix sums (CellNM = differences)
//   double x[cap], y[cap], z[cap]  positions            (MolList, P:232-234,
//   double vx[cap] vy[cap] vz[cap] velocities            redesigned as SoA,
//   double fx[cap] fy[cap] fz[cap] F_new of the last pass  cell-sorted, padded)
//   int32  id[cap]
// Atoms are sorted by (cell, z, id); cells are ordered (cx_local, cy, cz) with z
// fastest, so every (cx, cy) column is one contiguous, z-sorted run.
// A *staging* buffer (per worker) has the same per-slice SoA arrays (no
// cell_start) plus int32 key[cap] = destination global cell (slice*ncell + cell).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace dsea {

struct Geo {
    double b[3];
    double l[3];
    double rc, rc2, dt, ushift;
    int cells[3];   // global cells per axis (cells[0] = c * n_slices)
    int c;          // cells per slice along x
    int ns;         // n_slices
    int ncell;      // cells per slice = c * cells[1] * cells[2]
    int cap;        // atoms per slot
    float rc2_screen;  // fp32 pre-screen radius^2 (rc^2 + margin)
    int cell_max;      // k_bin_gather shared-memory rows per cell (larger cells: global path)
    int thermo;        // NVT: per-slice isokinetic scaling before the drift (Q23)
    double T_target;   // thermostat temperature
};

struct SlotLayout {
    size_t slot_bytes;
    size_t off_x, off_y, off_z, off_vx, off_vy, off_vz, off_fx, off_fy, off_fz, off_id;
};

inline SlotLayout make_slot_layout(int ncell, int cap) {
    SlotLayout L;
    auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
    size_t o = al(sizeof(int32_t) * (size_t)(ncell + 1));
    size_t dbl = al(sizeof(double) * (size_t)cap);
    L.off_x = o; o += dbl;
    L.off_y = o; o += dbl;
    L.off_z = o; o += dbl;
    L.off_vx = o; o += dbl;
    L.off_vy = o; o += dbl;
    L.off_vz = o; o += dbl;
    L.off_fx = o; o += dbl;
    L.off_fy = o; o += dbl;
    L.off_fz = o; o += dbl;
    L.off_id = o; o += al(sizeof(int32_t) * (size_t)cap);
    L.slot_bytes = o;
    return L;
}

// Device view of a slot buffer.
// Bin record of one arrival: written by k_bin_place, ranked and gathered by k_bin_gather.
struct BinRec {
    double z;        // position z (first sort key, Q21)
    int32_t src;     // staging index
    int32_t id;      // atom id (second sort key)
};

struct BufView {
    char* base;
    SlotLayout L;
    int32_t* cnt;    // [ns*ncell] per-cell arrival counters / cursors, by slice (not sent)
    BinRec* perm;    // [nslots*cap] bin scratch, by slot (not sent)
    int remote;      // slots live in the ring successor's memory (peer backend)
    int nslots;      // slots of the buffer: slice j lives in slot j % nslots (a pool of
                     // nslots < ns slots when only a window of slices is ever live,
                     // P:121-122 "s slots", s N_b > N_S; NEXT-3)
    int perm_slots;  // slots of the bin scratch: slice m uses perm[wrap(m + poff, perm_slots) * cap ..]
    int soff;        // slot offset of the launch: slice j of super-cycle K lives in slot
                     // (K ns + j) mod nslots -- slots follow the global sequence number, so a
                     // window of live slices that spans a super-cycle boundary (the previous
                     // cycle's last slice is finalised after the next cycle's first block)
                     // never aliases.  The host normalises soff to the launch's lowest slice,
                     // so j + soff lies in [0, 2 nslots) and the kernels wrap with one compare
                     // (wrap_slot); 0 for a full buffer
    int poff;        // the same for the bin scratch (perm_slots)
};

// Device view of a staging buffer (flat SoA over ns*cap entries).
struct StgView {
    // staged atom i of slice j at index ((j + soff) % pool) * cap + i (a pool of `pool`
    // slices; soff as in BufView)
    double *x, *y, *z, *vx, *vy, *vz, *fx, *fy, *fz;
    int32_t *id, *key;
    int pool;        // slices the arrays hold (ns in the fused pass; a window on a ring)
    int soff;        // slot offset of the launch (BufView.soff)
    int32_t* n;      // [ns] atoms staged per slice
    double4* eatom;  // energy records (u_core, vir2, ke2, pairs) of the last force pass:
                     // FORCE_TILE one per tile [ns*tiles], FORCE_PIPE one per atom [ns*cap]
};

// Force-kernel tiling.  A tile is a run of consecutive (z-sorted) home atoms of one
// (cx_local, cy) column; tiles per slice = c * cells[1] * nzt.
enum { FORCE_TILE = 0, FORCE_PIPE = 1 };
struct Tiling {
    int kind;        // FORCE_TILE (k_force_tile, default) or FORCE_PIPE (k_force_pipe, A/B)
    int home;        // home atoms per tile (the column's last tile takes any remainder)
    int nzt;         // tiles per column
    int tiles;       // tiles per slice = c * cells[1] * nzt
    int smax;        // staged atoms capacity of one CTA
    int maxh;        // per-lane hit-list capacity (rows)
    size_t smem;     // dynamic shared memory bytes
    int off_hl, off_sp, off_q;     // FORCE_TILE: byte offsets of the hit lists, FP64 staging
                                   // and FP32 screening records in dynamic shared memory
    int grid;        // persistent grid (FORCE_PIPE) = SMs x resident CTAs per SM
    int per_sm;      // resident CTAs per SM
    unsigned long long* ctr;       // device: dynamic tile counter of this context (FORCE_PIPE)
    unsigned long long* ctr_base;  // host: counter value at the next launch
};

// Energy record of one (slice, timestep) unit.
struct UnitEnergy {
    double u_core;   // sum over in-cutoff ordered pairs of s6*(s6-1), s6 = r^-6
    double vir2;     // sum of s6*(2 s6 - 1)  (V = vir2 / 2)
    double ke2;      // sum of v.v after the kick (KE = ke2 / 2)
    double npairs;   // number of in-cutoff ordered pairs
    double natoms;   // atoms of the slice at this timestep
    double lambda;   // thermostat scale factor of the slice (1 without thermostat)
};

// Error record written by kernels (first error wins).
struct DevErr {
    int32_t code;    // 0 or a dsea_status
    int32_t slice;
    int32_t atom;    // atom id or -1
    int32_t aux;
};

// ---- kernel launchers (dsea_kernels.cu, dsea_force.cu) ----------------------
Tiling choose_tiling(const Geo& g, double mean_per_cell, int smem_optin);
int force_kernel_attr(const Tiling& T);     // resident CTAs per SM (< 1: cannot launch)
int force_launch(const Geo& g, const Tiling& T, BufView in, StgView stg, int32_t* out_cnt,
                 int j0, int nj, DevErr* err, cudaStream_t s);
size_t energy_records(const Geo& g, const Tiling& T);   // records of stg.eatom
void energy_launch(const Geo& g, const Tiling& T, StgView stg, int j0, int nj, UnitEnergy* e_out,
                   cudaStream_t s);
// the pipelined kernel (A/B: DSEA_FORCE=pipe)
Tiling pipe_tiling(const Geo& g, double mean_per_cell, int smem_optin);
int pipe_kernel_attr(const Tiling& T);
void pipe_launch(const Geo& g, const Tiling& T, BufView in, StgView stg, int32_t* out_cnt, int j0, int nj,
                 DevErr* err, cudaStream_t s);
// flat staging [0, n) from by-atom AoS arrays; ids: the atoms' ids (nullptr: 0..n-1)
void aos_to_stage_launch(StgView S, const double* xyz, const double* v, const double* f, const int32_t* ids,
                         int n, cudaStream_t s);
void slots_to_aos_launch(const Geo& g, BufView in, int which, double* out, unsigned long long* count,
                         cudaStream_t s);
void signal_launch(uint32_t* flags, int first, int n, uint32_t value, cudaStream_t s);
// NVT only: v <- lambda_j v, then the drift/walls/destination of md_v3b for the
// staged atoms of slices [j0, j0+nj) (lambda_j from e_out[j], written by k_energy)
void drift_launch(const Geo& g, StgView stg, int j0, int nj, const UnitEnergy* e_out, int32_t* out_cnt,
                  DevErr* err, cudaStream_t s);
void bin_scan_launch(const Geo& g, BufView out, int m0, int nm, DevErr* err, cudaStream_t s);
void bin_place_launch(const Geo& g, BufView out, StgView stg, int s0, int nsrc, int flat_count,
                      int m0, int nm, DevErr* err, cudaStream_t s);
void bin_gather_launch(const Geo& g, BufView out, StgView stg, int m0, int nm, DevErr* err,
                       cudaStream_t s);
void init_keys_launch(const Geo& g, StgView stg, int n, int32_t* out_cnt, DevErr* err,
                      cudaStream_t s);

}  // namespace dsea
