/*
 * dsea.h -- C ABI of the B200-native DSEAmd slice-streaming engine
 * (arXiv 2507.11289, "Cyclic Data Streaming on GPUs for Short Range Stencils
 * Applied to Molecular Dynamics").  Library: paper_2507_11289_b200/libdsea.so.
 *
 * Citations: P:n = PAPER.md line n, with the section / equation / algorithm.
 * Readings of passages the paper leaves open are listed in DESIGN.md §3 (Q1-Q19).
 *
 * The calls follow the paper's problem statement: prepare slices of the dataset
 * (§3), run super-cycles in which every worker advances every slice one
 * timestep (§3.1), store the slices, with the LJ case of §4:
 * box, density and cutoff, Algorithm 1 stepping.
 *
 * Conventions (all calls):
 *  - Every call returns dsea_status: 0 = OK, < 0 = error.  No C++ exception
 *    crosses the ABI.  After an error, dsea_last_error(ctx) names the cause.
 *  - The library owns every device allocation.  The caller owns every host
 *    array passed in; the library never keeps a caller pointer past the call.
 *  - Per-atom host arrays are ordered by atom id, AoS, 3 doubles per atom:
 *    id = ((ix*ny + iy)*nz + iz)*4 + k for FCC cell (ix,iy,iz) and basis site k.
 *  - A context is not thread-safe; distinct contexts are independent.
 *  - One context drives one GPU (one process per GPU).  A ring of N_GPU GPUs is
 *    N_GPU processes, each with its own context, connected by dsea_ring_connect.
 *  - Units: reduced LJ units, sigma = epsilon = m = k_B = 1.
 *  - There is no CPU fallback: calls that need a GPU return DSEA_ECUDA when
 *    no device is usable.
 */
#ifndef DSEA_H
#define DSEA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dsea_ctx dsea_ctx; /* opaque; owns all device memory */

typedef enum {
    DSEA_OK = 0,
    DSEA_EINVAL = -1,    /* bad argument: null pointer, n < 1, rho <= 0, rc <= 0, dt <= 0,
                            short buffer, atom outside the box in dsea_set_state */
    DSEA_EGEOM = -2,     /* infeasible geometry: slice width < rc, cell edge < rc, fewer
                            than 3 cells in y or z, or (single GPU, staged) N_S < 2 + 2W */
    DSEA_ESTATE = -3,    /* call order: step before slice, read-back on a rank that does
                            not hold the state, ring not connected */
    DSEA_ECAPACITY = -4, /* a slice outgrew its padded slot capacity, or a force tile its
                            shared-memory staging (message names slice and timestep) */
    DSEA_EUNSTABLE = -5, /* an atom moved more than one slice in one step, or a non-finite
                            position (message names atom id and timestep) */
    DSEA_ECUDA = -6,     /* CUDA runtime error or no usable device */
    DSEA_ENOMEM = -7,    /* device or host allocation failed */
    DSEA_EPEER = -8      /* NCCL unavailable or ring setup / transfer failed */
} dsea_status;

/* Box and run parameters (§4).  The box holds nx*ny*nz FCC
 * unit cells of edge a = (4/rho)^(1/3): b_d = n_d * a, N = 4*nx*ny*nz.  x is the
 * slicing axis and carries the mirror walls (§3, §4.2); y and z are
 * periodic (Q1).  The paper's cube is nx = ny = nz = N_i. */
typedef struct {
    int32_t nx, ny, nz; /* FCC unit cells per axis, each >= 1 */
    double rho;         /* density rho*sigma^3 > 0 */
    double rc;          /* cutoff radius > 0 (paper: 2.5) */
    double dt;          /* timestep > 0 (paper: ~1.8e-3; Q8: 0.0018) */
    double T0;          /* initial temperature for the velocity draw (Q9) */
    uint64_t seed;      /* splitmix64 seed of the velocity draw (Q9) */
} dsea_box_params;

/* Slicing and ring parameters (§3, §3.1). */
typedef struct {
    int32_t n_slices;          /* N_S; 0 -> paper rule floor(b_x / (c*rc)) */
    int32_t cells_per_slice_x; /* c >= 1 cells across a slice (paper: 1) */
    int32_t n_gpus;            /* N_GPU = ring length = number of processes, >= 1 */
    int32_t rank;              /* this process's ring position, 0 <= rank < n_gpus */
    int32_t device;            /* CUDA device ordinal for this context */
    int32_t workers_per_gpu;   /* W = N_wGPU >= 1 */
    int32_t mode;              /* DSEA_MODE_* below */
    int32_t slices_per_stage;  /* B >= 1 consecutive slices handled per stage (B = 1 is the
                                  paper's Table 1 schedule); 0 -> auto: enough atoms per
                                  launch, while keeping >= N_GPU*(2+W) blocks per super-cycle */
    double capacity_factor;    /* slot capacity / mean atoms per slice; 0 -> 1.25.  Above
                                  1.25 it declares regions denser than the mean (an
                                  inhomogeneous state): the force tiles' shared-memory
                                  staging is sized for capacity_factor / 1.25 x the mean
                                  density too */
} dsea_slice_params;

#define DSEA_MODE_AUTO 0   /* FUSED when n_gpus == 1 and W == 1, else STAGED */
#define DSEA_MODE_FUSED 1  /* n_gpus == 1, W == 1: all stages of a super-cycle fused into
                              one force launch and one bin pass (same results bitwise) */
#define DSEA_MODE_STAGED 2 /* the paper's per-stage schedule (Table 1),
                              generalised to W workers per GPU and N_GPU GPUs */

/* Derived geometry (valid after dsea_slice; dsea_geometry_compute gives it without
 * a context).  cells[0] = c * n_slices. */
typedef struct {
    double b[3];       /* box edges */
    double l[3];       /* cell edges, each >= rc */
    double w;          /* slice width b_x / N_S */
    double a;          /* FCC lattice constant */
    double u_shift;    /* rc^-6 - rc^-12 (Q6) */
    int32_t cells[3];  /* cells per axis */
    int32_t n_slices;  /* N_S */
    int32_t n_max;     /* Eq. (1): N_S / (2 + W*(O_in+O_out)), O = 1 */
    int32_t slot_capacity; /* atoms per slot (padded) */
    int64_t n_atoms;   /* N */
} dsea_geometry;

/* Per-timestep observables (Alg. 1; Q12: E = U(r_n) + KE(v_n)).
 * p = rho*T + 8 V / Vol with T = 2 KE / (3N). */
typedef struct {
    int64_t step;      /* absolute timestep index since dsea_init (0-based) */
    double U;          /* potential energy, sum over ordered pairs of 4(...)/2 */
    double KE;         /* kinetic energy after the velocity update of the same step */
    double V;          /* virial accumulator of Alg. 1 */
} dsea_energy;

/* x-resolved observables of one slice (§4.2 "DSEAmd yields spatially
 * resolved results"; reading Q24), summed over the timesteps this rank computed
 * since the last dsea_reset_profiles.  Per timestep the slice contributes its atom
 * count, the sums of its atoms' Algorithm 1 shares of U and V and its
 * post-kick kinetic energy.  Time averages are sum / samples; the slice volume is
 * w * b_y * b_z, so p_j = (n_j T_j + 8 V_j) / Vol_j with T_j = 2 KE_j / (3 n_j). */
typedef struct {
    int64_t samples;   /* timesteps accumulated */
    double n_sum;      /* sum of the slice's atom count */
    double U_sum;      /* sum of the slice's potential energy */
    double V_sum;      /* sum of the slice's virial accumulator */
    double KE_sum;     /* sum of the slice's kinetic energy (after the kick, before scaling) */
} dsea_profile;

/* Counters for the benchmark harness (filled by dsea_get_stats). */
typedef struct {
    int64_t kernel_launches;   /* kernels this context launched since the last reset */
    int64_t force_launches;    /* of which force-kernel launches */
    int64_t atom_steps;        /* atom-timesteps processed by this rank */
    double force_ms;           /* summed CUDA-event time of force launches (timing enabled) */
    double bin_ms;             /* summed CUDA-event time of bin passes (timing enabled) */
    double hop_ms;             /* summed CUDA-event time of ring sends (timing enabled) */
    int64_t hop_bytes;         /* bytes sent to the ring successor */
    int64_t force_pairs;       /* in-cutoff ordered pairs evaluated (from the last step) */
} dsea_stats;

/* ---- lifecycle ---------------------------------------------------------------- */

/* Validate the box parameters, compute a and b, generate the FCC lattice
 * (offset a/4: Q10) and the velocities (Q9) on the host.
 * No device work.  *out receives a new context (NULL on error). */
dsea_status dsea_init(const dsea_box_params *box, dsea_ctx **out);

/* Validate the slicing (requirements (1)-(3) of P:63-73; l >= rc; >= 3
 * cells in y and z), bind the CUDA device, allocate the slot pools, bin the
 * host state into cell-sorted slices on the device and keep them resident on
 * rank 0 (replaces the round-robin load of P:93).  A ring with N_GPU > N_max
 * is legal (it runs at the Eq. (1) plateau) and only noted in
 * dsea_last_error.  May be called again to re-slice. */
dsea_status dsea_slice(dsea_ctx *ctx, const dsea_slice_params *sp);

/* n_gpus > 1 only: connect this rank to its ring neighbours with NCCL
 * point-to-point links.  ids = n_gpus consecutive 128-byte ncclUniqueId blobs;
 * link r carries slices from rank r to rank (r+1) mod n_gpus.  Every rank must
 * pass the same ids (create them on rank 0 with dsea_ring_unique_id and
 * broadcast).  Collective over the ring: all ranks call it. */
dsea_status dsea_ring_connect(dsea_ctx *ctx, const void *ids, int32_t n_ids);

/* Write one fresh 128-byte ncclUniqueId into out (out_bytes >= 128). */
dsea_status dsea_ring_unique_id(void *out, size_t out_bytes);

/* Peer backend (default for bench.py).  The ring hop of P:118-119 runs on the copy
 * engines over NVLink (CUDA IPC mapping of the successor's input buffer): the last
 * worker on each GPU bins its finished slices into a local output pool (slice j in
 * slot j % pool), then a copy stream pushes them with cudaMemcpyAsync into the
 * successor's input slots and raises the successor's monotone ARRIVAL counter with
 * cuStreamWriteValue32; the successor's compute stream waits on that counter
 * (cuStreamWaitValue32, >=), and its consumption raises the predecessor's monotone
 * RELEASE counter, which the next push into the same slots waits on.  No SM and no
 * NCCL kernel is on the data path, so the hop overlaps the next block's force pass.
 * A/B paths (environment, every rank alike; a mismatch fails connect with
 * DSEA_EINVAL): DSEA_PEER_HOP=sm (bin kernels store straight into the successor's
 * slots, full-size buffers), DSEA_RING_COUNTERS=0 (one flag per slot instead of the
 * two counters).
 * dsea_ring_export writes this rank's IPC handles (input buffer, counter arrays) and
 * ring settings into out (cap >= *len; out = NULL queries *len).
 * dsea_ring_connect_peer takes the n_blobs = n_gpus blobs of all ranks, concatenated
 * in rank order (each blob_bytes long), checks that every rank runs the same slicing,
 * W, block partition and hop settings, and maps the successor's input buffer and
 * arrival counter and the predecessor's release counter.  Collective: every rank
 * calls it, then the caller must barrier before the first dsea_step.  Exclusive with
 * dsea_ring_connect on a context. */
dsea_status dsea_ring_export(dsea_ctx *ctx, void *out, size_t cap, size_t *len);
dsea_status dsea_ring_connect_peer(dsea_ctx *ctx, const void *blobs, size_t blob_bytes, int32_t n_blobs);

/* Leave the ring: close the peer mappings (or NCCL links).  Collective; call it on
 * every rank and barrier before dsea_destroy, because a rank must not free memory
 * that its neighbour still maps.  Idempotent. */
dsea_status dsea_ring_disconnect(dsea_ctx *ctx);

/* Advance the system n_steps timesteps (n_steps >= 0) by streaming the slices
 * through the ring of workers: ceil(n_steps / N_w) super-cycles of N_w =
 * N_GPU*W timesteps, the trailing workers of a partial last
 * super-cycle passing slices through unchanged (Q15).  Blocking: returns after
 * every GPU is idle; afterwards the state rests on rank 0.  Collective over the
 * ring: all ranks call it with the same n_steps. */
dsea_status dsea_step(dsea_ctx *ctx, int64_t n_steps);

void dsea_destroy(dsea_ctx *ctx); /* NULL-safe; frees all device memory */

/* Message of the last error or warning on ctx; valid until the next call on ctx.
 * Never NULL. */
const char *dsea_last_error(const dsea_ctx *ctx);

/* ---- state read-back and injection (rank 0 after dsea_step) ------------------ */

dsea_status dsea_get_geometry(const dsea_ctx *ctx, dsea_geometry *out);

/* xyz / vxyz / fxyz: caller-owned [3*n_atoms] arrays, filled by atom id.  Before
 * dsea_slice these return the host-generated initial state.  fxyz is F_new of
 * the last force pass (parity), zero before the first step. */
dsea_status dsea_get_positions(dsea_ctx *ctx, double *xyz, int64_t n_atoms);
dsea_status dsea_get_velocities(dsea_ctx *ctx, double *vxyz, int64_t n_atoms);
dsea_status dsea_get_forces(dsea_ctx *ctx, double *fxyz, int64_t n_atoms);

/* The engine's own binning of every atom as stored in the slot layout:
 * cell_xyz[3*n] = global cell (x, y, z), slice[n] = slice index. */
dsea_status dsea_get_cells(dsea_ctx *ctx, int32_t *cell_xyz, int32_t *slice, int64_t n_atoms);

/* The contents of one slice (the paper's "store slices", §3.1, one slot at a
 * time -- for states too large to gather by id, NEXT-3): the atoms of slice j in slot
 * order (cell-sorted, Q21): positions xyz[3n], velocities vxyz[3n], F_new of the last
 * force pass fxyz[3n] (any of the three may be NULL) and ids[n] (may be NULL).  Writes
 * min(cap, n_j) atoms; *n_written = n_j (call with cap = 0 to size the arrays).
 * Caller-owned arrays.  DSEA_EINVAL for j outside [0, N_S) or a null n_written;
 * DSEA_ESTATE before dsea_slice or on a rank that does not hold the state (rank 0 of a
 * ring holds it between calls, Q22). */
dsea_status dsea_get_slice(dsea_ctx *ctx, int32_t j, double *xyz, double *vxyz, double *fxyz, int32_t *ids,
                           int64_t cap, int64_t *n_written);

/* Energies of every timestep this rank computed since dsea_init, in step order.
 * Writes min(cap, available) records; *n_written gets the count written. */
dsea_status dsea_get_energies(dsea_ctx *ctx, dsea_energy *out, int64_t cap, int64_t *n_written);

/* Replace the state (positions, velocities, optional F_new; NULL -> zero, the Q7
 * convention) and re-bin on the device.  Positions must lie in [0,b_x] x [0,b_y)
 * x [0,b_z).  On a multi-GPU ring only rank 0 stores it (other ranks: no-op). */
dsea_status dsea_set_state(dsea_ctx *ctx, const double *xyz, const double *vxyz,
                           const double *fxyz_or_null, int64_t n_atoms);

/* NVT thermostat (§4.1: md_thermo_a/b compute the velocity scale factor,
 * md_v3b applies it; reading Q23).  enable != 0: every slice, every timestep, after
 * the kick: lambda_j = sqrt(T_target / T_j), T_j = sum v.v / (3 n_j) over the slice's
 * atoms (lambda = 1 for an empty or motionless slice), v <- lambda_j v, then the
 * position update.  Per slice, so the ring needs no extra exchange.  Energies keep
 * the post-kick (pre-scale) KE.  DSEA_EINVAL if enable and T_target <= 0 or not
 * finite; DSEA_ESTATE before dsea_slice.
 * Applies from the next dsea_step; on a ring every rank must set the same value. */
dsea_status dsea_set_thermostat(dsea_ctx *ctx, int32_t enable, double T_target);

/* Per-slice sums (dsea_profile) for slices 0..n_slices-1; n_slices must equal N_S
 * (DSEA_EINVAL otherwise).  On a ring each rank holds the timesteps it computed;
 * the caller sums over ranks.  dsea_reset_profiles zeroes them (dsea_slice does). */
dsea_status dsea_get_profiles(dsea_ctx *ctx, dsea_profile *out, int32_t n_slices);
dsea_status dsea_reset_profiles(dsea_ctx *ctx);

/* ---- thermodynamic observables (NEXT-1; §4.2 validation: u and p) ------ */

/* Per-timestep state point derived from the dsea_energy records (Alg. 1's U, KE, V,
 * P:250; reading Q24): T = 2 KE / (3 N) (k_B = m = 1, 3N degrees of freedom,
 * Q9/Q11), u = U / N, e = (U + KE) / N, p = rho T + 24 V / (3 Vol) = rho T + 8 V / Vol
 * (Alg. 1's V omits the factor 24 of sum r.F; Vol = b_x b_y b_z, rho = N / Vol). */
typedef struct {
    int64_t step;
    double T, p, u, e;
} dsea_thermo;

/* dsea_energy records in[0..n) of a box of n_atoms atoms and volume `volume` -> out[0..n)
 * (host only, no context: callers may merge the records of a ring's ranks first).
 * Caller-owned arrays; in and out may not alias.  DSEA_EINVAL on null pointers with
 * n > 0, n < 0, n_atoms <= 0 or volume <= 0. */
dsea_status dsea_thermo_compute(const dsea_energy *in, int64_t n, int64_t n_atoms, double volume,
                                dsea_thermo *out);

/* x-resolved time averages of one slice ("spatially resolved results";
 * reading Q24): slice centre x, mean atom count n, number density rho = n / Vol_j,
 * potential energy per atom u, temperature T = 2 KE / (3 n), pressure
 * p = rho T + 8 V / Vol_j with Vol_j = w b_y b_z.  Empty slices (n = 0) report u = T = 0. */
typedef struct {
    double x, n, rho, u, T, p;
    int64_t samples;
} dsea_xprofile;

/* Raw per-slice sums (dsea_get_profiles, summed over a ring's ranks by the caller)
 * -> averages out[0..n_slices) for the geometry geo (host only).  DSEA_EINVAL on null
 * pointers or n_slices != geo->n_slices. */
dsea_status dsea_xprofile_compute(const dsea_profile *raw, int32_t n_slices, const dsea_geometry *geo,
                                  dsea_xprofile *out);

/* ---- instrumentation ---------------------------------------------------------- */

/* enable != 0: bracket every force launch, bin pass and send with CUDA events on
 * the stream it runs on, summed into dsea_stats (costs one event pair per launch). */
dsea_status dsea_set_timing(dsea_ctx *ctx, int32_t enable);
dsea_status dsea_get_stats(dsea_ctx *ctx, dsea_stats *out);
dsea_status dsea_reset_stats(dsea_ctx *ctx);

/* ---- host-only helpers (no device needed; used by the CPU test suite) --------- */

/* The geometry dsea_slice would derive (DSEA_EGEOM if infeasible, out still filled). */
dsea_status dsea_geometry_compute(const dsea_box_params *box, const dsea_slice_params *sp,
                                  dsea_geometry *out);

/* The static stage schedule of one rank for n_cycles super-cycles (Table 1,
 * P:153-171, generalised to W workers and N_GPU ranks; 1-based slice numbers as in
 * the table).  Each row is 8 int32: {stage, recv, worker, process, bin, send,
 * cycle, timestep} with -1 for "none"; one row per (stage, worker) pair that
 * does something.  rows = NULL queries the count into *n_rows. */
dsea_status dsea_schedule(int32_t n_slices, int32_t n_gpus, int32_t rank, int32_t workers_per_gpu,
                          int32_t n_cycles, int32_t *rows, int64_t cap_rows, int64_t *n_rows);

/* The op list one rank's runtime executes for n_steps timesteps with B =
 * slices_per_stage slices per stage (the generalised Table 1 of dsea_schedule), in
 * stream order.  Each row is 7 int32: {kind (0 recv, 1 force, 2 pass-through,
 * 3 bin/finalise, 4 send), stage, worker (-1 for recv), first slice (0-based),
 * slice count, super-cycle, timestep relative to the call (force; else -1)}.
 * The list is in the order the default (copy-engine) ring executes it: pushes to the
 * successor leave in (super-cycle, slot) order.
 * rows = NULL queries the count into *n_rows.  Host only; used by the CPU tests to
 * check the cross-rank dependency order (no deadlock, every unit once). */
dsea_status dsea_plan_ops(int32_t n_slices, int32_t n_gpus, int32_t rank, int32_t workers_per_gpu,
                          int64_t n_steps, int32_t slices_per_stage, int32_t *rows, int64_t cap_rows,
                          int64_t *n_rows);

#ifdef __cplusplus
}
#endif
#endif /* DSEA_H */
