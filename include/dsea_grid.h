/*
 * dsea_grid.h -- C ABI of the second DSEA workload: an explicit short-range stencil
 * on a sliced Cartesian grid streamed through the same ring of GPUs as DSEAmd
 * (arXiv 2507.11289).  Library: paper_2507_11289_b200/libdsea.so (same library as
 * dsea.h; shares its status codes and its stage scheduler).
 *
 * Why: the paper presents DSEA as a framework for explicit algorithms on slices of
 * a dataset -- "the user of the framework has to write GPU kernels that implement
 * the algorithm and provide slices of the dataset" (P:19-20 abstract, §3,
 * keyword "stencil operations"; DNS named as future work, §5) -- and
 * implements only MD.  This workload runs a worker kernel
 * with input order O_in = 1 and output order O_out = 0 (§3) through the
 * identical Table-1 stage plan (§3.3) and ring hop as the MD engine.
 *
 * The step (readings G1-G4; oracle/grid.py is the CPU reference):
 *   u'[x,y,z] = u + r (s - 6u),  s = ((((u[x-1] + u[x+1]) + u[y-1]) + u[y+1])
 *                                     + u[z-1]) + u[z+1],
 *   FTCS diffusion du/dt = alpha lap u with r = alpha dt / h^2, every operation one
 *   IEEE double rounding in that order (no fused multiply-add: the result equals
 *   the oracle's bit for bit).  y and z periodic; x (the streaming axis) has mirror
 *   (homogeneous Neumann) walls -- the first and last slices never interact
 *   (requirement (3)).
 *
 * Conventions: as dsea.h.  Host fields are nx*ny*nz doubles, x-major with z fastest
 * (index (x*ny + y)*nz + z); slice j is planes [j*p, (j+1)*p), p = nx / n_slices.
 * The caller owns host arrays; the library owns device memory.  One context drives
 * one GPU; a ring is one context per GPU (process), connected with
 * dsea_grid_ring_export / dsea_grid_ring_connect_peer over NVLink.  After
 * dsea_grid_step returns, the field rests on rank 0 (reading Q22).
 */
#ifndef DSEA_GRID_H
#define DSEA_GRID_H

#include <stddef.h>
#include <stdint.h>

#include "dsea.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dsea_grid dsea_grid; /* opaque; owns all device memory */

/* Grid, slicing and ring parameters.
 *   nx, ny, nz        cells per axis (>= 3 each in y and z; nx = n_slices * p)
 *   n_slices          N_S >= 3; nx % n_slices == 0 (p >= 1 planes per slice)
 *   r                 alpha dt / h^2, 0 < r <= 1/6 (G3; DSEA_EINVAL otherwise)
 *   n_gpus, rank      ring length N_GPU and this process's position (0-based)
 *   device            CUDA device of this context
 *   workers_per_gpu   W = N_wGPU >= 1 (§3.1)
 *   mode              0 auto (fused whole-grid sweep when N_GPU = W = 1, else the
 *                     staged plan), 1 fused, 2 staged (a ring of one runs the plan)
 *   slices_per_stage  B slices per stage, 0 = automatic (as dsea_slice_params) */
typedef struct {
    int32_t nx, ny, nz;
    int32_t n_slices;
    double r;
    int32_t n_gpus, rank, device, workers_per_gpu, mode, slices_per_stage;
} dsea_grid_params;

typedef struct {
    int64_t kernel_launches;   /* stencil + copy kernels launched by dsea_grid_step */
    int64_t cell_steps;        /* cells x timesteps computed on this GPU */
    double stencil_ms;         /* summed device time of the stencil launches (timing on) */
    int64_t stencil_launches;  /* stencil launches timed */
    int64_t hop_bytes;         /* bytes pushed to the ring successor */
} dsea_grid_stats;

/* Validate parameters, allocate the slot buffers on `device` (input buffer + one
 * output buffer per worker, N_S slots each; flags for the peer ring).  DSEA_EINVAL
 * on bad parameters, DSEA_ECUDA without a device, DSEA_ENOMEM when memory is short.
 * *out is NULL on error. */
dsea_status dsea_grid_create(const dsea_grid_params *p, dsea_grid **out);

/* Upload (rank 0) / download (rank 0, after dsea_grid_step) the whole field:
 * nx*ny*nz doubles, layout above.  DSEA_EINVAL on a null pointer or a wrong count,
 * DSEA_ESTATE on a rank that does not hold the field. */
dsea_status dsea_grid_set_field(dsea_grid *g, const double *u, int64_t n_cells);
dsea_status dsea_grid_get_field(dsea_grid *g, double *u, int64_t n_cells);

/* Peer ring over NVLink (as dsea_ring_export / dsea_ring_connect_peer): export this
 * rank's CUDA IPC handles (input buffer, arrival and release flags) into `out`
 * (*len bytes; out = NULL queries the size), then give every rank all N_GPU blobs
 * in rank order.  Teardown: dsea_grid_ring_disconnect on every rank, a barrier,
 * then dsea_grid_destroy. */
dsea_status dsea_grid_ring_export(dsea_grid *g, void *out, size_t cap, size_t *len);
dsea_status dsea_grid_ring_connect_peer(dsea_grid *g, const void *blobs, size_t blob_bytes, int32_t n_blobs);
dsea_status dsea_grid_ring_disconnect(dsea_grid *g);

/* Advance n_steps >= 0 timesteps (blocking): super-cycles of N_w = N_GPU * W steps
 * through the stage plan; a trailing partial super-cycle passes slices through
 * (reading Q15).  DSEA_ESTATE when a ring of N_GPU > 1 is not connected. */
dsea_status dsea_grid_step(dsea_grid *g, int64_t n_steps);

/* Per-launch device timing of the stencil kernel (CUDA events on the compute
 * stream) and counters since the last reset. */
dsea_status dsea_grid_set_timing(dsea_grid *g, int32_t enable);
dsea_status dsea_grid_get_stats(dsea_grid *g, dsea_grid_stats *out);
dsea_status dsea_grid_reset_stats(dsea_grid *g);

const char *dsea_grid_last_error(const dsea_grid *g); /* valid until the next call on g */
void dsea_grid_destroy(dsea_grid *g);                 /* NULL-safe */

#ifdef __cplusplus
}
#endif

#endif /* DSEA_GRID_H */
