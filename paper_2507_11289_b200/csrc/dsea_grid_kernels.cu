// dsea_grid_kernels.cu -- sm_100a kernel of the stencil workload (include/dsea_grid.h).
//
// k_ftcs: one FTCS diffusion step (readings G1-G2) of the planes
// [x0, x1) of a field, reading planes x0-1 .. x1 of `in` and writing `out` at the same
// offsets (a ring worker reads its input buffer and writes its output buffer, whose
// slots share the layout).  HBM-bound: 16 algorithmic bytes per cell (one read, one
// write); a thread owns one (y, z) column of a tile and marches along x with the
// planes x-1, x, x+1 of its column in registers (each value leaves HBM once); the
// y/z neighbours come from the same plane, shared by the tile's threads through L1.
// Every operation is one IEEE double rounding in the oracle's order (__dadd_rn etc.:
// no FMA contraction), so the GPU equals oracle/grid.py bit for bit.
#include <cuda_runtime.h>
#include <cstdint>

namespace dsea {

// tile shape swept on B200 (G1, 512^3, one full sweep): 32 x 4 x 32 planes 4.07 TB/s;
// 32 x 8 x 16 3.97; 32 x 8 x 32 4.02; 32 x 8 x 64 3.93; 32 x 16 x 8 3.69.  The ring's
// per-block launches cover only a few slices, where 32-plane chunks leave too few CTAs
// (ring of 4, W = 2: 4.16e11 vs 4.67e11 cell-steps/s), so the default is 32 x 8 x 16
//
#ifndef DSEA_FTCS_TY
#define DSEA_FTCS_TY 8
#endif
#ifndef DSEA_FTCS_XCHUNK
#define DSEA_FTCS_XCHUNK 16
#endif
constexpr int FTCS_TZ = 32;                 // threads along z (one warp row: coalesced)
constexpr int FTCS_TY = DSEA_FTCS_TY;       // rows along y
constexpr int FTCS_XCHUNK = DSEA_FTCS_XCHUNK;  // planes marched by one CTA

__device__ __forceinline__ void pdl_wait_g() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release_g() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// The plane x+1 of the thread's own column is the only value it needs from HBM;
// the y/z neighbours are the same plane's values loaded by the tile's other threads
// (L1 hits).  Staging the plane tile in shared memory instead (two CTA barriers per
// plane) measured slower on B200: 3.15 vs 3.97 TB/s, and so did loading the next
// plane one iteration ahead (3.71 TB/s) and two interleaved x-marches per thread
// (3.84-3.96 TB/s).
__global__ void __launch_bounds__(FTCS_TZ* FTCS_TY)
k_ftcs(const double* __restrict__ in, double* __restrict__ out, int x0, int x1, int nx, int ny, int nz,
       double r)
{
    pdl_wait_g();
    pdl_release_g();
    const int z = blockIdx.x * FTCS_TZ + threadIdx.x;
    const int y = blockIdx.y * FTCS_TY + threadIdx.y;
    const int xs = x0 + blockIdx.z * FTCS_XCHUNK;
    if (z >= nz || y >= ny || xs >= x1) return;
    const int xe = min(x1, xs + FTCS_XCHUNK);
    const size_t plane = (size_t)ny * nz;
    const int ym = (y == 0) ? ny - 1 : y - 1, yp = (y == ny - 1) ? 0 : y + 1;   // periodic (G2)
    const int zm = (z == 0) ? nz - 1 : z - 1, zp = (z == nz - 1) ? 0 : z + 1;
    const size_t col = (size_t)y * nz + z;
    const size_t oym = (size_t)ym * nz + z, oyp = (size_t)yp * nz + z;
    const size_t ozm = (size_t)y * nz + zm, ozp = (size_t)y * nz + zp;
    // planes x-1 and x of this column; mirror ghost planes at x = 0 and nx-1 (G2)
    double uc = __ldg(in + (size_t)xs * plane + col);
    double um = (xs == 0) ? uc : __ldg(in + (size_t)(xs - 1) * plane + col);
    for (int x = xs; x < xe; x++) {
        const double* p = in + (size_t)x * plane;
        const double up = (x == nx - 1) ? uc : __ldg(p + plane + col);
        double s = __dadd_rn(um, up);
        s = __dadd_rn(s, __ldg(p + oym));
        s = __dadd_rn(s, __ldg(p + oyp));
        s = __dadd_rn(s, __ldg(p + ozm));
        s = __dadd_rn(s, __ldg(p + ozp));
        const double t = __dmul_rn(6.0, uc);
        const double d = __dsub_rn(s, t);
        const double q = __dmul_rn(r, d);
        out[(size_t)x * plane + col] = __dadd_rn(uc, q);
        um = uc;
        uc = up;
    }
}

// planes [x0, x1) of an nx x ny x nz field from `in` into `out` on stream s
void ftcs_launch(const double* in, double* out, int x0, int x1, int nx, int ny, int nz, double r, bool pdl,
                 cudaStream_t s)
{
    if (x1 <= x0) return;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((nz + FTCS_TZ - 1) / FTCS_TZ, (ny + FTCS_TY - 1) / FTCS_TY,
                       (x1 - x0 + FTCS_XCHUNK - 1) / FTCS_XCHUNK);
    cfg.blockDim = dim3(FTCS_TZ, FTCS_TY, 1);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_ftcs, in, out, x0, x1, nx, ny, nz, r);
}

}  // namespace dsea
