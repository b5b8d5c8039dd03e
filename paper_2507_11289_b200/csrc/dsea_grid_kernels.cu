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
// k_ftcs_tma (default where it applies): the same arithmetic with the planes staged
// in shared memory by the bulk-copy engine (cp.async.bulk, mbarrier completion) on a
// ring of NS plane buffers, so each SM keeps whole planes in flight instead of one
// 8-byte load per thread; see the comment above k_ftcs_tma.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <cstring>

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


// ---- k_ftcs_tma: bulk-copy plane pipeline -------------------------------------------
// Work item = (y-tile of `rows` consecutive y rows at full z extent, x chunk).  Per
// plane the tile's rows are one contiguous run of rows*nz doubles, and its two y-halo
// rows (periodic, G2) are one row each: three cp.async.bulk copies into one stage of
// (rows_max+2) x nz doubles, completed on that stage's mbarrier.  One CTA per SM
// (persistent, items b, b+G, ...), NS stages in a ring, one load issued per stage
// released -- the load sequence runs on across items, so the pipeline fills once per
// CTA.  A thread owns up to CPT cells q = k*FT_NT + tid of the tile (coalesced along
// z) and keeps planes x-1 and x of its cells in registers; the stencil reads plane x's
// y/z neighbours and plane x+1 from shared memory.  The host picks the tiling so the
// items fill the SMs in one wave with equal work (for G1, 512^3: 37 y-tiles of 13-14
// rows x 4 x-chunks of 128 planes = 148 items); y-tiles of one x-chunk run in lockstep,
// so a tile's halo rows are L2 hits of its neighbours' loads.
constexpr int FT_NT = 512;     // threads per CTA (one CTA per SM)
constexpr int FT_CPT = 14;     // max cells per thread (tile <= FT_NT*FT_CPT cells)

struct FtcsTiling {
    int nyt, nxc;        // y-tiles, x-chunks
    int rows_max;        // rows of the largest y-tile
    int ns;              // pipeline stages
    int grid;            // CTAs
    size_t stage_bytes;  // (rows_max + 2) * nz * 8, rounded to 128
    size_t smem;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t cnt)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t phase)
{
    asm volatile(
        "{\n .reg .pred p;\n"
        "FT_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra FT_WAIT_%=;\n}\n" ::"r"(a),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}

struct FtItem {
    int y0, rows, xs, xe;
};
__device__ __forceinline__ FtItem ft_item(int i, int x0, int x1, int ny, const FtcsTiling& t)
{
    const int yt = i % t.nyt, xc = i / t.nyt;
    const int P = x1 - x0;
    FtItem it;
    it.y0 = (int)((long long)yt * ny / t.nyt);
    it.rows = (int)((long long)(yt + 1) * ny / t.nyt) - it.y0;
    it.xs = x0 + (int)((long long)xc * P / t.nxc);
    it.xe = x0 + (int)((long long)(xc + 1) * P / t.nxc);
    return it;
}

__global__ void __launch_bounds__(FT_NT, 1)
k_ftcs_tma(const double* __restrict__ in, double* __restrict__ out, int x0, int x1, int nx, int ny, int nz,
           double r, FtcsTiling t)
{
    extern __shared__ __align__(128) unsigned char ft_smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(ft_smem);               // [ns] full barriers
    unsigned char* stages = ft_smem + 128;
    const int tid = threadIdx.x;
    const int nitems = t.nyt * t.nxc;
    const size_t plane = (size_t)ny * nz;
    const uint32_t bar0 = smem_u32(bar), stg0 = smem_u32(stages);
    const uint32_t row_bytes = (uint32_t)nz * 8u;

    // producer cursor (thread 0): item, next plane to load
    int p_item = blockIdx.x, p_plane = 0, p_last = -1;
    FtItem pit{};
    uint32_t nl = 0;                                                    // loads issued
    auto p_start = [&]() {
        if (p_item < nitems) {
            pit = ft_item(p_item, x0, x1, ny, t);
            p_plane = max(pit.xs - 1, 0);
            p_last = min(pit.xe, nx - 1);
        }
    };
    auto issue = [&]() {                                                // thread 0 only
        if (p_item >= nitems) return;
        const int st = (int)(nl % (uint32_t)t.ns);
        const uint32_t b = bar0 + 8u * st;
        const uint32_t d = stg0 + (uint32_t)(st * t.stage_bytes);
        const double* src = in + (size_t)p_plane * plane;
        const int ym = pit.y0 == 0 ? ny - 1 : pit.y0 - 1;
        const int yp = (pit.y0 + pit.rows) % ny;
        mbar_expect_tx(b, (uint32_t)(pit.rows + 2) * row_bytes);
        bulk_g2s(d, src + (size_t)ym * nz, row_bytes, b);
        bulk_g2s(d + row_bytes, src + (size_t)pit.y0 * nz, (uint32_t)pit.rows * row_bytes, b);
        bulk_g2s(d + (uint32_t)(pit.rows + 1) * row_bytes, src + (size_t)yp * nz, row_bytes, b);
        nl++;
        if (++p_plane > p_last) {
            p_item += gridDim.x;
            p_start();
        }
    };

    if (tid == 0) {
        for (int s = 0; s < t.ns; s++) mbar_init(bar0 + 8u * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait_g();
    pdl_release_g();
    if (tid == 0) {
        p_start();
        for (int s = 0; s < t.ns; s++) issue();
    }

    uint32_t nc = 0;                                                    // loads consumed
    auto stage_ptr = [&](uint32_t k) {
        return reinterpret_cast<const double*>(stages + (size_t)(k % (uint32_t)t.ns) * t.stage_bytes);
    };
    auto wait = [&](uint32_t k) { mbar_wait(bar0 + 8u * (k % (uint32_t)t.ns), (k / (uint32_t)t.ns) & 1u); };
    auto release = [&]() {
        __syncthreads();                                                // every thread is done with stage nc
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue();
        }
        nc++;
    };

    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
        const FtItem it = ft_item(item, x0, x1, ny, t);
        const int ncell = it.rows * nz;
        // this thread's cells: q = k*FT_NT + tid; z == 0 / z == nz-1 flags for the wrap
        uint32_t zlo = 0, zhi = 0;
#pragma unroll
        for (int k = 0; k < FT_CPT; k++) {
            const int q = k * FT_NT + tid;
            const int z = q % nz;
            if (z == 0) zlo |= 1u << k;
            if (z == nz - 1) zhi |= 1u << k;
        }
        double um[FT_CPT], uc[FT_CPT];
        if (it.xs > 0) {                                                // plane xs-1: only the own cells
            wait(nc);
            const double* S = stage_ptr(nc) + nz;
#pragma unroll
            for (int k = 0; k < FT_CPT; k++) {
                const int q = k * FT_NT + tid;
                if (q < ncell) um[k] = S[q];
            }
            release();
        }
        wait(nc);
        {
            const double* S = stage_ptr(nc) + nz;
#pragma unroll
            for (int k = 0; k < FT_CPT; k++) {
                const int q = k * FT_NT + tid;
                if (q < ncell) {
                    uc[k] = S[q];
                    if (it.xs == 0) um[k] = uc[k];                      // mirror ghost plane (G2)
                }
            }
        }
        for (int x = it.xs; x < it.xe; x++) {
            const bool last = x == nx - 1;
            if (!last) wait(nc + 1);
            const double* S = stage_ptr(nc) + nz;                       // plane x, row 0 of the tile
            const double* U = stage_ptr(nc + 1) + nz;                   // plane x+1
            double* o = out + (size_t)x * plane + (size_t)it.y0 * nz;
#pragma unroll
            for (int k = 0; k < FT_CPT; k++) {
                const int q = k * FT_NT + tid;
                if (q < ncell) {
                    const double up = last ? uc[k] : U[q];
                    const int qm = (zlo >> k & 1u) ? q + nz - 1 : q - 1;
                    const int qp = (zhi >> k & 1u) ? q - nz + 1 : q + 1;
                    double s = __dadd_rn(um[k], up);
                    s = __dadd_rn(s, S[q - nz]);
                    s = __dadd_rn(s, S[q + nz]);
                    s = __dadd_rn(s, S[qm]);
                    s = __dadd_rn(s, S[qp]);
                    const double tt = __dmul_rn(6.0, uc[k]);
                    const double d = __dsub_rn(s, tt);
                    const double qq = __dmul_rn(r, d);
                    __stcs(o + q, __dadd_rn(uc[k], qq));
                    um[k] = uc[k];
                    uc[k] = up;
                }
            }
            release();
        }
        if (it.xe < nx) release();                                      // plane xe (the last "up")
    }
}

namespace {
int env_int(const char* k, int dflt)
{
    const char* e = getenv(k);
    return (e && *e) ? atoi(e) : dflt;
}

// tiling of one launch: equal-work items filling the SMs (cost = the busiest CTA's
// rows x planes, + 1 x-halo plane per item, + a small weight for the y-halo rows);
// returns false where the kernel does not apply (odd nz: 16-byte bulk copies; a row
// too long for the stages)
bool ftcs_tiling(int P, int nx, int ny, int nz, FtcsTiling& t)
{
    (void)nx;
    if (nz % 2 != 0 || P <= 0) return false;
    static int sms = 0, smem_optin = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    }
    t.ns = env_int("DSEA_FTCS_NS", 3);
    if (t.ns < 2) t.ns = 2;
    const size_t row = (size_t)nz * 8;
    const long budget = (long)smem_optin - 128 - 1024;
    int rmax = (int)std::min<long>((long)(budget / ((long)t.ns * (long)row)) - 2, (long)FT_NT * FT_CPT / nz);
    if (env_int("DSEA_FTCS_ROWS", 0) > 0) rmax = std::min(rmax, env_int("DSEA_FTCS_ROWS", 0));
    if (rmax < 1) return false;
    const int G = sms;
    const int nyt_min = (ny + rmax - 1) / rmax;
    double best = 1e300;
    for (int nyt = nyt_min; nyt <= std::min(ny, 8 * nyt_min); nyt++) {
        const int rows = (ny + nyt - 1) / nyt;
        for (int nxc = 1; nxc <= std::min(P, 8 * G); nxc++) {
            const long items = (long)nyt * nxc;
            const long waves = (items + G - 1) / G;
            const int planes = (P + nxc - 1) / nxc;
            const double cost = (double)waves * (rows + 0.3) * (planes + 1.0);
            if (cost < best - 1e-9) {
                best = cost;
                t.nyt = nyt;
                t.nxc = nxc;
                t.rows_max = rows;
            }
            if (items >= 4L * G) break;
        }
    }
    t.grid = (int)std::min<long>((long)t.nyt * t.nxc, G);
    if (env_int("DSEA_FTCS_GRID", 0) > 0) t.grid = std::min(t.grid, env_int("DSEA_FTCS_GRID", 0));   // tests: several items per CTA
    t.stage_bytes = (((size_t)(t.rows_max + 2) * row) + 127) / 128 * 128;
    t.smem = 128 + (size_t)t.ns * t.stage_bytes;
    return t.smem <= (size_t)smem_optin;
}
}  // namespace

// planes [x0, x1) of an nx x ny x nz field from `in` into `out` on stream s; the
// bulk-copy kernel by default (DSEA_FTCS=col: the register-column kernel)
void ftcs_launch(const double* in, double* out, int x0, int x1, int nx, int ny, int nz, double r, bool pdl,
                 cudaStream_t s)
{
    if (x1 <= x0) return;
    const char* fe = getenv("DSEA_FTCS");            // A/B and tests: read per launch
    const bool col = fe && std::strcmp(fe, "col") == 0;
    FtcsTiling t{};
    if (!col && ftcs_tiling(x1 - x0, nx, ny, nz, t)) {
        static size_t attr = 0;
        if (t.smem > attr) {
            cudaFuncSetAttribute(k_ftcs_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t.smem);
            attr = t.smem;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(t.grid, 1, 1);
        cfg.blockDim = dim3(FT_NT, 1, 1);
        cfg.dynamicSmemBytes = t.smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, k_ftcs_tma, in, out, x0, x1, nx, ny, nz, r, t);
        return;
    }
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
