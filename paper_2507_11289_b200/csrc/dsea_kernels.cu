// dsea_kernels.cu -- sm_100a kernels of the DSEAmd hot path (arXiv 2507.11289).
//
//  k_force        Algorithm 1 for the atoms of one slice j, reading the
//                 positions of slices j-1, j, j+1 (O_in = 1, §4), fused
//                 with the velocity update (md_v3aa), the position update and
//                 the destination-slice decision of md_v3b and with the
//                 U/V collection of stat_collect.
//  k_bin_scan     \
//  k_bin_place     > finalisation of an output slice (§3.3): stable, data-
//  k_bin_gather   /  determined counting sort of the arrivals by (cell, z, id).
//  k_init_keys    initial binning of a host state (replaces the slice load).
//
// FP64 throughout for the physics.  The force kernel pre-screens candidate
// pairs in FP32 with a safety margin and evaluates the survivors exactly in FP64
// with the inclusive test r^2 <= rc^2, so no FP64 cycles are spent on the
// ~85% of stencil candidates beyond the cutoff.  No tensor cores: this is not a
// dense contraction.  Results are deterministic: every sum has a fixed order that
// depends only on the input slot contents.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <algorithm>
#include "dsea_internal.h"
#include "../../include/dsea.h"

#include "dsea_device.cuh"

namespace dsea {

// ------------------------------------------------------------------------------
// Persistent pipelined force kernel (default).  Same arithmetic and the same
// per-atom summation order as k_force above, organised for latency hiding:
//   * one producer warp per CTA walks the CTA's tiles (round robin over all tiles of
//     slices [j0, j0+nj)), builds each tile's 27-piece table, and stages the 9
//     neighbour columns into one of two shared-memory buffers;
//   * four consumer warps pull 16-atom chunks from the current buffer and move on
//     to the next buffer as soon as the chunks run out -- no CTA-wide barrier;
//   * buffers change hands through mbarriers (full: producer -> consumers, empty:
//     consumers -> producer).
// Energies are written per atom (u, v, ke, pairs) and reduced per slice in a fixed
// order by k_energy, so the result does not depend on which warp took which chunk.
// ------------------------------------------------------------------------------

#ifndef DSEA_PIPE_CW
#define DSEA_PIPE_CW 4
#endif
#ifndef DSEA_PIPE_HOME
#define DSEA_PIPE_HOME (DSEA_PIPE_CW * 16)
#endif
constexpr int PIPE_CWARPS = DSEA_PIPE_CW;           // consumer warps
constexpr int PIPE_CT = 32 * PIPE_CWARPS;           // consumer threads (hit-list columns)
constexpr int PIPE_THREADS = PIPE_CT + 64;          // + two producer warps
constexpr int PIPE_MINB = PIPE_CWARPS >= 8 ? 1 : 2; // resident CTAs per SM
constexpr int PIPE_HOME = DSEA_PIPE_HOME;           // home atoms per tile
constexpr int PIPE_PAD = 64;                        // slack after each staged array

struct PipeMeta {
    int j, nhome, self_base, home_first, nchunks, end, next_chunk, pad;
    int c_lo[9], c_hi[9];
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// producer-side wait: try_wait with a suspend-time hint parks the producer warp until
// the consumers release the buffer (hardware wake-up), so the wait does not spend
// issue slots that the consumer warps of the SM need
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAITS_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(200000u)
        : "memory");
}

struct PipeBuf {
    double *sx, *sy, *sz;
    float *fx, *fy, *fz;
};

__device__ __forceinline__ PipeBuf pipe_buf(unsigned char* smem, int smax, int b) {
    const size_t per = (size_t)smax * 3 * sizeof(double) + (size_t)(smax + PIPE_PAD) * 3 * sizeof(float);
    unsigned char* base = smem + (size_t)b * per;
    PipeBuf B;
    B.sx = reinterpret_cast<double*>(base);
    B.sy = B.sx + smax;
    B.sz = B.sy + smax;
    B.fx = reinterpret_cast<float*>(B.sz + smax);
    B.fy = B.fx + smax + PIPE_PAD;
    B.fz = B.fy + smax + PIPE_PAD;
    return B;
}

size_t pipe_smem_bytes(int smax, int maxh)
{
    const size_t per = (size_t)smax * 3 * sizeof(double) + (size_t)(smax + PIPE_PAD) * 3 * sizeof(float);
    return 2 * per + (size_t)maxh * PIPE_CT * sizeof(uint16_t);
}

template <int JPAR, bool NVT>
__global__ void __launch_bounds__(PIPE_THREADS, PIPE_MINB)
k_force_pipe(Geo g, Tiling T, BufView in, StgView stg, int32_t* __restrict__ out_cnt, int j0, int nj,
             DevErr* __restrict__ err, unsigned long long* __restrict__ tile_ctr,
             unsigned long long ctr_base)
{
    pdl_wait();
    pdl_release();
    constexpr int IL = 32 / JPAR;           // atoms per chunk; JPAR lanes per atom
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ PipeMeta meta[2];
    __shared__ __align__(8) uint64_t full_bar[2], empty_bar[2];
    __shared__ int pt_dst[27], pt_end[27];                 // producer-private piece table
    __shared__ const double* pt_x[27];
    __shared__ const double* pt_y[27];
    __shared__ const double* pt_z[27];
    __shared__ double pt_dy[27], pt_dz[27];
    uint16_t* hl = reinterpret_cast<uint16_t*>(smem + 2 * ((size_t)T.smax * 3 * sizeof(double) +
                                                             (size_t)(T.smax + PIPE_PAD) * 3 * sizeof(float)));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int CY = g.cells[1], CZ = g.cells[2];
    if (tid == 0) {
        for (int b = 0; b < 2; b++) {
            mbar_init(&full_bar[b], 64);                // every producer lane arrives
            mbar_init(&empty_bar[b], PIPE_CWARPS);      // one arrival per consumer warp
        }
    }
    __syncthreads();

    if (warp >= PIPE_CWARPS) {
        // ============================ producer (2 warps) ============================
        // warp P0 builds each tile's piece table; both producer warps stage it.
        const int pw = warp - PIPE_CWARPS, pl = pw * 32 + lane;
        __shared__ int sh_he, sh_ok, sh_total, sh_main_start, sh_main_dst, sh_tile;
        int it = 0;
        const long long ntiles = (long long)nj * T.tiles;
        for (;;) {
            // dynamic tile scheduling: CTAs that start late (SMs busy with other work,
            // e.g. NCCL) simply take fewer tiles
            if (pl == 0) sh_tile = (int)(atomicAdd(tile_ctr, 1ull) - ctr_base);
            asm volatile("bar.sync 1, 64;" ::: "memory");
            const long long t = sh_tile;
            asm volatile("bar.sync 1, 64;" ::: "memory");
            if (t >= ntiles) break;
            const int j = j0 + (int)(t / T.tiles);
            const int tile = (int)(t % T.tiles);
            const int tt = tile % T.nzt;
            const int rest = tile / T.nzt;
            const int cyi = rest % CY;
            const int cxl = rest / CY;
            const int32_t* csj = slot_cs(in, j);
            if (tile == 0 && pl == 0) stg.n[j] = csj[g.ncell];
            const int colbase_h = (cxl * CY + cyi) * CZ;
            const int col_first = csj[colbase_h], col_end = csj[colbase_h + CZ];
            const int h0 = col_first + tt * PIPE_HOME;
            const int h1 = (tt == T.nzt - 1) ? col_end : min(col_end, h0 + PIPE_HOME);
            const double* zj = slot_d(in, j, in.L.off_z);
            const double ox = (double)(j * g.c + cxl) * g.l[0];
            const double oy = (double)cyi * g.l[1];
            int hb = h0;
            while (hb < h1) {
                asm volatile("bar.sync 1, 64;" ::: "memory");   // previous staging done: pt_* free
                double oz = zj[hb];
                if (pw == 0) {
                    int he = h1;
                    int cnt = 0, start = 0, src_slice = 0, excl = 0, total = 0;
                    double dyv = 0.0, dzv = 0.0;
                    bool ok = true;
                    for (;;) {
                        const double zfirst = zj[hb];
                        const double zlast = zj[he - 1];
                        const int z0 = (int)floor((zfirst - g.rc - 1e-9) / g.l[2]);
                        const int z1 = (int)floor((zlast + g.rc + 1e-9) / g.l[2]);
                        cnt = 0; start = 0; src_slice = 0; dyv = 0.0; dzv = 0.0;
                        if (lane < 27) {
                            const int col = lane / 3, q = lane % 3;
                            const int dxk = col / 3 - 1, dyk = col % 3 - 1;
                            const int gx = j * g.c + cxl + dxk;
                            if (gx >= 0 && gx < g.cells[0]) {
                                const int m = gx / g.c, cx2 = gx - m * g.c;
                                int cyy = cyi + dyk;
                                if (cyy < 0) { cyy += CY; dyv = -g.b[1]; }
                                else if (cyy >= CY) { cyy -= CY; dyv = g.b[1]; }
                                const int zlo = max(z0, -1), zhi = min(z1, CZ);
                                int a0 = 0, b0 = -1;
                                if (q == 0) { if (zlo < 0) { a0 = zlo + CZ; b0 = CZ - 1; dzv = -g.b[2]; } }
                                else if (q == 1) { a0 = max(zlo, 0); b0 = min(zhi, CZ - 1); }
                                else { if (zhi >= CZ) { a0 = 0; b0 = zhi - CZ; dzv = g.b[2]; } }
                                if (b0 >= a0) {
                                    const int32_t* cs = slot_cs(in, m);
                                    const int colbase = (cx2 * CY + cyy) * CZ;
                                    start = cs[colbase + a0];
                                    cnt = cs[colbase + b0 + 1] - start;
                                    src_slice = m;
                                }
                            }
                        }
                        const int grp = lane - lane % 3;
                        const int coltot = __shfl_sync(FULLMASK, cnt, grp) + __shfl_sync(FULLMASK, cnt, min(grp + 1, 31)) +
                                           __shfl_sync(FULLMASK, cnt, min(grp + 2, 31));
                        const int span = cnt + ((lane < 27 && lane % 3 == 2) ? (coltot & 1) : 0);
                        int incl = span;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int v = __shfl_up_sync(FULLMASK, incl, o);
                            if (lane >= o) incl += v;
                        }
                        excl = incl - span;
                        total = __shfl_sync(FULLMASK, incl, 31);
                        if (total <= T.smax) break;
                        if (he - hb <= 16) { ok = false; break; }
                        he = hb + (((he - hb) / 2 + 15) & ~15);
                    }
                    if (lane < 27) {
                        pt_dst[lane] = excl;
                        pt_end[lane] = excl + cnt;
                        pt_x[lane] = slot_d(in, src_slice, in.L.off_x) + start;
                        pt_y[lane] = slot_d(in, src_slice, in.L.off_y) + start;
                        pt_z[lane] = slot_d(in, src_slice, in.L.off_z) + start;
                        pt_dy[lane] = dyv;
                        pt_dz[lane] = dzv;
                    }
                    if (lane == 13) { sh_main_start = start; sh_main_dst = excl; }
                    if (lane == 0) { sh_he = he; sh_ok = ok ? 1 : 0; sh_total = total; }
                }
                asm volatile("bar.sync 1, 64;" ::: "memory");
                const int he = sh_he, total = sh_total;
                if (!sh_ok) {
                    if (pl == 0) set_err(err, DSEA_ECAPACITY, j, -1, total);
                    break;
                }
                // ---- claim a buffer ----
                const int b = it & 1;
                if (it >= 2) mbar_wait_sleep(&empty_bar[b], ((it >> 1) - 1) & 1);
                const PipeBuf B = pipe_buf(smem, T.smax, b);
                PipeMeta& M = meta[b];
                if (pw == 0) {
                    if (lane < 9) {
                        const int lo = pt_dst[3 * lane], hi = pt_end[3 * lane + 2];
                        M.c_lo[lane] = lo;
                        M.c_hi[lane] = hi;
                        if ((hi - lo) & 1) {  // far-away dummy: never passes the screen
                            B.fx[hi] = 1e30f; B.fy[hi] = 1e30f; B.fz[hi] = 1e30f;
                            B.sx[hi] = 1e300; B.sy[hi] = 1e300; B.sz[hi] = 1e300;
                        }
                    }
                    if (lane == 0) {
                        M.j = j;
                        M.nhome = he - hb;
                        M.home_first = hb;
                        M.self_base = sh_main_dst + (hb - sh_main_start);
                        M.nchunks = (he - hb + IL - 1) / IL;
                        M.next_chunk = 0;
                        M.end = 0;
                    }
                }
                // ---- stage: 64 lanes, each resolves 4 indices, then 12 loads in flight ----
                int pc = 0;
                for (int base = pl; base < total; base += 256) {
                    int pcs[4], off[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const int sidx = base + 64 * u;
                        while (pc < 26 && sidx >= pt_end[pc]) pc++;   // monotone piece cursor
                        const bool ok = sidx < total && sidx >= pt_dst[pc] && sidx < pt_end[pc];
                        pcs[u] = ok ? pc : -1;
                        off[u] = sidx - pt_dst[pc];
                    }
                    double xv[4], yv[4], zv[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        if (pcs[u] >= 0) {
                            xv[u] = __ldg(pt_x[pcs[u]] + off[u]);
                            yv[u] = __ldg(pt_y[pcs[u]] + off[u]);
                            zv[u] = __ldg(pt_z[pcs[u]] + off[u]);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        if (pcs[u] >= 0) {
                            const int d = base + 64 * u;
                            const double x = xv[u], y = yv[u] + pt_dy[pcs[u]], z = zv[u] + pt_dz[pcs[u]];
                            B.sx[d] = x; B.sy[d] = y; B.sz[d] = z;
                            B.fx[d] = (float)(x - ox); B.fy[d] = (float)(y - oy); B.fz[d] = (float)(z - oz);
                        }
                    }
                }
                __syncwarp();
                mbar_arrive(&full_bar[b]);  // 64 arrivals: each lane releases its own stores
                it++;
                hb = he;
            }
        }
        // end marker
        const int b = it & 1;
        if (it >= 2) mbar_wait(&empty_bar[b], ((it >> 1) - 1) & 1);
        if (pl == 0) meta[b].end = 1;
        __syncwarp();
        mbar_arrive(&full_bar[b]);
        return;
    }

    // ================================ consumers ================================
    const int il = lane % IL, par = lane / IL;
    const float rc2s = g.rc2_screen;
    const double rc2 = g.rc2;
    const int maxh = T.maxh;
    constexpr int SEG_PAIRS = 8 * JPAR;     // candidate pairs per segment (8 per lane)
    constexpr int seg_need = 16;            // max appends per lane per segment
    const float2 m1 = make_float2(-1.f, -1.f);
    int it = 0;
    for (;;) {
        const int b = it & 1;
        mbar_wait(&full_bar[b], (it >> 1) & 1);
        PipeMeta& M = meta[b];
        if (M.end) break;
        const PipeBuf B = pipe_buf(smem, T.smax, b);
        const int j = M.j, nhome = M.nhome, self_base = M.self_base, home_first = M.home_first;
        const int nchunks = M.nchunks;
        const float2* X2 = reinterpret_cast<const float2*>(B.fx);
        const float2* Y2 = reinterpret_cast<const float2*>(B.fy);
        const float2* Z2 = reinterpret_cast<const float2*>(B.fz);
        for (;;) {
            int chv = 0;
            if (lane == 0) chv = atomicAdd(&M.next_chunk, 1);
            const int ch = __shfl_sync(FULLMASK, chv, 0);
            if (ch >= nchunks) break;
            const int q = ch * IL + il;
            const bool valid = q < nhome;
            const int si = self_base + (valid ? q : nhome - 1);
            const double xi = B.sx[si], yi = B.sy[si], zi = B.sz[si];
            const float xf = valid ? B.fx[si] : 1e30f, yf = B.fy[si], zf = B.fz[si];
            const float2 xi2 = make_float2(xf, xf), yi2 = make_float2(yf, yf), zi2 = make_float2(zf, zf);
            const double zmin = B.sz[self_base + ch * IL];
            const double zmax = B.sz[self_base + min(ch * IL + IL, nhome) - 1];
            int wb = 0;
            if (lane < 9 || (lane >= 16 && lane < 25)) {
                const int col = lane < 9 ? lane : lane - 16;
                int lo = M.c_lo[col], hi = M.c_hi[col];
                const int base = lo;
                if (lane < 9) {
                    const double key = zmin - g.rc - 1e-9;
                    while (lo < hi) { const int mid = (lo + hi) >> 1; if (B.sz[mid] < key) lo = mid + 1; else hi = mid; }
                    wb = base + ((lo - base) & ~1);
                } else {
                    const double key = zmax + g.rc + 1e-9;
                    while (lo < hi) { const int mid = (lo + hi) >> 1; if (B.sz[mid] <= key) lo = mid + 1; else hi = mid; }
                    wb = base + ((lo - base + 1) & ~1);
                }
            }
            // integration inputs of this lane's atom, loaded now, used after the pair work
            const int gi = home_first + (valid ? q : 0);
            double fxo = 0, fyo = 0, fzo = 0, vx0 = 0, vy0 = 0, vz0 = 0;
            int aid = 0;
            if (valid && par == 0) {
                fxo = __ldg(slot_d(in, j, in.L.off_fx) + gi);
                fyo = __ldg(slot_d(in, j, in.L.off_fy) + gi);
                fzo = __ldg(slot_d(in, j, in.L.off_fz) + gi);
                vx0 = __ldg(slot_d(in, j, in.L.off_vx) + gi);
                vy0 = __ldg(slot_d(in, j, in.L.off_vy) + gi);
                vz0 = __ldg(slot_d(in, j, in.L.off_vz) + gi);
                aid = __ldg(slot_i(in, j, in.L.off_id) + gi);
            }
            double fx = 0.0, fy = 0.0, fz = 0.0, e_u = 0.0, e_v = 0.0;
            int e_np = 0;
            int ho = tid;                        // next free hit-list slot of this lane
            auto flush = [&]() {
                // the JPAR lanes of an atom pool their hit lists and split the combined
                // list evenly: lane imbalance is then only atom-to-atom variance.
                // Lanes read each other's lists: warp barriers order those reads after
                // the owners' appends and before the owners append the next segment
                // (without the second one a lane leaving the divergent loop early can
                // overwrite entries its partner has not read yet).
                __syncwarp();
                const int mycnt = (ho - tid) / PIPE_CT;
                int pre[JPAR + 1];
                pre[0] = 0;
#pragma unroll
                for (int p = 0; p < JPAR; p++) pre[p + 1] = pre[p] + __shfl_sync(FULLMASK, mycnt, il + p * IL);
                const int tot = pre[JPAR];
                const int e0 = (par * tot) / JPAR, e1 = ((par + 1) * tot) / JPAR;
                const int tcol = tid - lane + il;                  // hit-list column of (il, 0)
                for (int e = e0; e < e1; e++) {
                    int p = 0;
#pragma unroll
                    for (int u = 1; u < JPAR; u++) p += (e >= pre[u]);
                    int pb = 0;
#pragma unroll
                    for (int u = 1; u < JPAR; u++) pb = (p == u) ? pre[u] : pb;
                    const int kk = hl[(e - pb) * PIPE_CT + tcol + p * IL];
                    const double dx = xi - B.sx[kk];
                    const double dy = yi - B.sy[kk];
                    const double dz = zi - B.sz[kk];
                    const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
                    if (r2 <= rc2 && kk != si) {      // inclusive cutoff; i != j
                        const double s = rcp64(r2);
                        // f = s^4 (2 s^3 - 1) with s^4 = (s^2)^2 formed beside s^3: one
                        // dependent multiply less on each hit's force chain than s (s^3 t)
                        // (C4 force launch -0.65 %); gq = s^3 t feeds only the virial
                        const double s2 = s * s;
                        const double s3 = s2 * s;                  // r^-6
                        const double s4 = s2 * s2;
                        const double t = fma(2.0, s3, -1.0);       // 2 r^-6 - 1
                        const double gq = s3 * t;                  // 2 r^-12 - r^-6
                        const double f = s4 * t;                   // F_abs / 24
                        fx = fma(dx, f, fx);
                        fy = fma(dy, f, fy);
                        fz = fma(dz, f, fz);
                        e_u += fma(s3, s3, -s3);
                        e_v += gq;
                        e_np += 1;
                    }
                }
                __syncwarp();
                ho = tid;
            };
            auto screen = [&](const float2 X, const float2 Y, const float2 Z, const int k) {
                const float2 dx = __ffma2_rn(X, m1, xi2);
                const float2 dy = __ffma2_rn(Y, m1, yi2);
                const float2 dz = __ffma2_rn(Z, m1, zi2);
                float2 r2 = __fmul2_rn(dz, dz);
                r2 = __ffma2_rn(dy, dy, r2);
                r2 = __ffma2_rn(dx, dx, r2);
                if (r2.x <= rc2s) { hl[ho] = (uint16_t)k; ho += PIPE_CT; }
                if (r2.y <= rc2s) { hl[ho] = (uint16_t)(k + 1); ho += PIPE_CT; }
            };
#pragma unroll 1
            for (int col = 0; col < 9; col++) {
                const int plo = __shfl_sync(FULLMASK, wb, col) >> 1;
                const int phi = __shfl_sync(FULLMASK, wb, 16 + col) >> 1;
                for (int s0 = plo; s0 < phi; s0 += SEG_PAIRS) {
                    const int e = min(phi, s0 + SEG_PAIRS);
                    // flush on the entry count only: the decision must not depend on which
                    // warp (tid) took the chunk, or the summation order would
                    if (__any_sync(FULLMASK, ho - tid + seg_need * PIPE_CT > maxh * PIPE_CT)) flush();
                    int m = s0 + par;
                    for (; m + 3 * JPAR < e; m += 4 * JPAR) {      // 4 pairs: all loads first
                        const float2 Xa = X2[m], Xb = X2[m + JPAR], Xc = X2[m + 2 * JPAR], Xd = X2[m + 3 * JPAR];
                        const float2 Ya = Y2[m], Yb = Y2[m + JPAR], Yc = Y2[m + 2 * JPAR], Yd = Y2[m + 3 * JPAR];
                        const float2 Za = Z2[m], Zb = Z2[m + JPAR], Zc = Z2[m + 2 * JPAR], Zd = Z2[m + 3 * JPAR];
                        screen(Xa, Ya, Za, 2 * m);
                        screen(Xb, Yb, Zb, 2 * (m + JPAR));
                        screen(Xc, Yc, Zc, 2 * (m + 2 * JPAR));
                        screen(Xd, Yd, Zd, 2 * (m + 3 * JPAR));
                    }
                    for (; m < e; m += JPAR) screen(X2[m], Y2[m], Z2[m], 2 * m);
                }
            }
            flush();
            // combine the two parity lanes of each atom (fixed order)
#pragma unroll
            for (int o = IL; o < 32; o <<= 1) {   // fixed xor tree over the atom's lanes
                fx += __shfl_xor_sync(FULLMASK, fx, o);
                fy += __shfl_xor_sync(FULLMASK, fy, o);
                fz += __shfl_xor_sync(FULLMASK, fz, o);
                e_u += __shfl_xor_sync(FULLMASK, e_u, o);
                e_v += __shfl_xor_sync(FULLMASK, e_v, o);
                e_np += __shfl_xor_sync(FULLMASK, e_np, o);
            }
            if (valid && par == 0) {
                const double Fx = 24.0 * fx, Fy = 24.0 * fy, Fz = 24.0 * fz;
                const double hdt = 0.5 * g.dt;
                const double vx = vx0 + (Fx + fxo) * hdt;
                const double vy = vy0 + (Fy + fyo) * hdt;
                const double vz = vz0 + (Fz + fzo) * hdt;
                const double ke2 = vx * vx + vy * vy + vz * vz;
                const size_t st = stg_index(stg, j, g.cap, gi);
                stg.eatom[st] = make_double4(e_u, e_v, ke2, (double)e_np);
                if (NVT) {
                    // NVT: the slice's scale factor needs every atom's kick first
                    // (k_energy -> lambda_j, then k_drift finishes md_v3b)
                    stg.x[st] = xi; stg.y[st] = yi; stg.z[st] = zi;
                    stg.vx[st] = vx; stg.vy[st] = vy; stg.vz[st] = vz;
                    stg.fx[st] = Fx; stg.fy[st] = Fy; stg.fz[st] = Fz;
                    stg.id[st] = aid;
                } else {
                    drift_store(g, stg, st, j, xi, yi, zi, vx, vy, vz, Fx, Fy, Fz, aid, out_cnt, err);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[b]);
        it++;
    }
}

// Per-slice energies in a fixed order: thread-strided sums, warp trees, warps in order.
constexpr int ENERGY_THREADS = 256;

__global__ void __launch_bounds__(ENERGY_THREADS)
k_energy(Geo g, StgView stg, int j0, int stride, int nrec, UnitEnergy* __restrict__ e_out)
{
    pdl_wait();
    pdl_release();
    const int j = j0 + blockIdx.x;
    const int n = stg.n[j];
    const double4* e = stg.eatom + (size_t)j * stride;
    const int nr = nrec > 0 ? nrec : n;     // per-tile records, or one per staged atom
    double a = 0, b = 0, c = 0, d = 0;
    for (int p = threadIdx.x; p < nr; p += ENERGY_THREADS) {
        const double4 v = e[p];
        a += v.x; b += v.y; c += v.z; d += v.w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(FULLMASK, a, o);
        b += __shfl_xor_sync(FULLMASK, b, o);
        c += __shfl_xor_sync(FULLMASK, c, o);
        d += __shfl_xor_sync(FULLMASK, d, o);
    }
    __shared__ double s[ENERGY_THREADS / 32][4];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { s[warp][0] = a; s[warp][1] = b; s[warp][2] = c; s[warp][3] = d; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double A = 0, B = 0, C = 0, D = 0;
        for (int w = 0; w < ENERGY_THREADS / 32; w++) { A += s[w][0]; B += s[w][1]; C += s[w][2]; D += s[w][3]; }
        UnitEnergy ue;
        ue.u_core = A; ue.vir2 = B; ue.ke2 = C; ue.npairs = D;
        ue.natoms = (double)n;
        // md_thermo_a/b, reading Q23: lambda_j = sqrt(T_target / T_j),
        // T_j = sum v.v / (3 n_j) after the kick; 1 for an empty or motionless slice
        double lam = 1.0;
        if (g.thermo && n > 0 && C > 0.0) lam = sqrt(g.T_target / (C / (3.0 * (double)n)));
        ue.lambda = lam;
        e_out[j] = ue;
    }
}

// NVT: scale the kicked velocities of slice j by lambda_j (the velocity scaling of
// md_v3b), then the position update and destination as in the NVE path.
constexpr int DRIFT_THREADS = 256;

__global__ void __launch_bounds__(DRIFT_THREADS)
k_drift(Geo g, StgView stg, int j0, const UnitEnergy* __restrict__ e_out, int32_t* __restrict__ out_cnt,
        DevErr* __restrict__ err)
{
    pdl_wait();
    pdl_release();
    const int j = j0 + blockIdx.y;
    const int n = stg.n[j];
    const double lam = e_out[j].lambda;
    for (int i = blockIdx.x * DRIFT_THREADS + threadIdx.x; i < n; i += gridDim.x * DRIFT_THREADS) {
        const size_t st = stg_index(stg, j, g.cap, i);
        drift_store(g, stg, st, j, stg.x[st], stg.y[st], stg.z[st], lam * stg.vx[st], lam * stg.vy[st],
                    lam * stg.vz[st], stg.fx[st], stg.fy[st], stg.fz[st], stg.id[st], out_cnt, err);
    }
}

// ------------------------------------------------------------------------------
// Bin pass 1: exclusive scan of the arrival counts of slot m -> cell_start; the
// counters become cursors.  One CTA per slot.
// ------------------------------------------------------------------------------
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_ITEMS = 4;                        // counters per thread per chunk
constexpr int SCAN_CHUNK = SCAN_THREADS * SCAN_ITEMS;

// Chunks of SCAN_CHUNK counters: coalesced load into shared memory, each thread scans
// SCAN_ITEMS consecutive ones, a block-wide scan of the thread sums, coalesced stores;
// the running total carries over to the next chunk.
__global__ void __launch_bounds__(SCAN_THREADS)
k_bin_scan(Geo g, BufView out, int m0, DevErr* err)
{
    pdl_wait();
    pdl_release();
    __shared__ int buf[SCAN_CHUNK];
    __shared__ int wsum[32];
    __shared__ int carry_s;
    const int m = m0 + blockIdx.x;
    int32_t* cnt = out.cnt + (size_t)m * g.ncell;
    int32_t* cs = slot_cs_w(out, m);
    const int n = g.ncell;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int carry = 0;
    for (int c0 = 0; c0 < n; c0 += SCAN_CHUNK) {
        const int len = min(SCAN_CHUNK, n - c0);
        for (int i = threadIdx.x; i < SCAN_CHUNK; i += SCAN_THREADS) buf[i] = i < len ? cnt[c0 + i] : 0;
        __syncthreads();
        int v[SCAN_ITEMS];
        int sum = 0;
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; k++) { v[k] = buf[threadIdx.x * SCAN_ITEMS + k]; sum += v[k]; }
        int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(FULLMASK, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const int w = wsum[lane];
            int iw = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(FULLMASK, iw, o);
                if (lane >= o) iw += u;
            }
            wsum[lane] = iw - w;
            if (lane == 31) carry_s = iw;   // chunk total
        }
        __syncthreads();
        int run = carry + wsum[warp] + incl - sum;
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; k++) { buf[threadIdx.x * SCAN_ITEMS + k] = run; run += v[k]; }
        __syncthreads();
        for (int i = threadIdx.x; i < len; i += SCAN_THREADS) {
            cs[c0 + i] = buf[i];
            cnt[c0 + i] = buf[i];
        }
        carry += carry_s;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        cs[n] = carry;
        if (carry > g.cap) set_err(err, DSEA_ECAPACITY, m, -1, carry);
    }
    if (out.remote) __threadfence_system();
}

// ------------------------------------------------------------------------------
// Bin pass 2: every staged atom whose destination slot is in [m0, m0+nm) takes a
// position in its cell (order within the cell fixed later by pass 3).
// ------------------------------------------------------------------------------
constexpr int PLACE_THREADS = 256;

__global__ void __launch_bounds__(PLACE_THREADS)
k_bin_place(Geo g, BufView out, StgView stg, int s0, int flat_count, int m0, int nm)
{
    pdl_wait();
    pdl_release();
    int base, n;
    if (flat_count > 0) { base = 0; n = flat_count; }
    else { const int s = s0 + blockIdx.y; base = wrap_slot(s + stg.soff, stg.pool) * g.cap; n = stg.n[s]; }
    const int p = blockIdx.x * PLACE_THREADS + threadIdx.x;
    const int lane = threadIdx.x & 31;
    int key = -1, m = 0;
    if (p < n) {
        key = stg.key[base + p];
        if (key >= 0) {
            m = key / g.ncell;
            if (m < m0 || m >= m0 + nm) key = -1;
        }
    }
    // warp-aggregated cursor: consecutive staged atoms come from one source cell and
    // mostly stay in one destination cell, so the lanes of a key share one atomicAdd
    // (their order within the cell is irrelevant: the gather ranks a cell by (z, id))
    const unsigned peers = __match_any_sync(FULLMASK, key >= 0 ? key : -2 - lane);
    const int leader = __ffs(peers) - 1;
    int pos = 0;
    if (key >= 0 && lane == leader)
        pos = atomicAdd(&out.cnt[(size_t)key], __popc(peers));   // key = m ncell + cell
    pos = __shfl_sync(FULLMASK, pos, leader) + __popc(peers & ((1u << lane) - 1u));
    if (key >= 0 && pos < g.cap) {
        // the sort keys travel with the index (coalesced reads here), so the gather
        // ranks a cell without a dependent round trip to staging
        BinRec r;
        r.z = stg.z[base + p];
        r.src = base + p;
        r.id = stg.id[base + p];
        out.perm[(size_t)wrap_slot(m + out.poff, out.perm_slots) * g.cap + pos] = r;
    }
}

// ------------------------------------------------------------------------------
// Bin pass 3: one half-warp per cell (cells hold ~13 atoms at rho 0.8, rc 2.5)
// ranks its arrivals by (z, id) -- a data-determined order, identical for every
// schedule -- and gathers them from staging into the slot; resets the cell's
// counter.  The records (z, src, id) come from k_bin_place; up to CM per cell are
// ranked in shared memory (rows padded against bank conflicts between the two
// half-warps), larger cells straight from the records in global memory.
// ------------------------------------------------------------------------------
constexpr int GATHER_THREADS = 256;
constexpr int GATHER_CELLS = GATHER_THREADS / 16;   // cells per CTA

// 32 registers = 8 CTAs of 256 threads per SM: the gather is latency-bound (a cell's
// records, then its staged atoms) and needs every resident warp.  A division on the
// slot path (wrap_slot) once took it to 64 registers and half the occupancy (1.8x slower).
template <int CM>
__global__ void __launch_bounds__(GATHER_THREADS)
k_bin_gather(Geo g, BufView out, StgView stg, int m0)
{
    pdl_wait();
    pdl_release();
    __shared__ double kz[GATHER_CELLS][CM + 1];
    __shared__ int kid[GATHER_CELLS][CM + 1];
    __shared__ int ksrc[GATHER_CELLS][CM + 1];
    const int sub = threadIdx.x & 15, hw = threadIdx.x >> 4;
    const unsigned hmask = 0xffffu << (threadIdx.x & 16);
    const int m = m0 + blockIdx.y;
    const int c = blockIdx.x * GATHER_CELLS + hw;
    if (c >= g.ncell) return;
    const int32_t* cs = slot_cs(out, m);
    const int st = cs[c], en = cs[c + 1];
    if (sub == 0) out.cnt[(size_t)m * g.ncell + c] = 0;
    if (cs[g.ncell] > g.cap) return;  // capacity error already flagged by the scan
    const int n = en - st;
    const BinRec* R = out.perm + (size_t)wrap_slot(m + out.poff, out.perm_slots) * g.cap + st;
    // one slot base in a register; the array offsets stay kernel parameters (10 live
    // 64-bit pointers would double the register count and halve the occupancy)
    char* const sb = out.base + (size_t)wrap_slot(m + out.soff, out.nslots) * out.L.slot_bytes;
    auto put = [&](int src, double z, int id, int rank) {
        const size_t d8 = (size_t)(st + rank) * sizeof(double);
        *reinterpret_cast<double*>(sb + out.L.off_x + d8) = stg.x[src];
        *reinterpret_cast<double*>(sb + out.L.off_y + d8) = stg.y[src];
        *reinterpret_cast<double*>(sb + out.L.off_z + d8) = z;
        *reinterpret_cast<double*>(sb + out.L.off_vx + d8) = stg.vx[src];
        *reinterpret_cast<double*>(sb + out.L.off_vy + d8) = stg.vy[src];
        *reinterpret_cast<double*>(sb + out.L.off_vz + d8) = stg.vz[src];
        *reinterpret_cast<double*>(sb + out.L.off_fx + d8) = stg.fx[src];
        *reinterpret_cast<double*>(sb + out.L.off_fy + d8) = stg.fy[src];
        *reinterpret_cast<double*>(sb + out.L.off_fz + d8) = stg.fz[src];
        *reinterpret_cast<int32_t*>(sb + out.L.off_id + (size_t)(st + rank) * sizeof(int32_t)) = id;
    };
    if (n <= CM) {
        for (int e = sub; e < n; e += 16) {
            const BinRec r = R[e];
            ksrc[hw][e] = r.src;
            kz[hw][e] = r.z;
            kid[hw][e] = r.id;
        }
        __syncwarp(hmask);
        for (int e = sub; e < n; e += 16) {
            const double z = kz[hw][e];
            const int id = kid[hw][e];
            int rank = 0;
            for (int e2 = 0; e2 < n; e2++) {
                const double z2 = kz[hw][e2];
                rank += (z2 < z) || (z2 == z && kid[hw][e2] < id);
            }
            put(ksrc[hw][e], z, id, rank);
        }
    } else {
        for (int e = sub; e < n; e += 16) {
            const BinRec r = R[e];
            int rank = 0;
            for (int e2 = 0; e2 < n; e2++) {
                const BinRec r2 = R[e2];
                rank += (r2.z < r.z) || (r2.z == r.z && r2.id < r.id);
            }
            put(r.src, r.z, r.id, rank);
        }
    }
    if (out.remote) __threadfence_system();
}

// ------------------------------------------------------------------------------
// Initial binning: key of every uploaded atom (flat staging), counted per cell.
// ------------------------------------------------------------------------------
__global__ void k_init_keys(Geo g, StgView stg, int n, int32_t* __restrict__ out_cnt, DevErr* err)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const double x = stg.x[p], y = stg.y[p], z = stg.z[p];
    if (!(x >= 0.0 && x <= g.b[0] && y >= 0.0 && y < g.b[1] && z >= 0.0 && z < g.b[2])) {
        set_err(err, DSEA_EINVAL, -1, stg.id[p], 0);
        stg.key[p] = -1;
        return;
    }
    const int cxg = cell_coord(x, g.l[0], g.cells[0]);
    const int cyg = cell_coord(y, g.l[1], g.cells[1]);
    const int czg = cell_coord(z, g.l[2], g.cells[2]);
    const int m = cxg / g.c;
    const int key = m * g.ncell + ((cxg - m * g.c) * g.cells[1] + cyg) * g.cells[2] + czg;
    stg.key[p] = key;
    atomicAdd(&out_cnt[key], 1);
}

// ------------------------------------------------------------------------------
// Host-facing conversions done on the device: by-id AoS arrays (the ABI layout) to
// staging SoA on upload, and slot SoA back to by-id AoS on read-back, so that the
// host only issues contiguous copies.
// ------------------------------------------------------------------------------
__global__ void k_aos_to_stage(StgView S, const double* __restrict__ xyz, const double* __restrict__ v,
                               const double* __restrict__ f, const int32_t* __restrict__ ids, int n)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    S.x[p] = xyz[3 * (size_t)p]; S.y[p] = xyz[3 * (size_t)p + 1]; S.z[p] = xyz[3 * (size_t)p + 2];
    S.vx[p] = v[3 * (size_t)p]; S.vy[p] = v[3 * (size_t)p + 1]; S.vz[p] = v[3 * (size_t)p + 2];
    if (f) { S.fx[p] = f[3 * (size_t)p]; S.fy[p] = f[3 * (size_t)p + 1]; S.fz[p] = f[3 * (size_t)p + 2]; }
    else { S.fx[p] = 0.0; S.fy[p] = 0.0; S.fz[p] = 0.0; }
    S.id[p] = ids ? ids[p] : p;
}

__global__ void k_slots_to_aos(Geo g, BufView in, int which, double* __restrict__ out,
                               unsigned long long* __restrict__ count)
{
    const int j = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = slot_cs(in, j)[g.ncell];
    const bool ok = i < n;
    if (ok) {
        const size_t o0 = which == 0 ? in.L.off_x : which == 1 ? in.L.off_vx : in.L.off_fx;
        const size_t o1 = which == 0 ? in.L.off_y : which == 1 ? in.L.off_vy : in.L.off_fy;
        const size_t o2 = which == 0 ? in.L.off_z : which == 1 ? in.L.off_vz : in.L.off_fz;
        const size_t id = (size_t)slot_i(in, j, in.L.off_id)[i];
        out[3 * id] = slot_d(in, j, o0)[i];
        out[3 * id + 1] = slot_d(in, j, o1)[i];
        out[3 * id + 2] = slot_d(in, j, o2)[i];
    }
    const unsigned b = __ballot_sync(FULLMASK, ok);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(count, (unsigned long long)__popc(b));
}

void aos_to_stage_launch(StgView S, const double* xyz, const double* v, const double* f, const int32_t* ids,
                         int n, cudaStream_t s)
{
    k_aos_to_stage<<<(n + 255) / 256, 256, 0, s>>>(S, xyz, v, f, ids, n);
}

void slots_to_aos_launch(const Geo& g, BufView in, int which, double* out, unsigned long long* count,
                         cudaStream_t s)
{
    dim3 grid((g.cap + 255) / 256, g.ns);
    k_slots_to_aos<<<grid, 256, 0, s>>>(g, in, which, out, count);
}

// ------------------------------------------------------------------------------
// Host-side launchers of the pipelined force kernel (A/B against k_force_tile,
// DSEA_FORCE=pipe) and of the bin / energy / helper kernels
// ------------------------------------------------------------------------------
static size_t pipe_smem_attr = 0;    // largest dynamic smem set on k_force_pipe so far

Tiling pipe_tiling(const Geo& g, double mean_per_cell, int smem_optin)
{
    Tiling T{};
    T.kind = FORCE_PIPE;
    T.maxh = (int)env_num("DSEA_MAXH", 64);
    const int CZ = g.cells[2];
    const double mean_col = mean_per_cell * CZ;               // atoms per column
    const double dens = mean_per_cell / g.l[2];                // atoms per sigma of column
    T.home = PIPE_HOME;
    T.nzt = std::max(1, (int)std::ceil(1.25 * mean_col / PIPE_HOME) + 1);
    T.tiles = g.c * g.cells[1] * T.nzt;
    const double per_col_p = std::min(mean_col + 2.0 * mean_per_cell,
                                      PIPE_HOME + (2.0 * g.rc + g.l[2]) * dens);
    const double expected_p = 9.0 * per_col_p + 18.0;
    T.smax = ((int)(env_num("DSEA_PIPE_MARGIN", 1.2) * expected_p + 64.0) + 31) / 32 * 32;
    while (T.smax > 32 && pipe_smem_bytes(T.smax, T.maxh) > (size_t)smem_optin) T.smax -= 32;
    if (T.smax > 65504) T.smax = 65504;
    T.smem = pipe_smem_bytes(T.smax, T.maxh);
    return T;
}

int pipe_kernel_attr(const Tiling& T)
{
    // the attribute is process-wide: keep the largest request of any context
    if (T.smem > pipe_smem_attr) {
        cudaError_t e = cudaFuncSetAttribute(k_force_pipe<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)T.smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_force_pipe<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)T.smem);
        if (e != cudaSuccess) return -1;
        pipe_smem_attr = T.smem;
    }
    int per_sm = 0, per_sm_nvt = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_force_pipe<2, false>, PIPE_THREADS, T.smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_nvt, k_force_pipe<2, true>, PIPE_THREADS, T.smem);
    return std::min(per_sm, per_sm_nvt);   // one grid size serves both instantiations
}

void pipe_launch(const Geo& g, const Tiling& T, BufView in, StgView stg, int32_t* out_cnt, int j0, int nj,
                 DevErr* err, cudaStream_t s)
{
    // the tile counter is never reset: each launch consumes exactly ntiles + grid
    // increments, so the host tracks the base of every launch
    // NVE: force + kick + drift + destination in one pass; NVT: force + kick (the
    // drift needs the slice's lambda, k_drift)
    if (g.thermo)
        launch(k_force_pipe<2, true>, T.grid, PIPE_THREADS, T.smem, s, g, T, in, stg, out_cnt, j0, nj, err,
               T.ctr, *T.ctr_base);
    else
        launch(k_force_pipe<2, false>, T.grid, PIPE_THREADS, T.smem, s, g, T, in, stg, out_cnt, j0, nj, err,
               T.ctr, *T.ctr_base);
    *T.ctr_base += (unsigned long long)nj * T.tiles + T.grid;
}

// Ring-hop signal (peer backend): after the bin kernels wrote slots [first, first+n)
// straight into the successor's input buffer over NVLink, publish their arrival
// count in the successor's flag array (or a release count in the predecessor's).
__global__ void k_signal(uint32_t* __restrict__ flags, int first, int n, uint32_t value)
{
    pdl_wait();
    pdl_release();
    __threadfence_system();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        volatile uint32_t* f = flags + first + i;
        *f = value;
    }
    __threadfence_system();
}

void signal_launch(uint32_t* flags, int first, int n, uint32_t value, cudaStream_t s)
{
    launch(k_signal, 1, 64, 0, s, flags, first, n, value);
}

size_t energy_records(const Geo& g, const Tiling& T)
{
    return T.kind == FORCE_PIPE ? (size_t)g.ns * g.cap : (size_t)g.ns * T.tiles;
}

void energy_launch(const Geo& g, const Tiling& T, StgView stg, int j0, int nj, UnitEnergy* e_out, cudaStream_t s)
{
    // records of slice j: one per tile (k_force_tile) or one per staged atom (k_force_pipe)
    const int stride = T.kind == FORCE_PIPE ? g.cap : T.tiles;
    launch(k_energy, nj, ENERGY_THREADS, 0, s, g, stg, j0, stride, T.kind == FORCE_PIPE ? 0 : T.tiles, e_out);
}

void drift_launch(const Geo& g, StgView stg, int j0, int nj, const UnitEnergy* e_out, int32_t* out_cnt,
                  DevErr* err, cudaStream_t s)
{
    dim3 grid((unsigned)std::max(1, std::min((g.cap + DRIFT_THREADS - 1) / DRIFT_THREADS, 64)), (unsigned)nj);
    launch(k_drift, grid, DRIFT_THREADS, 0, s, g, stg, j0, e_out, out_cnt, err);
}

void bin_scan_launch(const Geo& g, BufView out, int m0, int nm, DevErr* err, cudaStream_t s)
{
    launch(k_bin_scan, nm, SCAN_THREADS, 0, s, g, out, m0, err);
}

void bin_place_launch(const Geo& g, BufView out, StgView stg, int s0, int nsrc, int flat_count,
                      int m0, int nm, DevErr* err, cudaStream_t s)
{
    (void)err;
    if (flat_count > 0) {
        dim3 grid((flat_count + PLACE_THREADS - 1) / PLACE_THREADS, 1);
        launch(k_bin_place, grid, PLACE_THREADS, 0, s, g, out, stg, 0, flat_count, m0, nm);
    } else {
        dim3 grid((g.cap + PLACE_THREADS - 1) / PLACE_THREADS, nsrc);
        launch(k_bin_place, grid, PLACE_THREADS, 0, s, g, out, stg, s0, 0, m0, nm);
    }
}

void bin_gather_launch(const Geo& g, BufView out, StgView stg, int m0, int nm, DevErr* err,
                       cudaStream_t s)
{
    (void)err;
    dim3 grid((g.ncell + GATHER_CELLS - 1) / GATHER_CELLS, nm);
    if (g.cell_max <= 32) launch(k_bin_gather<32>, grid, GATHER_THREADS, 0, s, g, out, stg, m0);
    else if (g.cell_max <= 64) launch(k_bin_gather<64>, grid, GATHER_THREADS, 0, s, g, out, stg, m0);
    else launch(k_bin_gather<128>, grid, GATHER_THREADS, 0, s, g, out, stg, m0);
}

void init_keys_launch(const Geo& g, StgView stg, int n, int32_t* out_cnt, DevErr* err,
                      cudaStream_t s)
{
    k_init_keys<<<(n + 255) / 256, 256, 0, s>>>(g, stg, n, out_cnt, err);
}

}  // namespace dsea
