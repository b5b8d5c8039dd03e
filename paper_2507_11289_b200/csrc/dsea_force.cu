// dsea_force.cu -- k_force_tile, the default force kernel of the DSEAmd hot path
// (arXiv 2507.11289): md_v3a + stat_collect (§4.1, Algorithm 1 force loop
// P:257-271), fused with md_v3aa (velocity update) and the position update
// and destination decision of md_v3b for the atoms of slices
// [j0, j0 + nj), each reading its left and right neighbour slices (O_in = 1).
//
// A tile is up to TILE_ATOMS consecutive, z-sorted home atoms of one (cx, cy) column of
// slice j.  Persistent CTAs (2 of 8 warps per SM at rho 0.8, rc 2.5) claim tiles from a
// counter; per tile:
//   1. a piece table: 9 neighbour columns x {low z-image, main run, high z-image}, the
//      cells within one cell (l >= rc) of the home atoms' cells (periodic images in y
//      and z pre-shifted, x walls: absent columns, readings Q1/Q2).  The first
//      warp out of chunks builds the NEXT tile's table while the others still work on
//      the current one, so the dependent cell_start loads never stall the CTA;
//   2. all warps stage the pieces into shared memory twice: FP64 (x, y, z) for the exact
//      pair work and an FP32 screening record (x, y, z, w = x^2+y^2+z^2) relative to the
//      tile centre, two atoms per 32 bytes so that one pair of LDS.128 feeds a packed
//      FFMA2 test of two candidates;
//   3. warps claim 16-atom chunks.  Lane (il, par) screens every other candidate pair of
//      the chunk's z-window in each column against atom il with the dot form
//      |ri - rj|^2 - |ri|^2 = wj - 2 ri.rj  <=  rc^2 + margin - wi  (3 FFMA2 per two
//      candidates) and appends survivors to the atom's two-ended hit list; the two lanes
//      of an atom then evaluate half of the list each, exactly in FP64 with the inclusive
//      test r^2 <= rc^2;
//   4. lane (il, 0) kicks, drifts, mirrors/wraps and keys its atom.
// Energies are summed per chunk (fixed xor tree), per tile in chunk order and per slice
// in tile order by k_energy: every sum has a fixed order that depends only on the input
// slots, so results are bitwise reproducible across launches, schedules and GPU counts.
// No tensor cores: this is not a dense contraction.
#include <algorithm>
#include <string>
#include "dsea_device.cuh"

namespace dsea {

#ifndef DSEA_TILE_WARPS
#define DSEA_TILE_WARPS 8   // measured (C4 force): 4 warps 8.82 ms, 8 warps + 128-row lists 8.59 ms, 16 warps 9.70 ms
#endif
#ifndef DSEA_TILE_ILP
#define DSEA_TILE_ILP 2
#endif
#ifndef DSEA_TILE_LM
#define DSEA_TILE_LM 128
#endif
constexpr int TILE_WARPS = DSEA_TILE_WARPS;
constexpr int TILE_THREADS = 32 * TILE_WARPS;
constexpr int TILE_HOME = 16 * TILE_WARPS;      // home atoms in flight: one 16-atom chunk per warp
#ifndef DSEA_TILE_CHUNKS
#define DSEA_TILE_CHUNKS TILE_WARPS
#endif
constexpr int TILE_CHUNKS = DSEA_TILE_CHUNKS;   // 16-atom chunks per tile (claimed by the warps)
constexpr int TILE_ATOMS = 16 * TILE_CHUNKS;    // home atoms per (sub)tile
constexpr int TILE_ILP = DSEA_TILE_ILP;         // hits in flight per lane in the FP64 pass
constexpr int TILE_LM = DSEA_TILE_LM;           // hit-list rows per home atom (shared by its two lanes)
#ifndef DSEA_ROWPAD
#define DSEA_ROWPAD 16  // row stride 2*TILE_HOME + 16 bytes: rows rotate the banks (C4: pad 4 8.48 ms, 8 8.44, 16 8.42)
#endif
#ifndef DSEA_STAGE_SHFL
#define DSEA_STAGE_SHFL 1
#endif
#ifndef DSEA_STAGE_SU
#define DSEA_STAGE_SU 4  // staged atoms per thread whose loads are in flight together (8: 0.3 % slower)
#endif
constexpr int TILE_ROW = 2 * TILE_HOME + DSEA_ROWPAD;   // bytes per hit-list row (the pad rotates the banks)

// The piece table of one (sub)tile, built by warp 0 one step ahead.
struct TileTable {
    int valid;                                  // 0: no more tiles for this CTA
    int ok;                                     // 0: not even one home atom fits (ECAPACITY)
    int t;                                      // flat tile index (slice j0 + t / tiles)
    int hb, he, h1;                             // home range [hb, he) of the tile [.., h1)
    int total, self_base;                       // staged atoms; staging index of atom hb
    int pt_dst[27], pt_end[27];                 // piece p occupies staging [pt_dst, pt_end)
    const double* pt_x[27];                     // source x of the piece (y, z at fixed offsets)
    double pt_dy[27], pt_dz[27];                // periodic image shifts
    int c_lo[9], c_hi[9];                       // column runs (c_hi before the even padding)
    double ox, oy, oz;                          // tile centre (origin of the FP32 records)
};

size_t tile_smem_bytes(int smax)
{
    return (size_t)TILE_LM * TILE_ROW + 16 + (size_t)smax * (3 * sizeof(double) + 16) + 256;
}

// hit-list traffic through explicit shared-window addresses (volatile: kept in program
// order with each other and with the warp barriers that separate appends from reads)
__device__ __forceinline__ void sts_u16(unsigned a, int v)
{
    asm volatile("{\n\t.reg .b16 t;\n\tcvt.u16.u32 t, %1;\n\tst.shared.u16 [%0], t;\n\t}" ::"r"(a), "r"(v));
}
__device__ __forceinline__ int lds_u16(unsigned a)
{
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds_f64(unsigned a)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

// Warp 0: the table of the home range starting at atom hb of flat tile t (hb < 0: a new
// tile), skipping empty tiles (whose energy records are zero).  The home atoms' cells
// come from the column's cell_start (no position loads); the range is halved until its
// neighbourhood fits the staging capacity.
__device__ void build_table(const Geo& g, const Tiling& T, const BufView& in, const StgView& stg, int j0,
                            long long ntiles, int t, int hb, TileTable& A,
                            unsigned long long* __restrict__ tile_ctr, unsigned long long ctr_base)
{
    const int lane = threadIdx.x & 31;
    const int CY = g.cells[1], CZ = g.cells[2];
    int j = 0, tile = 0, cxl = 0, cyi = 0, h1 = 0, colbase_h = 0;
    const int32_t* csj = nullptr;
    for (;;) {
        if (hb < 0) {   // a new tile: claimed from the launch's counter (CTAs that start late
                        // -- SMs busy with other kernels -- simply take fewer tiles)
            unsigned long long c = 0;
            if (lane == 0) c = atomicAdd(tile_ctr, 1ull) - ctr_base;
            c = __shfl_sync(FULLMASK, c, 0);
            t = c >= (unsigned long long)ntiles ? (int)ntiles : (int)c;
        }
        if (t >= ntiles) {
            if (lane == 0) A.valid = 0;
            return;
        }
        j = j0 + t / T.tiles;
        tile = t % T.tiles;
        const int tt = tile % T.nzt, rest = tile / T.nzt;
        cyi = rest % CY;
        cxl = rest / CY;
        csj = slot_cs(in, j);
        colbase_h = (cxl * CY + cyi) * CZ;
        if (tile == 0 && lane == 0) stg.n[j] = csj[g.ncell];
        const int col_first = csj[colbase_h], col_end = csj[colbase_h + CZ];
        const int h0 = col_first + tt * T.home;
        h1 = (tt == T.nzt - 1) ? col_end : min(col_end, h0 + T.home);
        if (hb < 0) hb = h0;
        if (hb < h1) break;
        if (lane == 0) stg.eatom[(size_t)j * T.tiles + tile] = make_double4(0.0, 0.0, 0.0, 0.0);
        hb = -1;
    }
    // cell (along z) of home atom a: the number of cells c >= 1 of the column with
    // cell_start <= a
    auto cell_of = [&](int a) {
        int n = 0;
        for (int c = 1 + lane; c < CZ; c += 32) n += (csj[colbase_h + c] <= a);
        return __reduce_add_sync(FULLMASK, n);
    };
    const int czb = cell_of(hb);
    int he = min(h1, hb + TILE_ATOMS);
    int cnt = 0, start = 0, src_slice = 0, excl = 0, total = 0, cze = 0;
    double dyv = 0.0, dzv = 0.0;
    bool ok = true;
    for (;;) {
        cze = cell_of(he - 1);
        const int z0 = czb - 1, z1 = cze + 1;   // l_z >= rc: one cell on each side suffices
        cnt = 0; start = 0; src_slice = 0; dyv = 0.0; dzv = 0.0;
        if (lane < 27) {
            const int col = lane / 3, qq = lane % 3;
            const int dxk = col / 3 - 1, dyk = col % 3 - 1;
            const int gx = j * g.c + cxl + dxk;
            if (gx >= 0 && gx < g.cells[0]) {       // x walls: no column beyond (Q2)
                const int m = gx / g.c, cx2 = gx - m * g.c;
                int cyy = cyi + dyk;                 // y periodic (Q1)
                if (cyy < 0) { cyy += CY; dyv = -g.b[1]; }
                else if (cyy >= CY) { cyy -= CY; dyv = g.b[1]; }
                const int zlo = max(z0, -1), zhi = min(z1, CZ);
                int a0 = 0, b0 = -1;                 // z periodic: low image, main, high image
                if (qq == 0) { if (zlo < 0) { a0 = zlo + CZ; b0 = CZ - 1; dzv = -g.b[2]; } }
                else if (qq == 1) { a0 = max(zlo, 0); b0 = min(zhi, CZ - 1); }
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
        // each column starts at an even staging index: its last piece carries the pad
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
        if (he - hb <= 1) { ok = false; break; }
        he = hb + (he - hb > 32 ? (((he - hb) / 2 + 15) & ~15) : (he - hb) / 2);
    }
    if (lane < 27) {
        A.pt_dst[lane] = excl;
        A.pt_end[lane] = excl + cnt;
        A.pt_x[lane] = slot_d(in, src_slice, in.L.off_x) + start;
        A.pt_dy[lane] = dyv;
        A.pt_dz[lane] = dzv;
    }
    // column `lane` = pieces 3 lane .. 3 lane + 2 (piece 13 = the home column's main run)
    const int cl = __shfl_sync(FULLMASK, excl, min(3 * lane, 31));
    const int chh = __shfl_sync(FULLMASK, excl + cnt, min(3 * lane + 2, 31));
    if (lane < 9) { A.c_lo[lane] = cl; A.c_hi[lane] = chh; }
    const int main_dst = __shfl_sync(FULLMASK, excl, 13), main_start = __shfl_sync(FULLMASK, start, 13);
    if (lane == 0) {
        A.valid = 1;
        A.ok = ok ? 1 : 0;
        A.t = t;
        A.hb = hb;
        A.he = he;
        A.h1 = h1;
        A.total = total;
        A.self_base = main_dst + (hb - main_start);
        A.ox = ((double)(j * g.c + cxl) + 0.5) * g.l[0];
        A.oy = ((double)cyi + 0.5) * g.l[1];
        A.oz = 0.5 * (double)(czb + cze + 1) * g.l[2];
    }
}

#ifndef DSEA_ABL
#define DSEA_ABL 0     // ablation builds for timing studies only (1: no pair work, 2: no FP64 pass)
#endif

#ifndef DSEA_TILE_MINB
#define DSEA_TILE_MINB (16 / TILE_WARPS)   // resident CTAs per SM the registers must allow
#endif

template <bool NVT>
__global__ void __launch_bounds__(TILE_THREADS, DSEA_TILE_MINB)
k_force_tile(Geo g, Tiling T, BufView in, StgView stg, int32_t* __restrict__ out_cnt, int j0, int nj,
             DevErr* __restrict__ err, unsigned long long* __restrict__ tile_ctr, unsigned long long ctr_base)
{
    pdl_wait();
    pdl_release();
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ TileTable TT[2];
    __shared__ double4 s_ce[TILE_CHUNKS];       // chunk energy records of the current sub-tile
    __shared__ int s_chunk;                     // next chunk to claim
    __shared__ int s_tbl;                       // the next table has a builder
    // dynamic shared memory (byte offsets from the host: a base ptxas sees as a constant
    // is rematerialised with S2R/LEA at every hit-list append instead of kept in a register):
    //   off_hl   u16 hit lists [TILE_LM] rows of TILE_ROW bytes (2 per home atom)
    //   off_sp   FP64 staged positions [smax][3]
    //   off_q    FP32 screening records [smax/2 + 8][8]: x0 x1 y0 y1 z0 z1 w0 w1 (the
    //            tail pairs read past a window's end are masked)
    double* sp = reinterpret_cast<double*>(smem + T.off_sp);
    float* qf = reinterpret_cast<float*>(smem + T.off_q);
    const float4* q4 = reinterpret_cast<const float4*>(qf);
    float4* q4w = reinterpret_cast<float4*>(qf);   // pair p: [2p] = x0 x1 y0 y1, [2p+1] = z0 z1 w0 w1
    uint16_t* hl = reinterpret_cast<uint16_t*>(smem + T.off_hl);
#define spd(k, d) sp[3 * (k) + (d)]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long ntiles = (long long)nj * T.tiles;
    const size_t yoff = (in.L.off_y - in.L.off_x) / sizeof(double);
    const size_t zoff = (in.L.off_z - in.L.off_x) / sizeof(double);
    double e_u = 0.0, e_v = 0.0, e_k = 0.0, e_n = 0.0;         // tile record (thread 0)

    if (warp == 0) build_table(g, T, in, stg, j0, ntiles, 0, -1, TT[0], tile_ctr, ctr_base);
    __syncthreads();
    for (int cur = 0;; cur ^= 1) {
        const TileTable& A = TT[cur];
        if (!A.valid) break;
        if (!A.ok) {
            if (tid == 0) set_err(err, DSEA_ECAPACITY, j0 + A.t / T.tiles, -1, A.total);
            break;
        }
        const int j = j0 + A.t / T.tiles;
        const int hb = A.hb, nhome = A.he - hb, total = A.total, self_base = A.self_base;

        // ---- 2. stage the 27 pieces: FP64 positions + packed FP32 screening records ----
        {
            // rounds of SU items per thread: all loads of a round are issued before any is
            // used; warp-wide items (total is even): lanes 2q, 2q+1 hold the atoms of one
            // candidate pair and trade halves so that each writes one 16-byte record
            const double ox = A.ox, oy = A.oy, oz = A.oz;
            constexpr int SU = DSEA_STAGE_SU;
            int col = 0;
            for (int i0 = tid; i0 - lane < total; i0 += SU * TILE_THREADS) {
                double x[SU], y[SU], z[SU];
                bool real[SU];
#pragma unroll
                for (int u = 0; u < SU; u++) {
                    const int i = i0 + u * TILE_THREADS;
                    x[u] = 0.0; y[u] = 0.0; z[u] = 0.0; real[u] = false;
                    if (i < total) {
                        while (col < 8 && i >= A.pt_dst[3 * col + 3]) col++;
                        const int p = 3 * col + (i >= A.pt_dst[3 * col + 1]) + (i >= A.pt_dst[3 * col + 2]);
                        if (i < A.pt_end[p]) {
                            const double* px = A.pt_x[p] + (i - A.pt_dst[p]);
                            x[u] = __ldg(px);
                            y[u] = __ldg(px + yoff) + A.pt_dy[p];
                            z[u] = __ldg(px + zoff) + A.pt_dz[p];
                            real[u] = true;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < SU; u++) {
                    const int i = i0 + u * TILE_THREADS;
                    if (i - lane >= total) break;               // warp-uniform
                    float rx = 0.f, ry = 0.f, rz = 0.f, w = 1e30f;  // even padding: never passes the screen
                    if (real[u]) {
                        rx = (float)(x[u] - ox); ry = (float)(y[u] - oy); rz = (float)(z[u] - oz);
                        w = fmaf(rx, rx, fmaf(ry, ry, rz * rz));
                    }
                    if (i < total) { sp[3 * i] = x[u]; sp[3 * i + 1] = y[u]; sp[3 * i + 2] = z[u]; }
#if DSEA_STAGE_SHFL
                    const bool odd = lane & 1;
                    const float a = __shfl_xor_sync(FULLMASK, odd ? rx : rz, 1);   // even gets x1, odd z0
                    const float b = __shfl_xor_sync(FULLMASK, odd ? ry : w, 1);    // even gets y1, odd w0
                    if (i < total)
                        q4w[i] = odd ? make_float4(a, rz, b, w) : make_float4(rx, a, ry, b);
#else
                    if (i < total) {
                        const int qb = 8 * (i >> 1) + (i & 1);
                        qf[qb] = rx; qf[qb + 2] = ry; qf[qb + 4] = rz; qf[qb + 6] = w;
                    }
#endif
                }
            }
        }
        if (tid == 0) { s_chunk = 0; s_tbl = 0; }
        __syncthreads();

        // ---- 3./4. chunks: screen, pooled FP64 pair work, integration -------------------
        const int nchunks = DSEA_ABL == 1 ? 0 : (nhome + 15) >> 4;
        for (;;) {
            int chv = 0;
            if (lane == 0) chv = atomicAdd(&s_chunk, 1);
            const int ch = __shfl_sync(FULLMASK, chv, 0);
            if (ch >= nchunks) break;
            const int il = lane & 15, par = lane >> 4;
            const int q = ch * 16 + il;
            const bool valid = q < nhome;
            const int si = self_base + (valid ? q : nhome - 1);
            const int qbi = 8 * (si >> 1) + (si & 1);
            const float xf = qf[qbi], yf = qf[qbi + 2], zf = qf[qbi + 4], wf = qf[qbi + 6];
            const float thr = valid ? g.rc2_screen - wf : -1e30f;
            const float2 ax = make_float2(-2.f * xf, -2.f * xf);
            const float2 ay = make_float2(-2.f * yf, -2.f * yf);
            const float2 az = make_float2(-2.f * zf, -2.f * zf);
            const double xi = spd(si, 0), yi = spd(si, 1), zi = spd(si, 2);
            const double rc2 = g.rc2;
            // the chunk's z-window in each column (binary searches on the FP64 z, in
            // parallel: lanes 0-8 lower ends, lanes 16-24 upper ends), pair-aligned
            int wb = 0;
            {
                const double zmin = spd(self_base + ch * 16, 2);
                const double zmax = spd(self_base + min(ch * 16 + 16, nhome) - 1, 2);
                if (lane < 9 || (lane >= 16 && lane < 25)) {
                    const int col = lane < 9 ? lane : lane - 16;
                    int lo = A.c_lo[col], hi = A.c_hi[col];
                    const int base = lo;
                    if (lane < 9) {
                        const double key = zmin - g.rc - 1e-9;
                        while (lo < hi) { const int mid = (lo + hi) >> 1; if (spd(mid, 2) < key) lo = mid + 1; else hi = mid; }
                        wb = base + ((lo - base) & ~1);
                    } else {
                        const double key = zmax + g.rc + 1e-9;
                        while (lo < hi) { const int mid = (lo + hi) >> 1; if (spd(mid, 2) <= key) lo = mid + 1; else hi = mid; }
                        wb = base + ((lo - base + 1) & ~1);
                    }
                }
            }
            double fx = 0.0, fy = 0.0, fz = 0.0, sa = 0.0, sb = 0.0;   // sa = sum s6^2, sb = sum s6
            int np = 0;
            // hit list of home atom a = (16 warp + il) of the chunk slots: row r at byte
            // hls + r ROW + 2 a of the shared window (explicit 32-bit shared addresses: one
            // add per access); lane (il, 0) fills rows 0, 1, ... and lane (il, 1) rows
            // M-1, M-2, ... of the same list
            constexpr int ROW = TILE_ROW;
            const int M = T.maxh;                       // rows in use (<= TILE_LM; tests shrink it)
            const unsigned hls = (unsigned)__cvta_generic_to_shared(hl);
            const int hla = 2 * (warp * 16 + il);
            const int ho0 = hla + (par ? (M - 1) * ROW : 0);
            const int step = par ? -ROW : ROW;
            int ho = ho0;                               // this lane's next free entry

            // exact FP64 pair term of Algorithm 1 for the staged atom at byte
            // offset ko = 24 k of the FP64 staging
            const unsigned sps = (unsigned)__cvta_generic_to_shared(sp);
            const int sio = 24 * si;
            auto pair = [&](const int ko) {
                const double dx = xi - lds_f64(sps + ko);
                const double dy = yi - lds_f64(sps + ko + 8);
                const double dz = zi - lds_f64(sps + ko + 16);
                const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
                const bool ok = (r2 <= rc2) && (ko != sio);     // inclusive cutoff, i != j
                // a rejected candidate continues with r^2 = 1e300: every power below
                // underflows to 0, so it adds exactly nothing (no select on the results)
                const double s = rcp64(ok ? r2 : 1e300);
                const double s2 = s * s;
                const double s3 = s2 * s;                       // r^-6
                const double s4 = s2 * s2;
                const double f = s4 * (s3 - 0.5);              // F_abs / 48 = r^-2 (r^-12 - r^-6 / 2)
                fx = fma(dx, f, fx);
                fy = fma(dy, f, fy);
                fz = fma(dz, f, fz);
                sa = fma(s3, s3, sa);
                sb += s3;
                if (ok) np++;
            };
            // the two lanes of an atom take half of its list each: entry v of the list is
            // row v (v < c0, lane (il, 0)'s hits) or row M - 1 - (v - c0) (lane (il, 1)'s)
            auto flush = [&]() {
                __syncwarp();
                if (DSEA_ABL == 2) { ho = ho0; return; }
                const int c = (ho - ho0) / step;
                const int cp = __shfl_xor_sync(FULLMASK, c, 16);
                const int c0 = par ? cp : c;
                const int tot = c0 + (par ? c : cp);
                const int h = (tot + 1) >> 1;
                const int lo = par ? h : 0, hi = par ? tot : h;
                const unsigned ha = hls + hla;                   // entry v < c0 at ha + v ROW
                const unsigned hbb = ha + (M - 1 + c0) * ROW;    // entry v >= c0 at hbb - v ROW
                for (int e = lo; e < hi; e += TILE_ILP) {
                    int kk[TILE_ILP];
#pragma unroll
                    for (int u = 0; u < TILE_ILP; u++) {
                        const int eu = e + u;
                        kk[u] = eu < hi ? lds_u16(eu < c0 ? ha + eu * ROW : hbb - eu * ROW) : sio;
                    }
#pragma unroll
                    for (int u = 0; u < TILE_ILP; u++) pair(kk[u]);
                }
                __syncwarp();
                ho = ho0;
            };
            // wj - 2 ri.rj for candidates k, k+1 (P = x0 x1 y0 y1, Q = z0 z1 w0 w1); a hit
            // appends the candidate's FP64 staging offset 24 k
            auto test = [&](const float4 P, const float4 Q, const int ko) {   // ko = 24 k
                float2 tq = __ffma2_rn(make_float2(P.x, P.y), ax, make_float2(Q.z, Q.w));
                tq = __ffma2_rn(make_float2(P.z, P.w), ay, tq);
                tq = __ffma2_rn(make_float2(Q.x, Q.y), az, tq);
                if (tq.x <= thr) { sts_u16(hls + ho, ko); ho += step; }
                if (tq.y <= thr) { sts_u16(hls + ho, ko + 24); ho += step; }
            };

            for (int col = 0; col < 9; col++) {
                const int plo = __shfl_sync(FULLMASK, wb, col) >> 1;
                const int phi = __shfl_sync(FULLMASK, wb, 16 + col) >> 1;
                // spans of at most M/4 pairs (both lanes append at most M/2 entries); before
                // a span whose appends might not fit, flush.  The decision depends only on
                // the chunk's data (never on which warp took it)
                for (int s0 = plo; s0 < phi; s0 += M / 4) {
                    const int e = min(phi, s0 + M / 4);
                    const int hp = __shfl_xor_sync(FULLMASK, ho, 16);
                    if (__any_sync(FULLMASK, 2 * (e - s0) > (par ? ho - hp : hp - ho) / ROW + 1)) flush();
                    int m = s0 + par;
                    for (; m + 6 < e; m += 8) {         // 4 pairs, loads first
                        const float4 P0 = q4[2 * m], Q0 = q4[2 * m + 1];
                        const float4 P1 = q4[2 * m + 4], Q1 = q4[2 * m + 5];
                        const float4 P2 = q4[2 * m + 8], Q2 = q4[2 * m + 9];
                        const float4 P3 = q4[2 * m + 12], Q3 = q4[2 * m + 13];
                        const int ko = 48 * m;
                        test(P0, Q0, ko);
                        test(P1, Q1, ko + 96);
                        test(P2, Q2, ko + 192);
                        test(P3, Q3, ko + 288);
                    }
                    for (; m < e; m += 2) test(q4[2 * m], q4[2 * m + 1], 48 * m);
                }
            }
            flush();
            // combine the two lanes of each atom (commutative: both get the same value)
            fx += __shfl_xor_sync(FULLMASK, fx, 16);
            fy += __shfl_xor_sync(FULLMASK, fy, 16);
            fz += __shfl_xor_sync(FULLMASK, fz, 16);
            double ke2 = 0.0;
            if (valid && par == 0) {
                const int gi = hb + q;
                const double fxo = __ldg(slot_d(in, j, in.L.off_fx) + gi);
                const double fyo = __ldg(slot_d(in, j, in.L.off_fy) + gi);
                const double fzo = __ldg(slot_d(in, j, in.L.off_fz) + gi);
                const double vx0 = __ldg(slot_d(in, j, in.L.off_vx) + gi);
                const double vy0 = __ldg(slot_d(in, j, in.L.off_vy) + gi);
                const double vz0 = __ldg(slot_d(in, j, in.L.off_vz) + gi);
                const int aid = __ldg(slot_i(in, j, in.L.off_id) + gi);
                const double Fx = 48.0 * fx, Fy = 48.0 * fy, Fz = 48.0 * fz;
                const double hdt = 0.5 * g.dt;
                const double vx = vx0 + (Fx + fxo) * hdt;
                const double vy = vy0 + (Fy + fyo) * hdt;
                const double vz = vz0 + (Fz + fzo) * hdt;
                ke2 = vx * vx + vy * vy + vz * vz;
                const size_t st = stg_index(stg, j, g.cap, gi);
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
            // chunk energies: fixed xor tree
            double pn = (double)np;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                sa += __shfl_xor_sync(FULLMASK, sa, o);
                sb += __shfl_xor_sync(FULLMASK, sb, o);
                ke2 += __shfl_xor_sync(FULLMASK, ke2, o);
                pn += __shfl_xor_sync(FULLMASK, pn, o);
            }
            // u_core = sum s6 (s6 - 1), vir2 = sum s6 (2 s6 - 1)
            if (lane == 0) s_ce[ch] = make_double4(sa - sb, 2.0 * sa - sb, ke2, pn);
        }
        // ---- 1'. the next table: built by the first warp out of chunks, overlapping the
        // others' pair work (which warp builds it does not change its contents)
        {
            int own = 0;
            if (lane == 0) own = atomicExch(&s_tbl, 1) == 0;
            if (__shfl_sync(FULLMASK, own, 0))
                build_table(g, T, in, stg, j0, ntiles, A.t, A.he < A.h1 ? A.he : -1, TT[cur ^ 1], tile_ctr,
                            ctr_base);
        }
        __syncthreads();
        if (tid == 0) {
            for (int c = 0; c < nchunks; c++) {        // chunk order: independent of the warps
                const double4 r = s_ce[c];
                e_u += r.x; e_v += r.y; e_k += r.z; e_n += r.w;
            }
            if (A.he >= A.h1) {                         // the tile's last sub-tile: its record
                stg.eatom[(size_t)j * T.tiles + A.t % T.tiles] = make_double4(e_u, e_v, e_k, e_n);
                e_u = e_v = e_k = e_n = 0.0;
            }
        }
    }
#undef spd
}

// ------------------------------------------------------------------------------
// Host side: tiling choice and launch (both force kernels)
// ------------------------------------------------------------------------------
static size_t tile_smem_attr = 0;   // largest dynamic smem set on k_force_tile so far

static int tile_static_smem()
{
    cudaFuncAttributes a{};
    if (cudaFuncGetAttributes(&a, k_force_tile<false>) != cudaSuccess) return 2048;
    return (int)a.sharedSizeBytes;
}

Tiling choose_tiling(const Geo& g, double mean_per_cell, int smem_optin)
{
    const char* kind = getenv("DSEA_FORCE");
    if (kind && std::string(kind) == "pipe") return pipe_tiling(g, mean_per_cell, smem_optin);
    Tiling T{};
    T.kind = FORCE_TILE;
    T.home = TILE_ATOMS;
    T.maxh = std::max(8, std::min(TILE_LM, (int)env_num("DSEA_MAXH", TILE_LM)));
    const int CZ = g.cells[2];
    const double mean_col = mean_per_cell * CZ;                // atoms per column
    const double dens = mean_per_cell / g.l[2];                 // atoms per sigma of column
    T.nzt = std::max(1, (int)std::ceil(1.1 * mean_col / TILE_ATOMS) + 1);
    T.tiles = g.c * g.cells[1] * T.nzt;
    // staged atoms of a full tile: 9 columns x (home extent + 2 rc + a partial cell)
    auto staged = [&](int home) {
        const double per_col = std::min(mean_col + 2.0 * mean_per_cell, home + (2.0 * g.rc + g.l[2]) * dens);
        return 9.0 * per_col + 18.0;
    };
    // as many resident CTAs per SM as the staging of a full tile allows (16 / TILE_WARPS:
    // 2 CTAs of 8 warps at rho 0.8, rc 2.5); denser or longer-ranged workloads get fewer,
    // larger CTAs
    int per_sm_smem = 233472;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&per_sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    const int stat = tile_static_smem();
    const int want = ((int)(env_num("DSEA_TILE_MARGIN", 1.1) * staged(TILE_ATOMS) + 64.0) + 31) / 32 * 32;
    const int need16 = ((int)(1.3 * staged(8) + 64.0) + 31) / 32 * 32;    // a small sub-tile
    for (int per_sm = (int)env_num("DSEA_TILE_CTAS", 16 / TILE_WARPS); per_sm >= 1; per_sm--) {
        const long budget = (long)per_sm_smem / per_sm - 1024 - stat;
        const long fixed = (long)TILE_LM * TILE_ROW + 16 + 256;
        int cap = (int)((budget - fixed) / 40) / 32 * 32;
        cap = std::min(cap, (int)((smem_optin - fixed) / 40) / 32 * 32);
        if (cap >= need16 || per_sm == 1) {
            T.smax = std::min(want, cap);
            break;
        }
    }
    T.smax = std::min(std::max(T.smax, 64), 2720);     // hit lists hold 24 k in 16 bits
    T.smem = tile_smem_bytes(T.smax);
    T.off_hl = 0;
    T.off_sp = (TILE_LM * TILE_ROW + 15) / 16 * 16;
    T.off_q = T.off_sp + 24 * T.smax;
    return T;
}

int force_kernel_attr(const Tiling& T)
{
    if (T.kind == FORCE_PIPE) return pipe_kernel_attr(T);
    if (T.smem > tile_smem_attr) {
        cudaError_t e = cudaFuncSetAttribute(k_force_tile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)T.smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_force_tile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T.smem);
        if (e != cudaSuccess) return -1;
        tile_smem_attr = T.smem;
    }
    int a = 0, b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_force_tile<false>, TILE_THREADS, T.smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_force_tile<true>, TILE_THREADS, T.smem);
    return std::min(a, b);
}

int force_launch(const Geo& g, const Tiling& T, BufView in, StgView stg, int32_t* out_cnt, int j0, int nj,
                 DevErr* err, cudaStream_t s)
{
    if (T.kind == FORCE_PIPE) {
        pipe_launch(g, T, in, stg, out_cnt, j0, nj, err, s);
        return 1;
    }
    // NVE: force + kick + drift + destination in one pass; NVT: force + kick (the drift
    // needs the slice's lambda, k_drift)
    const long long ntiles = (long long)nj * T.tiles;
    const unsigned grid = (unsigned)std::min<long long>(ntiles, (long long)T.grid);
    // the tile counter is never reset: every launch consumes exactly ntiles + grid
    // increments (each CTA's last claim fails once), so the host tracks each launch's base
    if (g.thermo)
        launch(k_force_tile<true>, grid, TILE_THREADS, T.smem, s, g, T, in, stg, out_cnt, j0, nj, err, T.ctr,
               *T.ctr_base);
    else
        launch(k_force_tile<false>, grid, TILE_THREADS, T.smem, s, g, T, in, stg, out_cnt, j0, nj, err, T.ctr,
               *T.ctr_base);
    *T.ctr_base += (unsigned long long)ntiles + grid;
    return 1;
}

}  // namespace dsea
