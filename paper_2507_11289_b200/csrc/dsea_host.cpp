// dsea_host.cpp -- C ABI, host-side initialisation and the ring runtime of the
// B200-native DSEAmd engine (arXiv 2507.11289).  See include/dsea.h for the
// contract of every entry point and DESIGN.md for the design.
//
//  - geometry and slicing ........ P:63-73 §3, §4 (readings Q3, Q18)
//  - FCC lattice + velocities .... P:224-227 §4 (Q9, Q10); host, -ffp-contract=off
//  - stage schedule .............. Table 1 (§3.3) generalised to W workers
//                                  per GPU and N_GPU GPUs in a ring
//  - ring hop .................... P:118-119 §3.1, §3.4: one process per GPU;
//                                  default: copy-engine push over NVLink into the
//                                  successor's CUDA-IPC-mapped input slots, monotone
//                                  arrival/release counters as stream flags; NCCL
//                                  point-to-point and SM remote stores as comparisons
//  - stage plan .................. dsea_plan.h (shared with the stencil engine)
//  - super-cycle ................. P:89-92 §3.1
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <array>
#include <new>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dsea.h"
#include "dsea_internal.h"
#include "dsea_plan.h"

using namespace dsea;

// ------------------------------------------------------------------------------
// NCCL, loaded at run time (the process usually already has torch's copy).
// ------------------------------------------------------------------------------
namespace {
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl()
{
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return api;
#define LOADSYM(f, name) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, name))
    LOADSYM(GetUniqueId, "ncclGetUniqueId");
    LOADSYM(CommInitRank, "ncclCommInitRank");
    LOADSYM(CommDestroy, "ncclCommDestroy");
    LOADSYM(Send, "ncclSend");
    LOADSYM(Recv, "ncclRecv");
    LOADSYM(GroupStart, "ncclGroupStart");
    LOADSYM(GroupEnd, "ncclGroupEnd");
    LOADSYM(GetErrorString, "ncclGetErrorString");
#undef LOADSYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv &&
             api.GroupStart && api.GroupEnd && api.GetErrorString;
    return api;
}

// cuStreamWaitValue32 through the runtime's driver entry point (no libcuda link)
typedef int (*PFN_waitValue32)(cudaStream_t, unsigned long long, unsigned int, unsigned int);
PFN_waitValue32 wait_value32()
{
    static PFN_waitValue32 f = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            f = reinterpret_cast<PFN_waitValue32>(p);
    }
    return f;
}

// cuStreamWriteValue32 (same route): publishes a ring-hop flag from the copy stream
// without an SM, so it is not queued behind the persistent force kernel
typedef int (*PFN_writeValue32)(cudaStream_t, unsigned long long, unsigned int, unsigned int);
PFN_writeValue32 write_value32()
{
    static PFN_writeValue32 f = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            f = reinterpret_cast<PFN_writeValue32>(p);
    }
    return f;
}

}  // namespace

namespace dsea {
int stream_wait_geq32(cudaStream_t s, const uint32_t* addr, uint32_t v)
{
    return wait_value32() ? wait_value32()(s, (unsigned long long)addr, v, 0) : -1;
}
int stream_write32(cudaStream_t s, uint32_t* addr, uint32_t v)
{
    return write_value32() ? write_value32()(s, (unsigned long long)addr, v, 0) : -1;
}
bool stream_memops_available() { return wait_value32() && write_value32(); }
}  // namespace dsea

namespace {
struct PeerBlob {
    int32_t magic, rank, ns, pad;
    // settings every rank must share, or a stream wait is never satisfied and dsea_step
    // hangs: workers per GPU, block partition (count + hash), plan gap, hop options
    int32_t W, nblk, plan_gap, flags;
    uint64_t blocks_hash;
    cudaIpcMemHandle_t in, arr, rel;
};
constexpr int32_t PEER_MAGIC = 0x44534541;  // "DSEA"

}  // namespace

namespace dsea {
// ------------------------------------------------------------------------------
// Stage schedule (Table 1 generalised).  The slices of a super-cycle are grouped in
// blocks of B consecutive slices (B = 1 is the paper's schedule); flat blocks
// p = K*nblk + c run over the super-cycles K.  At stage k of a rank: receive block
// k; worker w processes block k-2-d*w (d = 2 for B = 1, d = 1 for B >= 2: a block's
// right neighbour slice is final one block earlier) and then finalises (bins) the
// slices whose three contributing units are done -- the last slice of the
// previous block and all but the last slice of this block; the last worker hands
// finalised slices to the ring successor.  Worker w of rank g in super-cycle K
// computes timestep K*N_w + g*W + w, or passes the block through unchanged when
// that timestep is beyond the requested count (Q15).  For B = 1 this is exactly
// Table 1: receive k, process k-2, send k-3.
// ------------------------------------------------------------------------------
// Partition of the N_S slices into the blocks of a super-cycle: nblk = ceil(N_S / B)
// blocks of balanced size (sizes differ by at most one slice, so no short tail block:
// a one-slice tail block cost up to 4 % on the C4 ring, profiles/r01/ring_tuning).
// Optional (DSEA_LEAD_BLOCKS=1, ring, B >= 4): the first two blocks have 2 slices
// ("lead" blocks), so rank g+1 can start a super-cycle after rank g processed 4 slices
// instead of 2 B.  Measured on 4 B200s (C4, B = 7): 0.9 % slower -- the steady-state
// lag between ranks is two blocks of the current size, so the earlier start only turns
// into a stall at the first full-size block and the drain keeps the full lag.
Blocks make_blocks(int ns, int ng, int B)
{
    Blocks bl;
    if (B < 1) B = 1;
    const char* e = getenv("DSEA_LEAD_BLOCKS");
    const bool lead = ng > 1 && B >= 4 && ns >= 4 + 2 * B && e && *e && atoi(e) != 0;
    int f = 0;
    if (lead)
        for (int k = 0; k < 2; k++) { bl.first.push_back(f); f += 2; }
    const int rest = ns - f;
    const int nb = (rest + B - 1) / B;
    for (int k = 0; k < nb; k++) bl.first.push_back(f + (int)((int64_t)rest * k / nb));
    bl.first.push_back(ns);
    bl.of.assign(ns, 0);
    for (int c = 0; c < bl.n(); c++)
        for (int s = bl.first[c]; s < bl.first[c + 1]; s++) bl.of[s] = c;
    bl.d = (B == 1) ? 2 : 1;
    return bl;
}


Plan build_plan(int ns, int ng, int rank, int W, int64_t n_steps, const Blocks& bl)
{
    Plan P;
    const int nblk = bl.n();
    const int d = bl.d;
    // past Eq. (1)'s bound: close each super-cycle before the next (see plan_gap).
    // With W > 1 the last slice is always finalised with its own block: worker w+1
    // processes the previous block in the same stage and, when the last block is a
    // single slice, needs it (found by tests/test_plan_sim.py).
    const bool plateau = plan_plateau(ng, W, bl);
    const bool early_fin = plateau || W > 1;
    const int gap = plan_gap(ng, W, bl);
    const int64_t nw = (int64_t)ng * W;
    const int64_t n_cycles = n_steps <= 0 ? 0 : (n_steps + nw - 1) / nw;
    const int64_t items = n_cycles * nblk;
    if (items == 0) return P;
    auto active = [&](int64_t K, int w) { return K * nw + (int64_t)rank * W + w < n_steps; };
    auto blk_first = [&](int c) { return bl.first[c]; };
    auto blk_count = [&](int c) { return bl.count(c); };
    // stage of flat block p: receive at sp(p), worker w processes it at sp(p) + 2 + d*w,
    // where sp(p) = p + gap * (p / nblk) (gap idle stages after each super-cycle)
    auto sp = [&](int64_t p) { return p + (int64_t)gap * (p / nblk); };
    int64_t r_lo = 0, r_hi = 0;  // flat blocks received
    if (ng > 1) {
        if (rank == 0) { r_lo = nblk; r_hi = items + nblk; }
        else { r_lo = 0; r_hi = items; }
    }
    const int64_t last_stage = std::max<int64_t>(sp(items - 1) + 3 + (int64_t)d * (W - 1),
                                                 r_hi > r_lo ? sp(r_hi - 1) : 0);
    // per stage: receives, then per worker its block (force or pass-through) and the
    // slices that block completes
    for (int64_t k = 0; k <= last_stage; k++) {
        for (int64_t p = r_lo; p < r_hi; p++)
            if (sp(p) == k) {
                const int c = (int)(p % nblk);
                for (int s = 0; s < blk_count(c); s++)
                    P.ops.push_back({OP_RECV, (int)k, -1, blk_first(c) + s, 1, (int)(p / nblk), -1});
            }
        for (int w = 0; w < W; w++) {
            // the flat block of worker w at stage k (at most one)
            int64_t p = -1;
            {
                const int64_t q = k - 2 - (int64_t)d * w;   // = sp(p)
                if (q >= 0) {
                    const int64_t K = q / ((int64_t)nblk + gap);
                    const int64_t c = q - K * ((int64_t)nblk + gap);
                    if (c < nblk) p = K * nblk + c;
                }
            }
            // after the last block: the last slice of the last super-cycle (Table 1's row N_S+3)
            if (!early_fin && k == sp(items - 1) + 3 + (int64_t)d * w) {
                const int64_t K = (items - 1) / nblk;
                if (active(K, w)) P.ops.push_back({OP_BIN, (int)k, w, ns - 1, 1, (int)K, -1});
                if (w == W - 1) P.ops.push_back({OP_SEND, (int)k, w, ns - 1, 1, (int)K, -1});
            }
            if (p < 0 || p >= items) continue;
            const int64_t K = p / nblk;
            const int c = (int)(p % nblk);
            if (active(K, w))
                P.ops.push_back({OP_FORCE, (int)k, w, blk_first(c), blk_count(c), (int)K,
                                 K * nw + (int64_t)rank * W + w});
            else
                P.ops.push_back({OP_PASS, (int)k, w, blk_first(c), blk_count(c), (int)K, -1});
            // finalise the slices whose three contributing units are now done: the last
            // slice of the previous block and all but the last of this block (Table 1);
            // the last slice of a super-cycle goes with the next super-cycle's first
            // block -- or, at the plateau, with its own block (x wall: no right
            // neighbour), so that a super-cycle is complete before the next one starts
            auto fin = [&](int64_t KK, int first, int cnt) {
                if (cnt <= 0) return;
                if (active(KK, w)) P.ops.push_back({OP_BIN, (int)k, w, first, cnt, (int)KK, -1});
                if (w == W - 1)
                    for (int s = 0; s < cnt; s++) P.ops.push_back({OP_SEND, (int)k, w, first + s, 1, (int)KK, -1});
            };
            if (early_fin) {
                const int first = c == 0 ? 0 : blk_first(c) - 1;
                const int last = c == nblk - 1 ? ns - 1 : blk_first(c) + blk_count(c) - 2;
                fin(K, first, last - first + 1);
            } else if (c != 0) {
                fin(K, blk_first(c) - 1, blk_count(c));         // [first-1, first+count-2]
            } else {
                if (p >= 1) fin(K - 1, ns - 1, 1);                // previous super-cycle's last slice
                fin(K, 0, blk_count(0) - 1);
            }
        }
    }
    P.n_stages = (int)(last_stage + 1);
    return P;
}

// push order within a stage: see order_pushes in dsea_plan.h
void order_pushes(std::vector<Op>& ops, int W)
{
    for (size_t i = 0; i + 1 < ops.size(); i++)
        if (ops[i].kind == OP_PASS && ops[i].worker == W - 1)
            for (size_t k = i + 1; k < ops.size() && ops[k].stage == ops[i].stage && ops[k].worker == ops[i].worker &&
                                   ops[k].kind == OP_BIN;
                 k++)
                if (ops[k].cycle < ops[i].cycle) std::rotate(ops.begin() + i, ops.begin() + k, ops.begin() + k + 1), i++;
}

// Idle stages between super-cycles.  With W > 1 workers, worker 0 starts super-cycle
// K+1 while the later workers still finish K; past Eq. (1)'s bound the
// data worker 0 waits for from the ring then depends on exactly those trailing
// blocks, and the stream order would deadlock.  There the ring is at its plateau
// anyway: a gap of d (W-1) stages lets every rank finish K first.
bool plan_plateau(int ng, int W, const Blocks& bl)
{
    if (ng == 1) return false;
    const int nblk = bl.n();
    const int d = bl.d;
    const char* e = getenv("DSEA_PLAN_GAP");           // sweeps: force on (1) / off (0)
    if (e && *e) return atoi(e) != 0;
    // threshold checked against a simulation of all ranks' streams (tests/test_plan_sim.py)
    return nblk < ng * (3 + d * (W - 1));
}

int plan_gap(int ng, int W, const Blocks& bl)
{
    return plan_plateau(ng, W, bl) ? bl.d * (W - 1) : 0;
}
}  // namespace dsea

namespace {
}  // namespace

// ------------------------------------------------------------------------------
// Context
// ------------------------------------------------------------------------------
struct dsea_ctx {
    dsea_box_params box{};
    double a = 0, b[3] = {0, 0, 0};
    int64_t N = 0;
    std::vector<double> h_xyz, h_v, h_f;  // host state by id (before dsea_slice)

    bool sliced = false;
    dsea_slice_params sp{};
    dsea_geometry geo{};
    Geo g{};
    Tiling T{};
    SlotLayout L{};
    int mode = DSEA_MODE_FUSED;
    int W = 1, NG = 1, rank = 0, device = 0, B = 1;
    Blocks bl;                            // block partition of a super-cycle (make_blocks)

    cudaStream_t cs = nullptr, ss = nullptr, rs = nullptr, es = nullptr, bs = nullptr;  // compute, send, recv, energy, remote bin
    BufView inb{};
    std::vector<BufView> outb;
    std::vector<StgView> stg;
    std::vector<void*> dallocs;
    UnitEnergy* e_dev = nullptr;
    size_t e_cap = 0;
    DevErr* err_dev = nullptr;
    unsigned long long* tile_ctr = nullptr;
    double* aos_dev = nullptr;            // by-id AoS scratch for set_state (per slice group) / get_* (3N)
    size_t aos_cap = 0;                   // doubles in aos_dev
    int32_t* ids_dev = nullptr;           // atom ids of an upload group
    int stg_pool = 0;                     // slices per staging buffer (StgView.pool)
    int out_pool = 0;                     // slots of the last worker's local output buffer
    std::vector<cudaEvent_t> ev_pslot;    // per slot of that pool: its last hop (push / send) done
    std::vector<char> pslot_rec;
    unsigned long long* count_dev = nullptr;
    unsigned long long tile_ctr_base = 0;
    std::vector<cudaEvent_t> ev_recv, ev_free, ev_bin, ev_send;
    std::vector<cudaEvent_t> ev_force;              // per worker: force done
    std::vector<cudaEvent_t> ev_energy;             // per (worker, block): energies of the block reduced
    std::vector<cudaEvent_t> ev_binblk;             // per block: last remote bin run done
    bool ce_hop = false;                            // peer hop: local bin + copy engine (default)
    cudaEvent_t ev_cs = nullptr;                    // compute-stream point for the bin stream

    bool connected = false;
    ncclComm_t send_comm = nullptr, recv_comm = nullptr;
    // peer backend: the last worker's bins write the finished slices straight into the
    // successor's input slots (CUDA IPC mapping over NVLink); arrival / release counts
    // travel through flag arrays (waits on local flags, writes by a signal kernel)
    bool peer = false;
    uint32_t* arr_dev = nullptr;        // [ns] local: arrivals into my input slots
    uint32_t* rel_dev = nullptr;        // [ns] local: releases of my successor's slots
    char* succ_in_base = nullptr;       // mapped successor input buffer
    uint32_t* succ_arr = nullptr;       // mapped successor arrival flags
    uint32_t* pred_rel = nullptr;       // mapped predecessor release flags
    std::vector<uint32_t> wr_cnt, exp_arr, rel_cnt;
    // copy-engine hop: monotone counters instead of per-slot flags (as the stencil
    // engine, dsea_grid.cpp): slots arrive / are released in (super-cycle, slot)
    // order, so the k-th arrival (release) of slot s is event (k-1) N_S + s + 1; one
    // stream memory op per hop / release instead of one per slot, and no release
    // kernel on the compute stream.  arr_dev[0] / rel_dev[0] hold the counters.
    bool ctr = false;
    uint32_t rel_init = 0;                          // successor's slots start occupied (it is rank 0)
    std::vector<uint32_t> push_k, rel_k;            // per slot: pushes made, releases made
    cudaEvent_t ev_bs = nullptr;                    // last push on the hop stream
    char* own_outb_last = nullptr;      // locally allocated last output buffer (unused when peer)

    // host mirror of the device state (rank 0), valid until the next mutation
    std::vector<char> mirror;
    bool mirror_valid = false;
    bool holds_state = false;

    std::vector<dsea_energy> energies;
    std::vector<dsea_profile> prof;       // per slice, x-resolved sums (Q24)
    int64_t steps_done = 0;

    bool timing = false;
    std::vector<cudaEvent_t> tev_pool;
    size_t tev_used = 0;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> tpairs;  // kind, (start, stop)
    dsea_stats stats{};

    std::string msg;
};

namespace {
dsea_status fail(dsea_ctx* c, dsea_status s, const char* fmt, ...)
{
    if (c) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        c->msg = buf;
    }
    return s;
}

#define CUDA_TRY(ctx, expr)                                                                   \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            return fail(ctx, _e == cudaErrorMemoryAllocation ? DSEA_ENOMEM : DSEA_ECUDA,      \
                        "%s: %s", #expr, cudaGetErrorString(_e));                            \
    } while (0)

// Geometry (§4) with the slicing of P:63-73 §3 and reading Q3.
dsea_status compute_geometry(const dsea_box_params* box, const dsea_slice_params* sp,
                             dsea_geometry* out, std::string* why)
{
    std::memset(out, 0, sizeof *out);
    const int c = sp->cells_per_slice_x;
    const double a = std::cbrt(4.0 / box->rho);
    out->a = a;
    out->b[0] = box->nx * a;
    out->b[1] = box->ny * a;
    out->b[2] = box->nz * a;
    out->n_atoms = 4LL * box->nx * box->ny * box->nz;
    const double sr6 = 1.0 / (box->rc * box->rc * box->rc * box->rc * box->rc * box->rc);
    out->u_shift = sr6 - sr6 * sr6;
    if (c < 1) { *why = "cells_per_slice_x must be >= 1"; return DSEA_EINVAL; }
    int ns = sp->n_slices > 0 ? sp->n_slices : (int)std::floor(out->b[0] / (c * box->rc));
    out->n_slices = ns;
    out->cells[0] = c * ns;
    out->cells[1] = (int)std::floor(out->b[1] / box->rc);
    out->cells[2] = (int)std::floor(out->b[2] / box->rc);
    for (int d = 0; d < 3; d++) out->l[d] = out->cells[d] > 0 ? out->b[d] / out->cells[d] : 0.0;
    out->w = ns > 0 ? out->b[0] / ns : 0.0;
    const int W = sp->workers_per_gpu > 0 ? sp->workers_per_gpu : 1;
    out->n_max = ns / (2 + W * 2);
    const double cf = sp->capacity_factor > 0 ? sp->capacity_factor : 1.25;
    const double mean = ns > 0 ? (double)out->n_atoms / ns : 0.0;
    long long cap = (long long)std::ceil(cf * mean + 4.0 * std::sqrt(mean) + 8.0);
    cap = (cap + 31) / 32 * 32;
    out->slot_capacity = (int)std::min<long long>(cap, 1LL << 30);
    char buf[256];
    if (ns < 1) { *why = "slice width: b_x < c*rc gives no slice"; return DSEA_EGEOM; }
    if (out->cells[1] < 3 || out->cells[2] < 3) {
        snprintf(buf, sizeof buf, "need >= 3 cells in y and z (got %d x %d); b_y, b_z >= 3 rc",
                 out->cells[1], out->cells[2]);
        *why = buf;
        return DSEA_EGEOM;
    }
    if (out->l[0] < box->rc || out->l[1] < box->rc || out->l[2] < box->rc) {
        snprintf(buf, sizeof buf, "cell edge below rc: l = (%.6g, %.6g, %.6g), rc = %.6g "
                 "(slice width %.6g with %d cells per slice)", out->l[0], out->l[1], out->l[2],
                 box->rc, out->w, c);
        *why = buf;
        return DSEA_EGEOM;
    }
    return DSEA_OK;
}

// FCC lattice, offset a/4 (Q10); id = ((ix*ny + iy)*nz + iz)*4 + k.
void host_lattice(const dsea_box_params& bx, double a, double* xyz)
{
    const double basis[4][3] = {{0.0, 0.0, 0.0}, {0.5, 0.5, 0.0}, {0.5, 0.0, 0.5}, {0.0, 0.5, 0.5}};
    int64_t id = 0;
    for (int ix = 0; ix < bx.nx; ix++)
        for (int iy = 0; iy < bx.ny; iy++)
            for (int iz = 0; iz < bx.nz; iz++)
                for (int k = 0; k < 4; k++, id++) {
                    xyz[3 * id + 0] = (ix + basis[k][0] + 0.25) * a;
                    xyz[3 * id + 1] = (iy + basis[k][1] + 0.25) * a;
                    xyz[3 * id + 2] = (iz + basis[k][2] + 0.25) * a;
                }
}

// Velocities "initialized according to the temperature", reading Q9:
// splitmix64 stream -> 53-bit uniforms -> Box-Muller cosine branch, drawn in id
// order x, y, z; zero momentum; exact rescale to T0 with 3N degrees of freedom.
struct SplitMix {
    uint64_t s;
    uint64_t next()
    {
        s += 0x9E3779B97F4A7C15ULL;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double uniform() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
};

void host_velocities(int64_t n, uint64_t seed, double T0, double* v)
{
    SplitMix rng{seed};
    for (int64_t i = 0; i < 3 * n; i++) {
        const double u1 = rng.uniform();
        const double u2 = rng.uniform();
        v[i] = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * 3.141592653589793 * u2);
    }
    for (int d = 0; d < 3; d++) {
        double s = 0.0;
        for (int64_t i = 0; i < n; i++) s += v[3 * i + d];
        const double mean = s / (double)n;
        for (int64_t i = 0; i < n; i++) v[3 * i + d] -= mean;
    }
    double s2 = 0.0;
    for (int64_t i = 0; i < n; i++)
        s2 += v[3 * i] * v[3 * i] + v[3 * i + 1] * v[3 * i + 1] + v[3 * i + 2] * v[3 * i + 2];
    const double f = std::sqrt(T0 / (s2 / (3.0 * (double)n)));
    for (int64_t i = 0; i < 3 * n; i++) v[i] *= f;
}

void disconnect(dsea_ctx* c)
{
    if (c->sliced) cudaSetDevice(c->device);
    if (c->peer) {
        cudaDeviceSynchronize();
        if (c->succ_in_base) cudaIpcCloseMemHandle(c->succ_in_base);
        if (c->succ_arr) cudaIpcCloseMemHandle(c->succ_arr);
        if (c->pred_rel) cudaIpcCloseMemHandle(c->pred_rel);
        c->succ_in_base = nullptr; c->succ_arr = nullptr; c->pred_rel = nullptr;
        c->peer = false;
        c->ce_hop = false;
        if (!c->outb.empty() && c->outb.back().remote) {
            c->outb.back().base = c->own_outb_last;
            c->outb.back().remote = 0;
        }
        c->connected = false;
    }
}

void free_device(dsea_ctx* c)
{
    if (c->sliced) cudaSetDevice(c->device);
    disconnect(c);
    if (c->connected) {
        if (nccl().ok) {
            // ncclCommDestroy finalizes collectively: destroy the two link
            // communicators in global link order (link r = rank r -> r+1) so that
            // every pair of ranks meets in the same order (no cross-order deadlock).
            const int send_link = c->rank, recv_link = (c->rank - 1 + c->NG) % c->NG;
            ncclComm_t first = send_link < recv_link ? c->send_comm : c->recv_comm;
            ncclComm_t second = send_link < recv_link ? c->recv_comm : c->send_comm;
            if (first) nccl().CommDestroy(first);
            if (second) nccl().CommDestroy(second);
        }
        c->send_comm = c->recv_comm = nullptr;
        c->connected = false;
    }
    for (void* p : c->dallocs) cudaFree(p);
    c->dallocs.clear();
    c->aos_dev = nullptr; c->aos_cap = 0; c->ids_dev = nullptr; c->count_dev = nullptr;
    for (cudaEvent_t e : c->ev_pslot) cudaEventDestroy(e);
    c->ev_pslot.clear(); c->pslot_rec.clear();
    for (auto* v : {&c->ev_recv, &c->ev_free, &c->ev_bin, &c->ev_send})
        for (cudaEvent_t e : *v) cudaEventDestroy(e);
    c->ev_recv.clear(); c->ev_free.clear(); c->ev_bin.clear(); c->ev_send.clear();
    for (cudaEvent_t e : c->tev_pool) cudaEventDestroy(e);
    c->tev_pool.clear();
    c->tpairs.clear();
    c->tev_used = 0;
    if (c->cs) cudaStreamDestroy(c->cs);
    if (c->ss) cudaStreamDestroy(c->ss);
    if (c->rs) cudaStreamDestroy(c->rs);
    if (c->es) cudaStreamDestroy(c->es);
    if (c->bs) cudaStreamDestroy(c->bs);
    for (cudaEvent_t e : c->ev_binblk) cudaEventDestroy(e);
    c->ev_binblk.clear();
    if (c->ev_cs) cudaEventDestroy(c->ev_cs);
    if (c->ev_bs) cudaEventDestroy(c->ev_bs);
    c->ev_bs = nullptr;
    c->ev_cs = nullptr;
    c->bs = nullptr;
    for (cudaEvent_t e : c->ev_force) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ev_energy) cudaEventDestroy(e);
    c->ev_force.clear(); c->ev_energy.clear();
    c->cs = c->ss = c->rs = c->es = nullptr;
    c->e_dev = nullptr; c->e_cap = 0;
    c->outb.clear(); c->stg.clear();
    c->sliced = false;
    c->holds_state = false;
    c->mirror_valid = false;
}

template <class T>
dsea_status dalloc(dsea_ctx* c, T** p, size_t count)
{
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, std::max<size_t>(count * sizeof(T), 256));
    if (e != cudaSuccess)
        return fail(c, DSEA_ENOMEM, "cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
    c->dallocs.push_back(q);
    *p = static_cast<T*>(q);
    return DSEA_OK;
}

// a slot buffer of `nslots` slots (slice j in slot j % nslots); the per-cell counters
// stay per slice (4 B per cell)
dsea_status alloc_buf(dsea_ctx* c, BufView* B, int nslots, int perm_slots)
{
    dsea_status s;
    B->L = c->L;
    B->nslots = nslots;
    B->perm_slots = perm_slots;
    B->soff = 0;
    B->poff = 0;
    if ((s = dalloc(c, &B->base, c->L.slot_bytes * (size_t)nslots))) return s;
    if ((s = dalloc(c, &B->cnt, (size_t)c->g.ns * c->g.ncell))) return s;
    if ((s = dalloc(c, &B->perm, (size_t)perm_slots * c->g.cap))) return s;
    CUDA_TRY(c, cudaMemset(B->cnt, 0, sizeof(int32_t) * (size_t)c->g.ns * c->g.ncell));
    // zeroed scratch: after a reported error no later pass can index out of bounds
    CUDA_TRY(c, cudaMemset(B->perm, 0, sizeof(BinRec) * (size_t)perm_slots * c->g.cap));
    CUDA_TRY(c, cudaMemset(B->base, 0, c->L.slot_bytes * (size_t)nslots));
    return DSEA_OK;
}

dsea_status alloc_stg(dsea_ctx* c, StgView* S)
{
    dsea_status s;
    S->pool = c->stg_pool;
    S->soff = 0;
    const size_t n = (size_t)c->stg_pool * c->g.cap;
    double** d[] = {&S->x, &S->y, &S->z, &S->vx, &S->vy, &S->vz, &S->fx, &S->fy, &S->fz};
    for (auto* p : d)
        if ((s = dalloc(c, p, n))) return s;
    if ((s = dalloc(c, &S->id, n))) return s;
    if ((s = dalloc(c, &S->key, n))) return s;
    if ((s = dalloc(c, &S->n, (size_t)c->g.ns))) return s;
    if ((s = dalloc(c, &S->eatom, energy_records(c->g, c->T)))) return s;
    CUDA_TRY(c, cudaMemset(S->key, 0, sizeof(int32_t) * n));
    CUDA_TRY(c, cudaMemset(S->n, 0, sizeof(int32_t) * (size_t)c->g.ns));
    return DSEA_OK;
}

dsea_status check_dev_err(dsea_ctx* c)
{
    DevErr e{};
    CUDA_TRY(c, cudaMemcpy(&e, c->err_dev, sizeof e, cudaMemcpyDeviceToHost));
    if (e.code == 0) return DSEA_OK;
    CUDA_TRY(c, cudaMemset(c->err_dev, 0, sizeof(DevErr)));
    switch (e.code) {
    case DSEA_ECAPACITY:
        return fail(c, DSEA_ECAPACITY, "capacity exceeded: slice %d needs %d (slot capacity %d, "
                    "force-tile staging capacity %d)", e.slice, e.aux, c->g.cap, c->T.smax);
    case DSEA_EUNSTABLE:
        return fail(c, DSEA_EUNSTABLE, "atom %d left slice %d for slice %d in one step (or became "
                    "non-finite): timestep too large", e.atom, e.slice, e.aux);
    case DSEA_EINVAL:
        return fail(c, DSEA_EINVAL, "atom %d lies outside [0,b_x] x [0,b_y) x [0,b_z)", e.atom);
    default:
        return fail(c, (dsea_status)e.code, "device error %d", e.code);
    }
}

// by-id AoS scratch of at least `doubles` doubles
dsea_status ensure_aos(dsea_ctx* c, size_t doubles)
{
    dsea_status s;
    if (!c->count_dev && (s = dalloc(c, &c->count_dev, 1))) return s;
    if (c->aos_cap >= doubles) return DSEA_OK;
    if (c->aos_dev) {
        cudaFree(c->aos_dev);
        c->dallocs.erase(std::remove(c->dallocs.begin(), c->dallocs.end(), (void*)c->aos_dev), c->dallocs.end());
        c->aos_dev = nullptr;
        c->aos_cap = 0;
    }
    if ((s = dalloc(c, &c->aos_dev, doubles))) return s;
    c->aos_cap = doubles;
    return DSEA_OK;
}

// Bin the flat host state (by id) into the slots of the input buffer.  The atoms are
// grouped on the host by destination slice (the same IEEE floor(x / l_x) as the
// device, Q4) into runs of at most inb.perm_slots slices whose atoms fit the staging
// buffer (a pool of stg_pool slices on a ring), and each group is uploaded and binned on its own; the
// slot contents do not depend on the grouping (cells are ordered by (z, id), Q21).
dsea_status upload_state(dsea_ctx* c, const double* xyz, const double* v, const double* f)
{
    const int64_t N = c->N;
    const int ns = c->g.ns;
    const size_t stg_cap = (size_t)c->stg_pool * c->g.cap;     // flat staging entries
    dsea_status s;
    if ((size_t)N <= stg_cap && ns <= c->inb.perm_slots) {
        // everything fits one group (fused pass, full buffers): upload by id as it is,
        // no host-side grouping (ids = staging index)
        if ((s = ensure_aos(c, std::max<size_t>((f ? 9 : 6) * (size_t)N, 1)))) return s;
        double* dx = c->aos_dev;
        double* dv = c->aos_dev + 3 * (size_t)N;
        double* df = f ? c->aos_dev + 6 * (size_t)N : nullptr;
        CUDA_TRY(c, cudaMemcpyAsync(dx, xyz, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, c->cs));
        CUDA_TRY(c, cudaMemcpyAsync(dv, v, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, c->cs));
        if (f) CUDA_TRY(c, cudaMemcpyAsync(df, f, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, c->cs));
        StgView& S = c->stg[0];
        if (N > 0) {
            aos_to_stage_launch(S, dx, dv, df, nullptr, (int)N, c->cs);
            init_keys_launch(c->g, S, (int)N, c->inb.cnt, c->err_dev, c->cs);
        }
        bin_scan_launch(c->g, c->inb, 0, ns, c->err_dev, c->cs);
        if (N > 0) bin_place_launch(c->g, c->inb, S, 0, 0, (int)N, 0, ns, c->err_dev, c->cs);
        bin_gather_launch(c->g, c->inb, S, 0, ns, c->err_dev, c->cs);
        c->stats.kernel_launches += N > 0 ? 5 : 2;
        CUDA_TRY(c, cudaStreamSynchronize(c->cs));
        CUDA_TRY(c, cudaGetLastError());
        if ((s = check_dev_err(c))) return s;
        c->holds_state = true;
        c->mirror_valid = false;
        return DSEA_OK;
    }
    std::vector<int32_t> slice_of((size_t)N);
    std::vector<int64_t> count((size_t)ns + 1, 0);
    for (int64_t i = 0; i < N; i++) {
        const double q = std::floor(xyz[3 * i] / c->g.l[0]);   // reading Q4 (IEEE division)
        const int cx = !(q >= 0.0) ? 0 : (q >= (double)(c->g.cells[0] - 1) ? c->g.cells[0] - 1 : (int)q);
        slice_of[(size_t)i] = cx / c->g.c;
        count[(size_t)slice_of[(size_t)i] + 1]++;
    }
    for (int j = 0; j < ns; j++) count[(size_t)j + 1] += count[(size_t)j];
    // atom ids sorted by slice, id order within a slice (stable counting sort)
    std::vector<int32_t> order((size_t)N);
    {
        std::vector<int64_t> cur(count.begin(), count.end() - 1);
        for (int64_t i = 0; i < N; i++) order[(size_t)cur[(size_t)slice_of[(size_t)i]]++] = (int32_t)i;
    }
    std::vector<int32_t>().swap(slice_of);
    // a group binds at most perm_slots slices (the bin scratch holds one slot per slice)
    const int maxs = std::max(1, c->inb.perm_slots);
    size_t max_group = 0;
    for (int m0 = 0; m0 < ns;) {   // largest group that fits the staging buffer
        int m1 = m0 + 1;
        while (m1 < ns && m1 - m0 < maxs && (size_t)(count[(size_t)m1 + 1] - count[(size_t)m0]) <= stg_cap) m1++;
        const size_t na = (size_t)(count[(size_t)m1] - count[(size_t)m0]);
        if (na > stg_cap)
            return fail(c, DSEA_ECAPACITY, "slice %d holds %zu atoms (staging capacity %zu)", m0, na, stg_cap);
        max_group = std::max(max_group, na);
        m0 = m1;
    }
    if ((s = ensure_aos(c, std::max<size_t>(9 * max_group, 1)))) return s;
    if (!c->ids_dev && (s = dalloc(c, &c->ids_dev, std::max<size_t>(stg_cap, 1)))) return s;
    std::vector<double> hx, hv, hf;
    for (int m0 = 0; m0 < ns;) {
        int m1 = m0 + 1;
        while (m1 < ns && m1 - m0 < maxs && (size_t)(count[(size_t)m1 + 1] - count[(size_t)m0]) <= stg_cap) m1++;
        const int64_t a0 = count[(size_t)m0], na = count[(size_t)m1] - a0;
        if (na > 0) {
            hx.resize((size_t)na * 3); hv.resize((size_t)na * 3); hf.resize((size_t)na * 3);
            for (int64_t k = 0; k < na; k++) {
                const int64_t id = order[(size_t)(a0 + k)];
                for (int d = 0; d < 3; d++) {
                    hx[(size_t)(3 * k + d)] = xyz[3 * id + d];
                    hv[(size_t)(3 * k + d)] = v[3 * id + d];
                    hf[(size_t)(3 * k + d)] = f ? f[3 * id + d] : 0.0;   // F_new = F_old = 0 (Q7)
                }
            }
            double* dx = c->aos_dev;
            double* dv = c->aos_dev + 3 * (size_t)na;
            double* df = c->aos_dev + 6 * (size_t)na;
            CUDA_TRY(c, cudaMemcpyAsync(dx, hx.data(), sizeof(double) * 3 * na, cudaMemcpyHostToDevice, c->cs));
            CUDA_TRY(c, cudaMemcpyAsync(dv, hv.data(), sizeof(double) * 3 * na, cudaMemcpyHostToDevice, c->cs));
            CUDA_TRY(c, cudaMemcpyAsync(df, hf.data(), sizeof(double) * 3 * na, cudaMemcpyHostToDevice, c->cs));
            CUDA_TRY(c, cudaMemcpyAsync(c->ids_dev, order.data() + a0, sizeof(int32_t) * na, cudaMemcpyHostToDevice,
                                        c->cs));
            StgView& S = c->stg[0];
            aos_to_stage_launch(S, dx, dv, df, c->ids_dev, (int)na, c->cs);
            init_keys_launch(c->g, S, (int)na, c->inb.cnt, c->err_dev, c->cs);
        }
        BufView ib = c->inb;
        ib.poff = -m0;                  // the group's slices in bin-scratch slots 0 .. m1-m0-1
        bin_scan_launch(c->g, ib, m0, m1 - m0, c->err_dev, c->cs);
        if (na > 0) bin_place_launch(c->g, ib, c->stg[0], 0, 0, (int)na, m0, m1 - m0, c->err_dev, c->cs);
        bin_gather_launch(c->g, ib, c->stg[0], m0, m1 - m0, c->err_dev, c->cs);
        c->stats.kernel_launches += na > 0 ? 5 : 2;
        CUDA_TRY(c, cudaStreamSynchronize(c->cs));   // the host group buffers are reused
        CUDA_TRY(c, cudaGetLastError());
        if ((s = check_dev_err(c))) return s;
        m0 = m1;
    }
    c->holds_state = true;
    c->mirror_valid = false;
    return DSEA_OK;
}

dsea_status fetch_mirror(dsea_ctx* c)
{
    if (c->mirror_valid) return DSEA_OK;
    const size_t bytes = c->L.slot_bytes * (size_t)c->g.ns;
    c->mirror.resize(bytes);
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaMemcpy(c->mirror.data(), c->inb.base, bytes, cudaMemcpyDeviceToHost));
    c->mirror_valid = true;
    return DSEA_OK;
}

// iterate atoms of the mirror: fn(slice, index_in_slot, cell_local, id, slot_base)
template <class F>
void for_each_atom(dsea_ctx* c, F fn)
{
    for (int j = 0; j < c->g.ns; j++) {
        const char* base = c->mirror.data() + (size_t)j * c->L.slot_bytes;
        const int32_t* cs = reinterpret_cast<const int32_t*>(base);
        const int32_t* ids = reinterpret_cast<const int32_t*>(base + c->L.off_id);
        for (int cell = 0; cell < c->g.ncell; cell++)
            for (int i = cs[cell]; i < cs[cell + 1]; i++) fn(j, i, cell, ids[i], base);
    }
}

// the host start state: FCC lattice (Q10) and velocities (Q9) by id; F = 0 (Q7,
// implicit: h_f stays empty until a caller sets forces)
dsea_status ensure_host_state(dsea_ctx* c)
{
    if (!c->h_xyz.empty()) return DSEA_OK;
    try {
        c->h_xyz.resize((size_t)c->N * 3);
        c->h_v.resize((size_t)c->N * 3);
    } catch (...) {
        c->h_xyz.clear(); c->h_v.clear();
        return fail(c, DSEA_ENOMEM, "host start state of %lld atoms", (long long)c->N);
    }
    host_lattice(c->box, c->a, c->h_xyz.data());
    host_velocities(c->N, c->box.seed, c->box.T0, c->h_v.data());
    return DSEA_OK;
}

dsea_status get_vec(dsea_ctx* c, double* out, int64_t n, int which)
{
    if (!c) return DSEA_EINVAL;
    if (!out || n != c->N) return fail(c, DSEA_EINVAL, "array of %lld atoms expected", (long long)c->N);
    if (!c->sliced) {
        dsea_status s = ensure_host_state(c);
        if (s) return s;
        const std::vector<double>& src = which == 0 ? c->h_xyz : which == 1 ? c->h_v : c->h_f;
        if (src.empty()) std::memset(out, 0, sizeof(double) * 3 * (size_t)c->N);   // forces: 0 (Q7)
        else std::memcpy(out, src.data(), sizeof(double) * 3 * (size_t)c->N);
        return DSEA_OK;
    }
    if (!c->holds_state) return fail(c, DSEA_ESTATE, "this rank does not hold the state (rank 0 does)");
    // scatter by id on the GPU, then one contiguous device-to-host copy
    dsea_status s = ensure_aos(c, 3 * (size_t)c->N);
    if (s) return s;
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaMemsetAsync(c->count_dev, 0, sizeof(unsigned long long), c->cs));
    slots_to_aos_launch(c->g, c->inb, which, c->aos_dev, c->count_dev, c->cs);
    unsigned long long seen = 0;
    CUDA_TRY(c, cudaMemcpyAsync(out, c->aos_dev, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->cs));
    CUDA_TRY(c, cudaMemcpyAsync(&seen, c->count_dev, sizeof seen, cudaMemcpyDeviceToHost, c->cs));
    CUDA_TRY(c, cudaStreamSynchronize(c->cs));
    if ((int64_t)seen != c->N)
        return fail(c, DSEA_ESTATE, "slots hold %llu atoms, expected %lld", seen, (long long)c->N);
    return DSEA_OK;
}

cudaEvent_t tev(dsea_ctx* c)
{
    if (c->tev_used == c->tev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        c->tev_pool.push_back(e);
    }
    return c->tev_pool[c->tev_used++];
}

enum { TK_FORCE = 0, TK_BIN = 1, TK_SEND = 2 };

dsea_status run_plan(dsea_ctx* c, int64_t n_steps)
{
    const int ns = c->g.ns;
    const Plan P = build_plan(ns, c->NG, c->rank, c->W, n_steps, c->bl);
    std::vector<char> sent(ns, 0);
    const size_t sb = c->L.slot_bytes;
    NcclApi& api = nccl();
    const int W = c->W;
    auto in_of = [&](int w) -> BufView& { return w == 0 ? c->inb : c->outb[w - 1]; };
    // pools: slice j of super-cycle K in slot (j + soff) % slots, soff = (K ns) % slots
    // (BufView.soff); views of a buffer / staging buffer for the ops of cycle K
    auto soff_of = [&](int cycle, int slots) {
        return (int)(((int64_t)(cycle % slots) * (int64_t)(ns % slots)) % slots);
    };
    // device views for a launch whose lowest slice is jmin: offsets normalised so that
    // j + off lies in [0, 2 slots) for the launch's slices (BufView.soff)
    auto norm = [&](int cycle, int slots, int jmin) {
        return (int)(((int64_t)jmin + soff_of(cycle, slots)) % slots) - jmin;
    };
    auto buf_at = [&](const BufView& B, int cycle, int jmin) {
        BufView v = B;
        v.soff = norm(cycle, B.nslots, jmin);
        v.poff = norm(cycle, B.perm_slots, jmin);
        return v;
    };
    auto stg_at = [&](int w, int cycle, int jmin) { StgView v = c->stg[w]; v.soff = norm(cycle, v.pool, jmin); return v; };
    // copy slices [j, j+n) between slot buffers of dst_slots / src_slots slots (slice s in
    // slot (s + off) % slots): one cudaMemcpyAsync per run that wraps around neither buffer
    auto copy_run = [&](char* dst, int dst_slots, int dst_off, const char* src, int src_slots, int src_off, int j,
                        int n, cudaStream_t st) -> dsea_status {
        for (int k = 0; k < n;) {
            const int sd = (int)((((int64_t)j + k + dst_off) % dst_slots + dst_slots) % dst_slots);
            const int ss_ = (int)((((int64_t)j + k + src_off) % src_slots + src_slots) % src_slots);
            const int run = std::min(n - k, std::min(dst_slots - sd, src_slots - ss_));
            CUDA_TRY(c, cudaMemcpyAsync(dst + (size_t)sd * sb, src + (size_t)ss_ * sb, sb * run,
                                        cudaMemcpyDeviceToDevice, st));
            k += run;
        }
        return DSEA_OK;
    };
    // the last worker's output pool: before slices [m, m+n) are written into it, the
    // hops that read the previous occupants of those slots must be done
    auto wait_pool = [&](int m, int n, int cycle, cudaStream_t st) -> dsea_status {
        BufView& ob = c->outb[W - 1];
        const int off = soff_of(cycle, ob.nslots);
        for (int sl = m; sl < m + n; sl++) {
            const int p = (sl + off) % ob.nslots;
            if (p < (int)c->pslot_rec.size() && c->pslot_rec[(size_t)p])
                CUDA_TRY(c, cudaStreamWaitEvent(st, c->ev_pslot[(size_t)p], 0));
        }
        return DSEA_OK;
    };
    auto record_pool = [&](int m, int n, int cycle, cudaStream_t st) -> dsea_status {
        BufView& ob = c->outb[W - 1];
        const int off = soff_of(cycle, ob.nslots);
        for (int sl = m; sl < m + n; sl++) {
            const int p = (sl + off) % ob.nslots;
            if (p >= (int)c->pslot_rec.size()) continue;
            CUDA_TRY(c, cudaEventRecord(c->ev_pslot[(size_t)p], st));
            c->pslot_rec[(size_t)p] = 1;
        }
        return DSEA_OK;
    };
    // counter mode (c->ctr): event number of the k-th arrival / release of slot s
    auto ev_no = [&](uint32_t k, int s) { return (k - 1) * (uint32_t)ns + (uint32_t)s + 1; };
    auto wait_arrival = [&](int s) -> dsea_status {
        const bool ok = c->ctr ? stream_wait_geq32(c->cs, c->arr_dev, ev_no(c->exp_arr[s], s)) == 0
                               : wait_value32()(c->cs, (unsigned long long)(c->arr_dev + s), c->exp_arr[s], 0) == 0;
        return ok ? DSEA_OK : fail(c, DSEA_EPEER, "cuStreamWaitValue32 (arrival) failed");
    };
    auto release_ctr = [&](int f0, int f1) -> dsea_status {   // slots [f0, f1] read for the last time
        if (f1 < f0) return DSEA_OK;
        for (int sl = f0; sl <= f1; sl++) c->rel_k[sl]++;
        if (stream_write32(c->cs, c->pred_rel, ev_no(c->rel_k[f1], f1)))
            return fail(c, DSEA_EPEER, "cuStreamWriteValue32 (release) failed");
        return DSEA_OK;
    };
    // counter mode: pushes must leave in (super-cycle, slot) order (order_pushes)
    std::vector<Op> ops = P.ops;
    if (c->ctr) order_pushes(ops, W);
    const size_t nops = ops.size();
    for (size_t oi = 0; oi < nops; oi++) {
        const Op& op = ops[oi];
        switch (op.kind) {
        case OP_RECV: {
            if (c->peer) {  // data arrives by remote stores; just count the expected arrival
                c->exp_arr[op.slice]++;
                break;
            }
            // all receives of this stage in one NCCL group (matched by order with the
            // predecessor's sends, one message per slice)
            size_t oe = oi;
            while (oe < nops && ops[oe].kind == OP_RECV && ops[oe].stage == op.stage) oe++;
            for (size_t q = oi; q < oe; q++)
                CUDA_TRY(c, cudaStreamWaitEvent(c->rs, c->ev_free[ops[q].slice], 0));
            api.GroupStart();
            for (size_t q = oi; q < oe; q++) {
                ncclResult_t r = api.Recv(c->inb.base + (size_t)ops[q].slice * sb, sb, ncclChar, 0,
                                          c->recv_comm, c->rs);
                if (r != ncclSuccess) { api.GroupEnd(); return fail(c, DSEA_EPEER, "ncclRecv: %s", api.GetErrorString(r)); }
            }
            ncclResult_t r = api.GroupEnd();
            if (r != ncclSuccess) return fail(c, DSEA_EPEER, "ncclGroupEnd (recv): %s", api.GetErrorString(r));
            for (size_t q = oi; q < oe; q++) CUDA_TRY(c, cudaEventRecord(c->ev_recv[ops[q].slice], c->rs));
            oi = oe - 1;
            break;
        }
        case OP_FORCE: {
            const int j = op.slice, n = op.count, w = op.worker;
            if (w == 0 && c->NG > 1 && !(c->rank == 0 && op.cycle == 0)) {
                const int need = std::min(j + n, ns - 1);   // right neighbour of the block
                if (c->peer) {
                    dsea_status s = wait_arrival(need);
                    if (s) return s;
                } else {
                    CUDA_TRY(c, cudaStreamWaitEvent(c->cs, c->ev_recv[need], 0));
                }
            }
            cudaEvent_t t0 = nullptr, t1 = nullptr;
            // this block's per-atom energy records of the previous super-cycle must be
            // reduced before the pass rewrites them (other blocks' reductions may still
            // run: they overlap this pass instead of stalling it)
            cudaEvent_t& ev_e = c->ev_energy[(size_t)w * c->bl.n() + c->bl.of[j]];
            CUDA_TRY(c, cudaStreamWaitEvent(c->cs, ev_e, 0));
            if (c->peer && !c->ce_hop && w == W - 1) {
                // staging of this block and the arrival counters it adds to were last read
                // by the remote bin runs of blocks c and c+1 one super-cycle ago
                CUDA_TRY(c, cudaStreamWaitEvent(c->cs, c->ev_binblk[(c->bl.of[j] + 1) % c->bl.n()], 0));
            }
            if (c->timing) { t0 = tev(c); t1 = tev(c); cudaEventRecord(t0, c->cs); }
            c->stats.kernel_launches +=
                force_launch(c->g, c->T, in_of(w), stg_at(w, op.cycle, j), c->outb[w].cnt, j, n, c->err_dev, c->cs);
            c->stats.force_launches++;
            if (c->timing) { cudaEventRecord(t1, c->cs); c->tpairs.push_back({TK_FORCE, {t0, t1}}); }
            if (c->g.thermo) {  // NVT: lambda_j on the critical path, then the drift
                UnitEnergy* eo = c->e_dev + (size_t)op.t_rel * ns;
                energy_launch(c->g, c->T, stg_at(w, op.cycle, j), j, n, eo, c->cs);
                drift_launch(c->g, stg_at(w, op.cycle, j), j, n, eo, c->outb[w].cnt, c->err_dev, c->cs);
                CUDA_TRY(c, cudaEventRecord(ev_e, c->cs));
                c->stats.kernel_launches += 2;
            } else {  // per-slice energy reduction off the critical path
                CUDA_TRY(c, cudaEventRecord(c->ev_force[w], c->cs));
                CUDA_TRY(c, cudaStreamWaitEvent(c->es, c->ev_force[w], 0));
                energy_launch(c->g, c->T, stg_at(w, op.cycle, j), j, n, c->e_dev + (size_t)op.t_rel * ns, c->es);
                CUDA_TRY(c, cudaEventRecord(ev_e, c->es));
                c->stats.kernel_launches++;
            }
            if (w == 0 && c->NG > 1) {
                // slot s is last read by the unit of slice s+1
                const int f0 = std::max(j - 1, 0), f1 = (j + n == ns) ? ns - 1 : j + n - 2;
                if (c->ctr) {
                    dsea_status s = release_ctr(f0, f1);
                    if (s) return s;
                } else if (c->peer) {
                    if (f1 >= f0) {  // release the slots to the predecessor (one count per cycle)
                        const uint32_t v = ++c->rel_cnt[f0];
                        for (int sl = f0 + 1; sl <= f1; sl++) c->rel_cnt[sl] = v;
                        signal_launch(c->pred_rel, f0, f1 - f0 + 1, v, c->cs);
                        c->stats.kernel_launches++;
                    }
                } else {
                    for (int sl = f0; sl <= f1; sl++) CUDA_TRY(c, cudaEventRecord(c->ev_free[sl], c->cs));
                }
            }
            break;
        }
        case OP_PASS: {
            const int j = op.slice, n = op.count, w = op.worker;
            if (w == 0 && c->NG > 1 && !(c->rank == 0 && op.cycle == 0)) {
                if (c->peer) {
                    dsea_status s = wait_arrival(j + n - 1);
                    if (s) return s;
                } else {
                    CUDA_TRY(c, cudaStreamWaitEvent(c->cs, c->ev_recv[j + n - 1], 0));
                }
            }
            if (c->ctr && w == W - 1 && c->NG > 1) {
                // push on the compute stream after every earlier push (hop stream) has
                // left, so the arrival counter stays in slot order
                CUDA_TRY(c, cudaStreamWaitEvent(c->cs, c->ev_bs, 0));
                for (int sl = j; sl < j + n; sl++) c->push_k[sl]++;
                const uint32_t need = c->push_k[j + n - 1] - 1 + c->rel_init;
                if (need > 0 && stream_wait_geq32(c->cs, c->rel_dev, ev_no(need, j + n - 1)))
                    return fail(c, DSEA_EPEER, "cuStreamWaitValue32 (release) failed");
                CUDA_TRY(c, cudaMemcpyAsync(c->succ_in_base + (size_t)j * sb, in_of(w).base + (size_t)j * sb, sb * n,
                                            cudaMemcpyDeviceToDevice, c->cs));
                if (stream_write32(c->cs, c->succ_arr, ev_no(c->push_k[j + n - 1], j + n - 1)))
                    return fail(c, DSEA_EPEER, "cuStreamWriteValue32 (arrival) failed");
                CUDA_TRY(c, cudaEventRecord(c->ev_bs, c->cs));
                if (w == 0) {
                    dsea_status s = release_ctr(j, j + n - 1);
                    if (s) return s;
                }
                break;
            }
            if (c->ctr && w == 0 && c->NG > 1) {       // (w < W-1: local copy, then release)
                BufView& src0 = in_of(0);
                if (src0.base != c->outb[0].base)
                    CUDA_TRY(c, cudaMemcpyAsync(c->outb[0].base + (size_t)j * sb, src0.base + (size_t)j * sb, sb * n,
                                                cudaMemcpyDeviceToDevice, c->cs));
                dsea_status s = release_ctr(j, j + n - 1);
                if (s) return s;
                break;
            }
            uint32_t wv = 0;
            if (w == W - 1 && c->NG > 1) {
                if (c->peer) {
                    wv = ++c->wr_cnt[j];
                    for (int sl = j + 1; sl < j + n; sl++) c->wr_cnt[sl] = wv;
                    for (int sl = j; sl < j + n; sl++)
                        if (wait_value32()(c->cs, (unsigned long long)(c->rel_dev + sl), wv, 0))
                            return fail(c, DSEA_EPEER, "cuStreamWaitValue32 (release) failed");
                } else {
                    for (int sl = j; sl < j + n; sl++)
                        if (sent[sl]) CUDA_TRY(c, cudaStreamWaitEvent(c->cs, c->ev_send[sl], 0));
                }
            }
            BufView& src = in_of(w);
            const bool to_succ = c->ce_hop && w == W - 1 && c->NG > 1;
            char* dst_base = to_succ ? c->succ_in_base : c->outb[w].base;
            const int dst_slots = to_succ ? ns : c->outb[w].nslots;
            if (!to_succ && w == W - 1 && c->NG > 1) {
                dsea_status s = wait_pool(j, n, op.cycle, c->cs);
                if (s) return s;
            }
            if (src.base != dst_base) {
                dsea_status s = copy_run(dst_base, dst_slots, soff_of(op.cycle, dst_slots), src.base, src.nslots,
                                         soff_of(op.cycle, src.nslots), j, n, c->cs);
                if (s) return s;
            }
            if (w == 0 && c->NG > 1) {
                if (c->peer) {
                    const uint32_t v = ++c->rel_cnt[j];
                    for (int sl = j + 1; sl < j + n; sl++) c->rel_cnt[sl] = v;
                    signal_launch(c->pred_rel, j, n, v, c->cs);
                } else {
                    for (int sl = j; sl < j + n; sl++) CUDA_TRY(c, cudaEventRecord(c->ev_free[sl], c->cs));
                }
            }
            if (w == W - 1 && c->NG > 1) {
                if (c->peer) signal_launch(c->succ_arr, j, n, wv, c->cs);
                else for (int sl = j; sl < j + n; sl++) CUDA_TRY(c, cudaEventRecord(c->ev_bin[sl], c->cs));
            }
            break;
        }
        case OP_BIN: {
            const int m = op.slice, n = op.count, w = op.worker;
            if (c->ce_hop && w == W - 1 && c->NG > 1) {
                // copy-engine hop: bin into the local last buffer on the compute stream,
                // then the copy stream pushes the finished slots over NVLink and raises
                // the successor's arrival flags -- neither needs an SM, so both overlap
                // the next block's (persistent, SM-filling) force pass
                {   // the pushes that read the previous occupants of these pool slots
                    dsea_status s = wait_pool(m, n, op.cycle, c->cs);
                    if (s) return s;
                }
                cudaEvent_t t0 = nullptr, t1 = nullptr;
                if (c->timing) { t0 = tev(c); t1 = tev(c); cudaEventRecord(t0, c->cs); }
                const int s0 = std::max(m - 1, 0), s1 = std::min(m + n, ns - 1);
                const BufView ob = buf_at(c->outb[w], op.cycle, s0);
                const StgView sv = stg_at(w, op.cycle, s0);
                bin_scan_launch(c->g, ob, m, n, c->err_dev, c->cs);
                bin_place_launch(c->g, ob, sv, s0, s1 - s0 + 1, 0, m, n, c->err_dev, c->cs);
                bin_gather_launch(c->g, ob, sv, m, n, c->err_dev, c->cs);
                c->stats.kernel_launches += 3;
                if (c->timing) { cudaEventRecord(t1, c->cs); c->tpairs.push_back({TK_BIN, {t0, t1}}); }
                const uint32_t wv = ++c->wr_cnt[m];
                for (int sl = m + 1; sl < m + n; sl++) c->wr_cnt[sl] = wv;
                CUDA_TRY(c, cudaEventRecord(c->ev_cs, c->cs));
                CUDA_TRY(c, cudaStreamWaitEvent(c->bs, c->ev_cs, 0));
                if (c->ctr) {                        // one wait on the successor's release counter
                    for (int sl = m; sl < m + n; sl++) c->push_k[sl]++;
                    const uint32_t need = c->push_k[m + n - 1] - 1 + c->rel_init;
                    if (need > 0 && stream_wait_geq32(c->bs, c->rel_dev, ev_no(need, m + n - 1)))
                        return fail(c, DSEA_EPEER, "cuStreamWaitValue32 (release) failed");
                } else {
                    for (int sl = m; sl < m + n; sl++)   // the successor released the previous occupants
                        if (wait_value32()(c->bs, (unsigned long long)(c->rel_dev + sl), wv, 0))
                            return fail(c, DSEA_EPEER, "cuStreamWaitValue32 (release) failed");
                }
                cudaEvent_t h0 = nullptr, h1 = nullptr;
                if (c->timing) { h0 = tev(c); h1 = tev(c); cudaEventRecord(h0, c->bs); }
                {
                    dsea_status s = copy_run(c->succ_in_base, ns, 0, ob.base, ob.nslots, ob.soff, m, n, c->bs);
                    if (s) return s;
                }
                if (c->ctr) {
                    if (stream_write32(c->bs, c->succ_arr, ev_no(c->push_k[m + n - 1], m + n - 1)))
                        return fail(c, DSEA_EPEER, "cuStreamWriteValue32 (arrival) failed");
                    CUDA_TRY(c, cudaEventRecord(c->ev_bs, c->bs));
                } else {
                    for (int sl = m; sl < m + n; sl++)
                        if (write_value32()(c->bs, (unsigned long long)(c->succ_arr + sl), wv, 0))
                            return fail(c, DSEA_EPEER, "cuStreamWriteValue32 (arrival) failed");
                }
                if (c->timing) { cudaEventRecord(h1, c->bs); c->tpairs.push_back({TK_SEND, {h0, h1}}); }
                {
                    dsea_status s = record_pool(m, n, op.cycle, c->bs);
                    if (s) return s;
                }
                c->stats.hop_bytes += (int64_t)sb * n;
                break;
            }
            uint32_t wv = 0;
            // the last worker's bins write into the successor over NVLink: run them on
            // their own stream so the transfer overlaps the next block's force pass
            const bool remote = c->peer && w == W - 1;
            cudaStream_t bst = remote ? c->bs : c->cs;
            if (remote) {
                CUDA_TRY(c, cudaEventRecord(c->ev_cs, c->cs));
                CUDA_TRY(c, cudaStreamWaitEvent(c->bs, c->ev_cs, 0));
            }
            if (w == W - 1 && c->NG > 1) {
                if (c->peer) {  // the successor must have released the previous occupants
                    wv = ++c->wr_cnt[m];
                    for (int sl = m + 1; sl < m + n; sl++) c->wr_cnt[sl] = wv;
                    for (int sl = m; sl < m + n; sl++)
                        if (wait_value32()(bst, (unsigned long long)(c->rel_dev + sl), wv, 0))
                            return fail(c, DSEA_EPEER, "cuStreamWaitValue32 (release) failed");
                } else {
                    for (int sl = m; sl < m + n; sl++)
                        if (sent[sl]) CUDA_TRY(c, cudaStreamWaitEvent(c->cs, c->ev_send[sl], 0));
                    dsea_status s = wait_pool(m, n, op.cycle, c->cs);
                    if (s) return s;
                }
            }
            cudaEvent_t t0 = nullptr, t1 = nullptr;
            if (c->timing) { t0 = tev(c); t1 = tev(c); cudaEventRecord(t0, bst); }
            const int s0 = std::max(m - 1, 0), s1 = std::min(m + n, ns - 1);
            const BufView ob = buf_at(c->outb[w], op.cycle, s0);
            const StgView sv = stg_at(w, op.cycle, s0);
            bin_scan_launch(c->g, ob, m, n, c->err_dev, bst);
            bin_place_launch(c->g, ob, sv, s0, s1 - s0 + 1, 0, m, n, c->err_dev, bst);
            bin_gather_launch(c->g, ob, sv, m, n, c->err_dev, bst);
            c->stats.kernel_launches += 3;
            if (c->timing) { cudaEventRecord(t1, bst); c->tpairs.push_back({TK_BIN, {t0, t1}}); }
            if (w == W - 1 && c->NG > 1) {
                if (c->peer) {  // the slices are already in the successor's memory: publish
                    signal_launch(c->succ_arr, m, n, wv, bst);
                    c->stats.kernel_launches++;
                    c->stats.hop_bytes += (int64_t)sb * n;
                    // keyed by the block of this run's last slot: a force pass on block c
                    // waits for the run covering slot (c+1)B, i.e. key c+1
                    CUDA_TRY(c, cudaEventRecord(c->ev_binblk[c->bl.of[m + n - 1]], bst));
                } else {
                    for (int sl = m; sl < m + n; sl++) CUDA_TRY(c, cudaEventRecord(c->ev_bin[sl], c->cs));
                }
            }
            break;
        }
        case OP_SEND: {
            size_t oe = oi;
            while (oe < nops && ops[oe].kind == OP_SEND && ops[oe].stage == op.stage) oe++;
            // ring of one: written into the input buffer; peer: written into the successor
            if (c->NG == 1 || c->peer) { oi = oe - 1; break; }
            for (size_t q = oi; q < oe; q++)
                CUDA_TRY(c, cudaStreamWaitEvent(c->ss, c->ev_bin[ops[q].slice], 0));
            cudaEvent_t t0 = nullptr, t1 = nullptr;
            if (c->timing) { t0 = tev(c); t1 = tev(c); cudaEventRecord(t0, c->ss); }
            api.GroupStart();
            for (size_t q = oi; q < oe; q++) {
                const BufView& ob = c->outb[W - 1];
                const int slot = (ops[q].slice + soff_of(ops[q].cycle, ob.nslots)) % ob.nslots;
                ncclResult_t r = api.Send(ob.base + (size_t)slot * sb, sb, ncclChar, 1,
                                          c->send_comm, c->ss);
                if (r != ncclSuccess) { api.GroupEnd(); return fail(c, DSEA_EPEER, "ncclSend: %s", api.GetErrorString(r)); }
            }
            ncclResult_t r = api.GroupEnd();
            if (r != ncclSuccess) return fail(c, DSEA_EPEER, "ncclGroupEnd (send): %s", api.GetErrorString(r));
            if (c->timing) { cudaEventRecord(t1, c->ss); c->tpairs.push_back({TK_SEND, {t0, t1}}); }
            for (size_t q = oi; q < oe; q++) {
                CUDA_TRY(c, cudaEventRecord(c->ev_send[ops[q].slice], c->ss));
                sent[ops[q].slice] = 1;
                c->stats.hop_bytes += (int64_t)sb;
                dsea_status s = record_pool(ops[q].slice, 1, ops[q].cycle, c->ss);
                if (s) return s;
            }
            oi = oe - 1;
            break;
        }
        }
    }
    if (c->peer && c->rank == 0) {  // the final super-cycle lands in rank 0's input buffer
        if (c->ctr) {
            if (c->exp_arr[ns - 1] > 0) {
                dsea_status s = wait_arrival(ns - 1);
                if (s) return s;
            }
        } else {
            for (int sl = 0; sl < ns; sl++)
                if (wait_value32()(c->cs, (unsigned long long)(c->arr_dev + sl), c->exp_arr[sl], 0))
                    return fail(c, DSEA_EPEER, "cuStreamWaitValue32 (final arrival) failed");
        }
    }
    return DSEA_OK;
}

dsea_status run_fused(dsea_ctx* c, int64_t n_steps)
{
    const int ns = c->g.ns;
    for (int64_t t = 0; t < n_steps; t++) {
        cudaEvent_t t0 = nullptr, t1 = nullptr, t2 = nullptr;
        if (c->timing) { t0 = tev(c); t1 = tev(c); t2 = tev(c); cudaEventRecord(t0, c->cs); }
        CUDA_TRY(c, cudaStreamWaitEvent(c->cs, c->ev_energy[0], 0));
        int nl = force_launch(c->g, c->T, c->inb, c->stg[0], c->inb.cnt, 0, ns, c->err_dev, c->cs);
        if (c->g.thermo) {  // NVT: lambda_j, then the drift
            UnitEnergy* eo = c->e_dev + (size_t)t * ns;
            energy_launch(c->g, c->T, c->stg[0], 0, ns, eo, c->cs);
            drift_launch(c->g, c->stg[0], 0, ns, eo, c->inb.cnt, c->err_dev, c->cs);
            CUDA_TRY(c, cudaEventRecord(c->ev_energy[0], c->cs));
            nl += 2;
        } else {
            CUDA_TRY(c, cudaEventRecord(c->ev_force[0], c->cs));
            CUDA_TRY(c, cudaStreamWaitEvent(c->es, c->ev_force[0], 0));
            energy_launch(c->g, c->T, c->stg[0], 0, ns, c->e_dev + (size_t)t * ns, c->es);
            CUDA_TRY(c, cudaEventRecord(c->ev_energy[0], c->es));
            nl++;
        }
        if (c->timing) cudaEventRecord(t1, c->cs);
        bin_scan_launch(c->g, c->inb, 0, ns, c->err_dev, c->cs);
        bin_place_launch(c->g, c->inb, c->stg[0], 0, ns, 0, 0, ns, c->err_dev, c->cs);
        bin_gather_launch(c->g, c->inb, c->stg[0], 0, ns, c->err_dev, c->cs);
        if (c->timing) {
            cudaEventRecord(t2, c->cs);
            c->tpairs.push_back({TK_FORCE, {t0, t1}});
            c->tpairs.push_back({TK_BIN, {t1, t2}});
        }
        c->stats.kernel_launches += 3 + nl;
        c->stats.force_launches += 1;
    }
    return DSEA_OK;
}
}  // namespace

// ==============================================================================
// C ABI
// ==============================================================================
extern "C" {

dsea_status dsea_init(const dsea_box_params* box, dsea_ctx** out)
{
    if (!out) return DSEA_EINVAL;
    *out = nullptr;
    if (!box || box->nx < 1 || box->ny < 1 || box->nz < 1 || !(box->rho > 0) || !(box->rc > 0) ||
        !(box->dt > 0) || !(box->T0 >= 0))
        return DSEA_EINVAL;
    const int64_t N = 4LL * box->nx * box->ny * box->nz;
    if (N > (1LL << 30)) return DSEA_EINVAL;
    dsea_ctx* c = new (std::nothrow) dsea_ctx();
    if (!c) return DSEA_ENOMEM;
    c->box = *box;
    c->a = std::cbrt(4.0 / box->rho);
    c->b[0] = box->nx * c->a;
    c->b[1] = box->ny * c->a;
    c->b[2] = box->nz * c->a;
    c->N = N;
    // the start state (FCC lattice + velocities by id) is generated on first use: only
    // the rank that uploads it (rank 0 of a ring) ever materialises the 48 B/atom host
    // arrays (at 1e9 atoms every other rank would otherwise hold 48 GB it never reads)
    *out = c;
    return DSEA_OK;
}

dsea_status dsea_geometry_compute(const dsea_box_params* box, const dsea_slice_params* sp,
                                  dsea_geometry* out)
{
    if (!box || !sp || !out || !(box->rho > 0) || !(box->rc > 0) || box->nx < 1 || box->ny < 1 ||
        box->nz < 1)
        return DSEA_EINVAL;
    std::string why;
    return compute_geometry(box, sp, out, &why);
}

dsea_status dsea_slice(dsea_ctx* c, const dsea_slice_params* sp)
{
    if (!c) return DSEA_EINVAL;
    if (!sp) return fail(c, DSEA_EINVAL, "null slice params");
    if (sp->n_gpus < 1 || sp->rank < 0 || sp->rank >= sp->n_gpus || sp->workers_per_gpu < 1 ||
        sp->device < 0 || sp->mode < 0 || sp->mode > 2)
        return fail(c, DSEA_EINVAL, "bad slice params (n_gpus %d, rank %d, W %d, device %d, mode %d)",
                    sp->n_gpus, sp->rank, sp->workers_per_gpu, sp->device, sp->mode);
    int mode = sp->mode;
    if (mode == DSEA_MODE_AUTO) mode = (sp->n_gpus == 1 && sp->workers_per_gpu == 1) ? DSEA_MODE_FUSED : DSEA_MODE_STAGED;
    if (mode == DSEA_MODE_FUSED && (sp->n_gpus != 1 || sp->workers_per_gpu != 1))
        return fail(c, DSEA_EINVAL, "fused mode needs n_gpus == 1 and workers_per_gpu == 1");
    dsea_geometry geo;
    std::string why;
    dsea_status s = compute_geometry(&c->box, sp, &geo, &why);
    if (s) return fail(c, s, "%s", why.c_str());
    // slices per stage (block size B): enough atoms per launch to fill a B200, but
    // keep >= N_GPU*(2+W) blocks per super-cycle so the ring stays busy (Eq. (1))
    int B = sp->slices_per_stage;
    if (B < 0) return fail(c, DSEA_EINVAL, "slices_per_stage < 0");
    if (B == 0) {
        // ~2e6 atoms per launch, but >= N_GPU (2 + W) - 1 blocks per super-cycle so the
        // ring stays busy (each rank trails its predecessor by two blocks; Eq. (1));
        // tuned on 2 and 4 B200s (profiles/r01/ring_tuning: C4 best at 8-9 blocks on 2
        // GPUs, 11 on 4)
        const int nb_t = (int)std::ceil((double)geo.n_atoms / 2.0e6);
        const int depth = sp->n_gpus > 1 ? sp->n_gpus * (2 + sp->workers_per_gpu) - 1 : 2 + sp->workers_per_gpu;
        const int nb = std::max(1, std::max(nb_t, depth));
        B = std::max(1, (geo.n_slices + nb - 1) / nb);
        while (B > 1 && (geo.n_slices + B - 1) / B < depth) B--;
        if (mode == DSEA_MODE_FUSED) B = 1;
    }
    B = std::min(B, std::max(1, geo.n_slices - 2));
    if (mode == DSEA_MODE_STAGED && sp->n_gpus == 1) {
        const int nblk = (geo.n_slices + B - 1) / B;
        const bool ok = B == 1 ? geo.n_slices >= 2 + 2 * sp->workers_per_gpu : nblk >= 2 + sp->workers_per_gpu;
        if (!ok)
            return fail(c, DSEA_EGEOM, "a ring of one with W = %d workers and %d slices per stage needs more "
                        "slices (N_S = %d; Eq. (1))", sp->workers_per_gpu, B, geo.n_slices);
    }

    // keep the current state (host mirror of the device or the host arrays)
    std::vector<double> xyz, v, f;
    if (c->sliced && c->holds_state) {
        xyz.resize((size_t)c->N * 3); v.resize((size_t)c->N * 3); f.resize((size_t)c->N * 3);
        if ((s = get_vec(c, xyz.data(), c->N, 0)) || (s = get_vec(c, v.data(), c->N, 1)) ||
            (s = get_vec(c, f.data(), c->N, 2)))
            return s;
    }
    // the host start state (never sliced yet) moves into the device slots of the
    // uploading rank; the host copy is released once the upload succeeded
    const bool from_host = !c->sliced && (sp->rank == 0 || sp->n_gpus == 1);
    if (from_host && (s = ensure_host_state(c))) return s;
    free_device(c);

    c->sp = *sp;
    c->mode = mode;
    c->geo = geo;
    c->W = sp->workers_per_gpu;
    c->B = B;
    c->NG = sp->n_gpus;
    c->bl = make_blocks(geo.n_slices, c->NG, B);
    c->rank = sp->rank;
    c->device = sp->device;

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(c, DSEA_ECUDA, "no CUDA device available (the engine has no CPU fallback)");
    if (sp->device >= ndev) return fail(c, DSEA_EINVAL, "device %d of %d", sp->device, ndev);
    CUDA_TRY(c, cudaSetDevice(sp->device));

    Geo& g = c->g;
    for (int d = 0; d < 3; d++) { g.b[d] = geo.b[d]; g.l[d] = geo.l[d]; g.cells[d] = geo.cells[d]; }
    g.rc = c->box.rc;
    g.rc2 = c->box.rc * c->box.rc;
    g.dt = c->box.dt;
    g.ushift = geo.u_shift;
    g.c = sp->cells_per_slice_x;
    g.ns = geo.n_slices;
    g.ncell = g.c * geo.cells[1] * geo.cells[2];
    g.cap = geo.slot_capacity;
    g.rc2_screen = (float)(g.rc2 * (1.0 + 1e-5) + 1e-3);
    {   // gather rows: about twice the mean cell occupancy (rarer larger cells: global path)
        const double mean_cell = (double)c->N / ((double)g.ns * g.ncell);
        g.cell_max = 32;
        while (g.cell_max < 128 && g.cell_max < 2.0 * mean_cell + 24.0) g.cell_max *= 2;
    }
    g.thermo = 0;          // NVE until dsea_set_thermostat
    g.T_target = 0.0;
    c->L = make_slot_layout(g.ncell, g.cap);

    int optin = 0;
    CUDA_TRY(c, cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, sp->device));
    // a capacity factor above the default declares denser regions than the mean: the
    // force tiles' shared-memory staging is sized for them too
    const double dens_scale = std::max(1.0, (sp->capacity_factor > 0 ? sp->capacity_factor : 1.25) / 1.25);
    const double mean_per_cell = dens_scale * (double)c->N / ((double)g.ns * g.ncell);
    c->T = choose_tiling(g, mean_per_cell, optin);
    const int per_sm = force_kernel_attr(c->T);
    if (per_sm < 1) return fail(c, DSEA_ECUDA, "cannot set %zu bytes of dynamic shared memory", c->T.smem);
    int sms = 0;
    CUDA_TRY(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, sp->device));
    c->T.grid = sms * per_sm;

    CUDA_TRY(c, cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
    CUDA_TRY(c, cudaStreamCreateWithFlags(&c->ss, cudaStreamNonBlocking));
    CUDA_TRY(c, cudaStreamCreateWithFlags(&c->rs, cudaStreamNonBlocking));
    CUDA_TRY(c, cudaStreamCreateWithFlags(&c->es, cudaStreamNonBlocking));
    CUDA_TRY(c, cudaStreamCreateWithFlags(&c->bs, cudaStreamNonBlocking));
    CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_cs, cudaEventDisableTiming));
    c->sliced = true;
    c->prof.assign((size_t)c->g.ns, dsea_profile{});

    // buffers: input buffer + one output buffer per worker; the last worker of a ring
    // of one writes straight back into the input buffer (local hand-off).  On the staged
    // schedule only a window of slices is live in a worker's staging buffer (a block's
    // pass writes B slices; the pending bins read one slice on each side) and in the
    // last worker's local output buffer of a ring (binned, then pushed or sent): pools
    // of stg_pool / out_pool slots (slice j in slot j % pool, P:121-122's circular
    // slot buffers, NEXT-3).  The input buffer keeps N_S slots: rank 0 holds the whole
    // state between calls (Q22).
    {
        int bmax = 1;
        for (int k = 0; k < c->bl.n(); k++) bmax = std::max(bmax, c->bl.count(k));
        const bool staged = mode == DSEA_MODE_STAGED;
        const char* hop = getenv("DSEA_PEER_HOP");
        // remote stores need the full buffers: the successor's slots are written directly,
        // and the remote bins run on their own stream, unordered with the next force pass
        // that would rewrite a pooled staging slot
        const bool sm_hop = c->NG > 1 && hop && std::strcmp(hop, "sm") == 0;
        c->stg_pool = (staged && c->T.kind == FORCE_TILE && !sm_hop) ? std::min(g.ns, 2 * bmax + 4) : g.ns;
        c->out_pool = (c->NG > 1 && !sm_hop) ? std::min(g.ns, 4 * bmax + 4) : g.ns;
        // pools only where the full buffers would not fit comfortably: full-size staging
        // and output buffers (no slot arithmetic, no upload grouping) while they take at
        // most a quarter of the device memory; DSEA_POOLS=1 forces the pools (tests),
        // DSEA_POOLS=0 forces full buffers (A/B)
        const size_t full_bytes =
            (size_t)g.ns * ((size_t)c->W * g.cap * (9 * sizeof(double) + 2 * sizeof(int32_t)) + c->L.slot_bytes +
                            (size_t)g.cap * sizeof(BinRec));
        size_t free_b = 0, total_b = 0;
        cudaMemGetInfo(&free_b, &total_b);
        const char* pe = getenv("DSEA_POOLS");
        const int force = (pe && *pe) ? atoi(pe) : -1;
        if (force == 0 || (force < 0 && full_bytes * 4 <= total_b)) c->stg_pool = c->out_pool = g.ns;
    }
    // the input buffer is binned into only by the fused pass / a ring of one (all slices
    // at once) and by the upload (groups of <= stg_pool slices)
    if ((s = alloc_buf(c, &c->inb, g.ns, c->NG == 1 ? g.ns : c->stg_pool))) return s;
    c->outb.resize(c->W);
    for (int w = 0; w < c->W; w++) {
        const bool alias = (w == c->W - 1) && c->NG == 1;
        const int np = w == c->W - 1 ? c->out_pool : g.ns;
        if (alias) c->outb[w] = c->inb;
        else if ((s = alloc_buf(c, &c->outb[w], np, np))) return s;
    }
    c->ev_pslot.resize((size_t)c->out_pool);
    for (auto& e : c->ev_pslot) CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->pslot_rec.assign((size_t)c->out_pool, 0);
    c->stg.resize(c->W);
    for (int w = 0; w < c->W; w++)
        if ((s = alloc_stg(c, &c->stg[w]))) return s;
    if ((s = dalloc(c, &c->err_dev, 1))) return s;
    if ((s = dalloc(c, &c->tile_ctr, 1))) return s;
    if ((s = dalloc(c, &c->arr_dev, (size_t)g.ns))) return s;
    if ((s = dalloc(c, &c->rel_dev, (size_t)g.ns))) return s;
    CUDA_TRY(c, cudaMemset(c->arr_dev, 0, sizeof(uint32_t) * g.ns));
    CUDA_TRY(c, cudaMemset(c->rel_dev, 0, sizeof(uint32_t) * g.ns));
    CUDA_TRY(c, cudaMemset(c->tile_ctr, 0, sizeof(unsigned long long)));
    c->tile_ctr_base = 0;
    c->T.ctr = c->tile_ctr;
    c->T.ctr_base = &c->tile_ctr_base;
    CUDA_TRY(c, cudaMemset(c->err_dev, 0, sizeof(DevErr)));
    {
        const int nblk = c->bl.n();
        c->ev_binblk.resize(nblk);
        for (int k = 0; k < nblk; k++) CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_binblk[k], cudaEventDisableTiming));
    }
    c->ev_force.resize(c->W);
    for (int w = 0; w < c->W; w++) CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_force[w], cudaEventDisableTiming));
    c->ev_energy.resize((size_t)c->W * c->bl.n());
    for (auto& e : c->ev_energy) CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto* v : {&c->ev_recv, &c->ev_free, &c->ev_bin, &c->ev_send}) {
        v->resize(g.ns);
        for (int j = 0; j < g.ns; j++) CUDA_TRY(c, cudaEventCreateWithFlags(&(*v)[j], cudaEventDisableTiming));
    }

    c->msg.clear();
    if (c->NG > geo.n_max)
        c->msg = "note: N_GPU exceeds N_max of Eq. (1); the ring runs at the plateau (P:364)";
    if (c->rank == 0 || c->NG == 1) {
        const std::vector<double>& X = from_host ? c->h_xyz : xyz;
        const std::vector<double>& V = from_host ? c->h_v : v;
        const std::vector<double>& F = from_host ? c->h_f : f;
        if (X.empty()) return fail(c, DSEA_ESTATE, "no state to slice");
        if ((s = upload_state(c, X.data(), V.data(), F.empty() ? nullptr : F.data()))) return s;
        if (from_host) {
            std::vector<double>().swap(c->h_xyz);
            std::vector<double>().swap(c->h_v);
            std::vector<double>().swap(c->h_f);
        }
    }
    return DSEA_OK;
}

dsea_status dsea_ring_unique_id(void* out, size_t out_bytes)
{
    if (!out || out_bytes < sizeof(ncclUniqueId)) return DSEA_EINVAL;
    NcclApi& api = nccl();
    if (!api.ok) return DSEA_EPEER;
    ncclUniqueId id;
    if (api.GetUniqueId(&id) != ncclSuccess) return DSEA_EPEER;
    std::memcpy(out, &id, sizeof id);
    return DSEA_OK;
}

dsea_status dsea_ring_connect(dsea_ctx* c, const void* ids, int32_t n_ids)
{
    if (!c) return DSEA_EINVAL;
    if (!c->sliced) return fail(c, DSEA_ESTATE, "dsea_ring_connect before dsea_slice");
    if (c->NG == 1) return DSEA_OK;
    if (!ids || n_ids != c->NG) return fail(c, DSEA_EINVAL, "need %d link ids, got %d", c->NG, n_ids);
    NcclApi& api = nccl();
    if (!api.ok) return fail(c, DSEA_EPEER, "libnccl.so.2 not loadable");
    CUDA_TRY(c, cudaSetDevice(c->device));
    // NCCL p2p is a rendezvous: a send of a pooled slot completes only once the
    // successor posts the receive, which waits on the successor's own progress -- with a
    // pool, rebinning a slot would wait on that send and the ring can deadlock. The NCCL
    // (comparison) backend therefore keeps a full-size last output buffer.
    if (c->out_pool < c->g.ns) {
        BufView& ob = c->outb[c->W - 1];
        for (void* q : {(void*)ob.base, (void*)ob.cnt, (void*)ob.perm}) {
            cudaFree(q);
            c->dallocs.erase(std::remove(c->dallocs.begin(), c->dallocs.end(), q), c->dallocs.end());
        }
        dsea_status s = alloc_buf(c, &ob, c->g.ns, c->g.ns);
        if (s) return s;
        for (size_t k = c->ev_pslot.size(); k < (size_t)c->g.ns; k++) {
            cudaEvent_t e;
            CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c->ev_pslot.push_back(e);
        }
        c->pslot_rec.assign((size_t)c->g.ns, 0);
        c->out_pool = c->g.ns;
    }
    const ncclUniqueId* u = static_cast<const ncclUniqueId*>(ids);
    const int prev = (c->rank - 1 + c->NG) % c->NG;
    api.GroupStart();
    ncclResult_t r1 = api.CommInitRank(&c->send_comm, 2, u[c->rank], 0);  // link rank -> rank+1
    ncclResult_t r2 = api.CommInitRank(&c->recv_comm, 2, u[prev], 1);     // link prev -> rank
    ncclResult_t r3 = api.GroupEnd();
    if (r1 != ncclSuccess || r2 != ncclSuccess || r3 != ncclSuccess)
        return fail(c, DSEA_EPEER, "ncclCommInitRank: %s / %s / %s", api.GetErrorString(r1),
                    api.GetErrorString(r2), api.GetErrorString(r3));
    c->connected = true;
    return DSEA_OK;
}

// the ring settings a peer blob carries (compared in dsea_ring_connect_peer)
static void peer_settings(const dsea_ctx* c, PeerBlob& b)
{
    b.W = c->W;
    b.nblk = c->bl.n();
    b.plan_gap = plan_gap(c->NG, c->W, c->bl);
    const char* hop = getenv("DSEA_PEER_HOP");
    const bool ce = !(hop && std::strcmp(hop, "sm") == 0);
    const char* ctr = getenv("DSEA_RING_COUNTERS");
    const bool cn = ce && !(ctr && *ctr && atoi(ctr) == 0);
    b.flags = (ce ? 1 : 0) | (cn ? 2 : 0);
    uint64_t h = 1469598103934665603ull;                  // FNV-1a of the block starts
    for (int f : c->bl.first) { h ^= (uint64_t)(uint32_t)f; h *= 1099511628211ull; }
    b.blocks_hash = h;
}

dsea_status dsea_ring_export(dsea_ctx* c, void* out, size_t cap, size_t* len)
{
    if (!c || !len) return DSEA_EINVAL;
    *len = sizeof(PeerBlob);
    if (!out) return DSEA_OK;
    if (cap < sizeof(PeerBlob)) return fail(c, DSEA_EINVAL, "export buffer needs %zu bytes", sizeof(PeerBlob));
    if (!c->sliced) return fail(c, DSEA_ESTATE, "dsea_ring_export before dsea_slice");
    CUDA_TRY(c, cudaSetDevice(c->device));
    PeerBlob b{};
    b.magic = PEER_MAGIC;
    b.rank = c->rank;
    b.ns = c->g.ns;
    peer_settings(c, b);
    CUDA_TRY(c, cudaIpcGetMemHandle(&b.in, c->inb.base));
    CUDA_TRY(c, cudaIpcGetMemHandle(&b.arr, c->arr_dev));
    CUDA_TRY(c, cudaIpcGetMemHandle(&b.rel, c->rel_dev));
    std::memcpy(out, &b, sizeof b);
    return DSEA_OK;
}

dsea_status dsea_ring_connect_peer(dsea_ctx* c, const void* blobs, size_t blob_bytes, int32_t n_blobs)
{
    if (!c) return DSEA_EINVAL;
    if (!c->sliced) return fail(c, DSEA_ESTATE, "dsea_ring_connect_peer before dsea_slice");
    if (c->NG == 1) return DSEA_OK;
    if (!blobs || n_blobs != c->NG || blob_bytes != sizeof(PeerBlob))
        return fail(c, DSEA_EINVAL, "need %d blobs of %zu bytes", c->NG, sizeof(PeerBlob));
    if (!wait_value32()) return fail(c, DSEA_EPEER, "cuStreamWaitValue32 unavailable");
    CUDA_TRY(c, cudaSetDevice(c->device));
    const PeerBlob* B = static_cast<const PeerBlob*>(blobs);
    const int succ = (c->rank + 1) % c->NG, pred = (c->rank - 1 + c->NG) % c->NG;
    for (int r = 0; r < c->NG; r++)
        if (B[r].magic != PEER_MAGIC || B[r].rank != r || B[r].ns != c->g.ns)
            return fail(c, DSEA_EINVAL, "peer blob %d is not a dsea_ring_export of rank %d", r, r);
    {
        PeerBlob mine{};
        peer_settings(c, mine);
        for (int r = 0; r < c->NG; r++)
            if (B[r].W != mine.W || B[r].nblk != mine.nblk || B[r].plan_gap != mine.plan_gap ||
                B[r].flags != mine.flags || B[r].blocks_hash != mine.blocks_hash)
                return fail(c, DSEA_EINVAL, "rank %d was sliced or configured differently (W %d/%d, blocks %d/%d, "
                            "plan gap %d/%d, hop flags %d/%d): every rank needs the same settings",
                            r, B[r].W, mine.W, B[r].nblk, mine.nblk, B[r].plan_gap, mine.plan_gap, B[r].flags,
                            mine.flags);
    }
    void* p = nullptr;
    CUDA_TRY(c, cudaIpcOpenMemHandle(&p, B[succ].in, cudaIpcMemLazyEnablePeerAccess));
    c->succ_in_base = static_cast<char*>(p);
    CUDA_TRY(c, cudaIpcOpenMemHandle(&p, B[succ].arr, cudaIpcMemLazyEnablePeerAccess));
    c->succ_arr = static_cast<uint32_t*>(p);
    CUDA_TRY(c, cudaIpcOpenMemHandle(&p, B[pred].rel, cudaIpcMemLazyEnablePeerAccess));
    c->pred_rel = static_cast<uint32_t*>(p);
    c->peer = true;
    // release counts start at 1 for an initially empty slot, 0 for rank 0's resident state
    const int ns = c->g.ns;
    std::vector<uint32_t> init(ns, succ == 0 ? 0u : 1u);
    CUDA_TRY(c, cudaMemcpy(c->rel_dev, init.data(), sizeof(uint32_t) * ns, cudaMemcpyHostToDevice));
    CUDA_TRY(c, cudaMemset(c->arr_dev, 0, sizeof(uint32_t) * ns));
    c->wr_cnt.assign(ns, 0u);
    c->exp_arr.assign(ns, 0u);
    c->rel_cnt.assign(ns, c->rank == 0 ? 0u : 1u);
    // hop: copy engine (default; local bin + cudaMemcpyAsync over NVLink + flag write)
    // or SM remote stores (DSEA_PEER_HOP=sm: the bin kernels write the successor's slots)
    const char* hop = getenv("DSEA_PEER_HOP");
    c->ce_hop = !(hop && std::strcmp(hop, "sm") == 0);
    const char* ctr = getenv("DSEA_RING_COUNTERS");      // A/B: 0 = per-slot flags
    c->ctr = c->ce_hop && !(ctr && *ctr && atoi(ctr) == 0);
    if (c->ctr) {
        CUDA_TRY(c, cudaMemset(c->rel_dev, 0, sizeof(uint32_t) * ns));
        c->rel_init = succ == 0 ? 1u : 0u;
        c->push_k.assign(ns, 0u);
        c->rel_k.assign(ns, 0u);
        if (!c->ev_bs) CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_bs, cudaEventDisableTiming));
    }
    if (c->ce_hop && !write_value32()) return fail(c, DSEA_EPEER, "cuStreamWriteValue32 unavailable");
    if (!c->ce_hop) {
        // the last worker's output buffer is the successor's input buffer (local scratch kept)
        BufView& last = c->outb[c->W - 1];
        c->own_outb_last = last.base;
        last.base = c->succ_in_base;
        last.remote = 1;
    }
    std::fill(c->pslot_rec.begin(), c->pslot_rec.end(), 0);
    CUDA_TRY(c, cudaDeviceSynchronize());
    c->connected = true;
    return DSEA_OK;
}

dsea_status dsea_ring_disconnect(dsea_ctx* c)
{
    if (!c) return DSEA_EINVAL;
    disconnect(c);
    if (c->connected) {  // NCCL links (destroy is collective: global link order)
        if (nccl().ok) {
            const int send_link = c->rank, recv_link = (c->rank - 1 + c->NG) % c->NG;
            ncclComm_t first = send_link < recv_link ? c->send_comm : c->recv_comm;
            ncclComm_t second = send_link < recv_link ? c->recv_comm : c->send_comm;
            if (first) nccl().CommDestroy(first);
            if (second) nccl().CommDestroy(second);
        }
        c->send_comm = c->recv_comm = nullptr;
        c->connected = false;
    }
    return DSEA_OK;
}

static dsea_status step_chunk(dsea_ctx* c, int64_t n_steps);

dsea_status dsea_step(dsea_ctx* c, int64_t n_steps)
{
    if (!c) return DSEA_EINVAL;
    if (n_steps < 0) return fail(c, DSEA_EINVAL, "n_steps < 0");
    if (!c->sliced) return fail(c, DSEA_ESTATE, "dsea_step before dsea_slice");
    if (c->NG > 1 && !c->connected) return fail(c, DSEA_ESTATE, "ring not connected (dsea_ring_connect)");
    if (n_steps == 0) return DSEA_OK;
    CUDA_TRY(c, cudaSetDevice(c->device));
    // bounded memory for any n: the call runs in chunks of whole super-cycles (at most
    // ~64 MB of per-(slice, timestep) energy records and a bounded stage plan each); the
    // ring's counters carry across chunks exactly as across calls, so the result equals
    // one call (and a chunk boundary costs one pipeline fill of the ring)
    const int64_t nw = (int64_t)c->NG * c->W;
    const int64_t max_steps = std::max<int64_t>(nw, ((64ll << 20) / ((int64_t)sizeof(UnitEnergy) * c->g.ns)) / nw * nw);
    for (int64_t done = 0; done < n_steps;) {
        const int64_t n = std::min(max_steps, n_steps - done);
        dsea_status s = step_chunk(c, n);
        if (s) return s;
        done += n;
    }
    return DSEA_OK;
}

static dsea_status step_chunk(dsea_ctx* c, int64_t n_steps)
{
    const int ns = c->g.ns;
    const int64_t nw = (int64_t)c->NG * c->W;
    const int64_t rows = ((n_steps + nw - 1) / nw) * nw;
    if ((size_t)rows * ns > c->e_cap) {
        if (c->e_dev) {
            cudaFree(c->e_dev);
            c->dallocs.erase(std::remove(c->dallocs.begin(), c->dallocs.end(), (void*)c->e_dev), c->dallocs.end());
            c->e_dev = nullptr;
        }
        dsea_status s = dalloc(c, &c->e_dev, (size_t)rows * ns);
        if (s) return s;
        c->e_cap = (size_t)rows * ns;
    }
    c->mirror_valid = false;
    c->tev_used = 0;
    c->tpairs.clear();
    cudaEvent_t tl0 = nullptr;   // timeline origin (timing on and DSEA_TIMELINE set)
    const char* tl_path = c->timing ? getenv("DSEA_TIMELINE") : nullptr;
    if (tl_path) { tl0 = tev(c); cudaEventRecord(tl0, c->cs); }
    dsea_status s = c->mode == DSEA_MODE_FUSED ? run_fused(c, n_steps) : run_plan(c, n_steps);
    if (const char* hd = getenv("DSEA_HANG_DEBUG"); hd && *hd && c->timing && !s) {
        // diagnosis of a hung ring: poll the streams; after the given seconds, report per
        // stream kind how many timed ops completed and which is the first pending one
        const double limit = atof(hd);
        const auto t0 = std::chrono::steady_clock::now();
        cudaStream_t sts[] = {c->cs, c->ss, c->rs, c->es, c->bs};
        for (;;) {
            bool idle = true;
            for (cudaStream_t st : sts) idle = idle && cudaStreamQuery(st) == cudaSuccess;
            if (idle) break;
            if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
                const char* names[] = {"force", "bin", "send"};
                int done[3] = {0, 0, 0}, total[3] = {0, 0, 0}, first[3] = {-1, -1, -1};
                for (size_t k = 0; k < c->tpairs.size(); k++) {
                    const int kd = c->tpairs[k].first;
                    total[kd]++;
                    if (cudaEventQuery(c->tpairs[k].second.second) == cudaSuccess) done[kd]++;
                    else if (first[kd] < 0) first[kd] = (int)k;
                }
                for (int kd = 0; kd < 3; kd++)
                    fprintf(stderr, "[dsea hang rank %d] %s: %d of %d done, first pending timed op #%d\n", c->rank,
                            names[kd], done[kd], total[kd], first[kd]);
                const char* sn[] = {"compute", "send", "recv", "energy", "hop"};
                for (int k = 0; k < 5; k++)
                    fprintf(stderr, "[dsea hang rank %d] stream %s %s\n", c->rank, sn[k],
                            cudaStreamQuery(sts[k]) == cudaSuccess ? "idle" : "busy");
                fflush(stderr);
                break;
            }
            std::this_thread::sleep_for(std::chrono::milliseconds(20));
        }
    }
    if (s) return s;
    CUDA_TRY(c, cudaStreamSynchronize(c->cs));
    CUDA_TRY(c, cudaStreamSynchronize(c->ss));
    CUDA_TRY(c, cudaStreamSynchronize(c->rs));
    CUDA_TRY(c, cudaStreamSynchronize(c->es));
    CUDA_TRY(c, cudaStreamSynchronize(c->bs));
    CUDA_TRY(c, cudaGetLastError());
    if ((s = check_dev_err(c))) return s;

    // timing
    FILE* tl = nullptr;
    if (tl0) {   // diagnostic timeline: one CSV per rank, intervals relative to the call start
        char fn[512];
        std::snprintf(fn, sizeof fn, "%s.rank%d.csv", tl_path, c->rank);
        tl = std::fopen(fn, "w");
        if (tl) std::fprintf(tl, "kind,start_ms,end_ms\n");
    }
    for (auto& tp : c->tpairs) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, tp.second.first, tp.second.second);
        if (tp.first == TK_FORCE) c->stats.force_ms += ms;
        else if (tp.first == TK_BIN) c->stats.bin_ms += ms;
        else c->stats.hop_ms += ms;
        if (tl) {
            float a = 0.f, b = 0.f;
            cudaEventElapsedTime(&a, tl0, tp.second.first);
            cudaEventElapsedTime(&b, tl0, tp.second.second);
            std::fprintf(tl, "%s,%.4f,%.4f\n", tp.first == TK_FORCE ? "force" : tp.first == TK_BIN ? "bin" : "hop",
                         a, b);
        }
    }
    if (tl) std::fclose(tl);
    c->tpairs.clear();

    // energies of the timesteps this rank computed, summed over slices in slice order
    std::vector<UnitEnergy> he((size_t)rows * ns);
    CUDA_TRY(c, cudaMemcpy(he.data(), c->e_dev, sizeof(UnitEnergy) * he.size(), cudaMemcpyDeviceToHost));
    double last_pairs = 0;
    for (int64_t t = 0; t < n_steps; t++) {
        const int64_t owner_g = (t % nw) / c->W;
        if (c->mode == DSEA_MODE_STAGED && owner_g != c->rank) continue;
        double uc = 0, v2 = 0, k2 = 0, np = 0;
        for (int j = 0; j < ns; j++) {
            const UnitEnergy& e = he[(size_t)t * ns + j];
            uc += e.u_core; v2 += e.vir2; k2 += e.ke2; np += e.npairs;
            dsea_profile& pr = c->prof[j];
            pr.samples += 1;
            pr.n_sum += e.natoms;
            pr.U_sum += 2.0 * e.u_core + 2.0 * c->g.ushift * e.npairs;
            pr.V_sum += 0.5 * e.vir2;
            pr.KE_sum += 0.5 * e.ke2;
        }
        dsea_energy r;
        r.step = c->steps_done + t;
        r.U = 2.0 * uc + 2.0 * c->g.ushift * np;
        r.V = 0.5 * v2;
        r.KE = 0.5 * k2;
        c->energies.push_back(r);
        c->stats.atom_steps += c->N;
        last_pairs = np;
    }
    c->stats.force_pairs = (int64_t)last_pairs;
    c->steps_done += n_steps;
    c->holds_state = (c->rank == 0);
    return DSEA_OK;
}

void dsea_destroy(dsea_ctx* c)
{
    if (!c) return;
    free_device(c);
    delete c;
}

const char* dsea_last_error(const dsea_ctx* c)
{
    if (!c) return "null context";
    return c->msg.c_str();
}

dsea_status dsea_get_geometry(const dsea_ctx* c, dsea_geometry* out)
{
    if (!c || !out) return DSEA_EINVAL;
    if (!c->sliced) return DSEA_ESTATE;
    *out = c->geo;
    return DSEA_OK;
}

dsea_status dsea_get_positions(dsea_ctx* c, double* xyz, int64_t n) { return get_vec(c, xyz, n, 0); }
dsea_status dsea_get_velocities(dsea_ctx* c, double* v, int64_t n) { return get_vec(c, v, n, 1); }
dsea_status dsea_get_forces(dsea_ctx* c, double* f, int64_t n) { return get_vec(c, f, n, 2); }

dsea_status dsea_get_cells(dsea_ctx* c, int32_t* cell_xyz, int32_t* slice, int64_t n)
{
    if (!c) return DSEA_EINVAL;
    if (!cell_xyz || !slice || n != c->N) return fail(c, DSEA_EINVAL, "array of %lld atoms expected", (long long)c->N);
    if (!c->sliced) return fail(c, DSEA_ESTATE, "dsea_get_cells before dsea_slice");
    if (!c->holds_state) return fail(c, DSEA_ESTATE, "this rank does not hold the state (rank 0 does)");
    dsea_status s = fetch_mirror(c);
    if (s) return s;
    const int CY = c->g.cells[1], CZ = c->g.cells[2];
    for_each_atom(c, [&](int j, int, int cell, int id, const char*) {
        const int cxl = cell / (CY * CZ);
        cell_xyz[3 * (int64_t)id + 0] = j * c->g.c + cxl;
        cell_xyz[3 * (int64_t)id + 1] = (cell / CZ) % CY;
        cell_xyz[3 * (int64_t)id + 2] = cell % CZ;
        slice[id] = j;
    });
    return DSEA_OK;
}

dsea_status dsea_get_slice(dsea_ctx* c, int32_t j, double* xyz, double* v, double* f, int32_t* ids, int64_t cap,
                           int64_t* n_written)
{
    if (!c || !n_written) return DSEA_EINVAL;
    if (!c->sliced) return fail(c, DSEA_ESTATE, "dsea_get_slice before dsea_slice");
    if (j < 0 || j >= c->g.ns) return fail(c, DSEA_EINVAL, "slice %d outside [0, %d)", j, c->g.ns);
    if (!c->holds_state) return fail(c, DSEA_ESTATE, "this rank does not hold the state (rank 0 does)");
    CUDA_TRY(c, cudaSetDevice(c->device));
    const char* slot = c->inb.base + (size_t)(j % c->inb.nslots) * c->L.slot_bytes;
    int32_t n = 0;
    CUDA_TRY(c, cudaMemcpy(&n, slot + sizeof(int32_t) * (size_t)c->g.ncell, sizeof n, cudaMemcpyDeviceToHost));
    *n_written = n;
    const int64_t k = std::min<int64_t>(cap, n);
    if (k <= 0) return DSEA_OK;
    std::vector<double> a((size_t)k), b((size_t)k), d((size_t)k);
    auto aos = [&](double* out, size_t ox, size_t oy, size_t oz) -> dsea_status {
        if (!out) return DSEA_OK;
        CUDA_TRY(c, cudaMemcpy(a.data(), slot + ox, sizeof(double) * k, cudaMemcpyDeviceToHost));
        CUDA_TRY(c, cudaMemcpy(b.data(), slot + oy, sizeof(double) * k, cudaMemcpyDeviceToHost));
        CUDA_TRY(c, cudaMemcpy(d.data(), slot + oz, sizeof(double) * k, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < k; i++) { out[3 * i] = a[(size_t)i]; out[3 * i + 1] = b[(size_t)i]; out[3 * i + 2] = d[(size_t)i]; }
        return DSEA_OK;
    };
    dsea_status s;
    if ((s = aos(xyz, c->L.off_x, c->L.off_y, c->L.off_z))) return s;
    if ((s = aos(v, c->L.off_vx, c->L.off_vy, c->L.off_vz))) return s;
    if ((s = aos(f, c->L.off_fx, c->L.off_fy, c->L.off_fz))) return s;
    if (ids) CUDA_TRY(c, cudaMemcpy(ids, slot + c->L.off_id, sizeof(int32_t) * k, cudaMemcpyDeviceToHost));
    return DSEA_OK;
}

dsea_status dsea_set_thermostat(dsea_ctx* c, int32_t enable, double T_target)
{
    if (!c) return DSEA_EINVAL;
    if (enable && !(std::isfinite(T_target) && T_target > 0.0))
        return fail(c, DSEA_EINVAL, "thermostat temperature must be > 0 (got %g)", T_target);
    if (!c->sliced) return fail(c, DSEA_ESTATE, "dsea_set_thermostat before dsea_slice");
    c->g.thermo = enable ? 1 : 0;
    c->g.T_target = enable ? T_target : 0.0;
    return DSEA_OK;
}

dsea_status dsea_get_profiles(dsea_ctx* c, dsea_profile* out, int32_t n_slices)
{
    if (!c || !out) return DSEA_EINVAL;
    if (!c->sliced) return fail(c, DSEA_ESTATE, "dsea_get_profiles before dsea_slice");
    if (n_slices != c->g.ns) return fail(c, DSEA_EINVAL, "%d slices expected", c->g.ns);
    for (int j = 0; j < n_slices; j++) out[j] = c->prof[(size_t)j];
    return DSEA_OK;
}

dsea_status dsea_reset_profiles(dsea_ctx* c)
{
    if (!c) return DSEA_EINVAL;
    for (auto& p : c->prof) p = dsea_profile{};
    return DSEA_OK;
}

dsea_status dsea_thermo_compute(const dsea_energy* in, int64_t n, int64_t n_atoms, double volume, dsea_thermo* out)
{
    if (n < 0 || n_atoms <= 0 || !(volume > 0.0) || (n > 0 && (!in || !out))) return DSEA_EINVAL;
    const double N = (double)n_atoms, rho = N / volume;
    for (int64_t i = 0; i < n; i++) {
        const dsea_energy& e = in[i];
        dsea_thermo& t = out[i];
        t.step = e.step;
        t.T = 2.0 * e.KE / (3.0 * N);                      // k_B = m = 1, 3N dof (Q9, Q11)
        t.p = rho * t.T + 24.0 * e.V / (3.0 * volume);     // Alg. 1's V: sum r.F = 24 V (Q24)
        t.u = e.U / N;
        t.e = (e.U + e.KE) / N;
    }
    return DSEA_OK;
}

dsea_status dsea_xprofile_compute(const dsea_profile* raw, int32_t n_slices, const dsea_geometry* geo,
                                  dsea_xprofile* out)
{
    if (!raw || !geo || !out || n_slices != geo->n_slices || n_slices < 1) return DSEA_EINVAL;
    const double vol = geo->w * geo->b[1] * geo->b[2];    // slice volume
    for (int j = 0; j < n_slices; j++) {
        const dsea_profile& r = raw[j];
        dsea_xprofile& o = out[j];
        const double s = r.samples > 0 ? (double)r.samples : 1.0;
        const double n = r.n_sum / s, ke = r.KE_sum / s, U = r.U_sum / s, V = r.V_sum / s;
        o.x = (j + 0.5) * geo->w;
        o.n = n;
        o.rho = n / vol;
        o.T = n > 0 ? 2.0 * ke / (3.0 * n) : 0.0;
        o.u = n > 0 ? U / n : 0.0;
        o.p = o.rho * o.T + 24.0 * V / (3.0 * vol);
        o.samples = r.samples;
    }
    return DSEA_OK;
}

dsea_status dsea_get_energies(dsea_ctx* c, dsea_energy* out, int64_t cap, int64_t* n_written)
{
    if (!c || !n_written) return DSEA_EINVAL;
    const int64_t n = std::min<int64_t>(cap, (int64_t)c->energies.size());
    if (n > 0 && !out) return fail(c, DSEA_EINVAL, "null output");
    for (int64_t i = 0; i < n; i++) out[i] = c->energies[(size_t)i];
    *n_written = n < 0 ? 0 : n;
    return DSEA_OK;
}

dsea_status dsea_set_state(dsea_ctx* c, const double* xyz, const double* v, const double* f, int64_t n)
{
    if (!c) return DSEA_EINVAL;
    if (!xyz || !v || n != c->N) return fail(c, DSEA_EINVAL, "positions and velocities of %lld atoms expected", (long long)c->N);
    if (!c->sliced) {
        c->h_xyz.assign(xyz, xyz + 3 * n);
        c->h_v.assign(v, v + 3 * n);
        if (f) c->h_f.assign(f, f + 3 * n);
        else c->h_f.clear();
        return DSEA_OK;
    }
    if (c->NG > 1 && c->rank != 0) return DSEA_OK;
    CUDA_TRY(c, cudaSetDevice(c->device));
    return upload_state(c, xyz, v, f);
}

dsea_status dsea_set_timing(dsea_ctx* c, int32_t enable)
{
    if (!c) return DSEA_EINVAL;
    c->timing = enable != 0;
    return DSEA_OK;
}

dsea_status dsea_get_stats(dsea_ctx* c, dsea_stats* out)
{
    if (!c || !out) return DSEA_EINVAL;
    *out = c->stats;
    return DSEA_OK;
}

dsea_status dsea_reset_stats(dsea_ctx* c)
{
    if (!c) return DSEA_EINVAL;
    std::memset(&c->stats, 0, sizeof c->stats);
    return DSEA_OK;
}

dsea_status dsea_plan_ops(int32_t n_slices, int32_t n_gpus, int32_t rank, int32_t W, int64_t n_steps,
                          int32_t slices_per_stage, int32_t* rows, int64_t cap_rows, int64_t* n_rows)
{
    if (!n_rows || n_slices < 1 || n_gpus < 1 || rank < 0 || rank >= n_gpus || W < 1 || n_steps < 0 ||
        slices_per_stage < 1 || slices_per_stage > n_slices)
        return DSEA_EINVAL;
    Plan P = build_plan(n_slices, n_gpus, rank, W, n_steps, make_blocks(n_slices, n_gpus, slices_per_stage));
    order_pushes(P.ops, W);   // as executed with the default copy-engine hop
    *n_rows = (int64_t)P.ops.size();
    if (!rows) return DSEA_OK;
    const int64_t n = std::min<int64_t>(cap_rows, (int64_t)P.ops.size());
    for (int64_t i = 0; i < n; i++) {
        const Op& op = P.ops[(size_t)i];
        int32_t* r = rows + 7 * i;
        r[0] = op.kind; r[1] = op.stage; r[2] = op.worker; r[3] = op.slice; r[4] = op.count;
        r[5] = op.cycle; r[6] = (int32_t)op.t_rel;
    }
    *n_rows = n;
    return DSEA_OK;
}

dsea_status dsea_schedule(int32_t n_slices, int32_t n_gpus, int32_t rank, int32_t W, int32_t n_cycles,
                          int32_t* rows, int64_t cap_rows, int64_t* n_rows)
{
    if (!n_rows || n_slices < 1 || n_gpus < 1 || rank < 0 || rank >= n_gpus || W < 1 || n_cycles < 0)
        return DSEA_EINVAL;
    const int64_t n_steps = (int64_t)n_cycles * n_gpus * W;
    const Plan P = build_plan(n_slices, n_gpus, rank, W, n_steps, make_blocks(n_slices, n_gpus, 1));
    // one row per (stage, worker) doing something; recv rows carry worker -1
    std::vector<std::array<int32_t, 8>> out;
    auto row_for = [&](int stage, int worker) -> std::array<int32_t, 8>& {
        for (auto& r : out)
            if (r[0] == stage && r[2] == worker) return r;
        out.push_back({stage, -1, worker, -1, -1, -1, -1, -1});
        return out.back();
    };
    for (const Op& op : P.ops) {
        const int st = op.stage + 1;  // 1-based like Table 1
        switch (op.kind) {
        case OP_RECV: row_for(st, -1)[1] = op.slice + 1; row_for(st, -1)[6] = op.cycle; break;
        case OP_FORCE:
        case OP_PASS: {
            auto& r = row_for(st, op.worker);
            r[3] = op.slice + 1; r[6] = op.cycle; r[7] = op.kind == OP_FORCE ? (int32_t)op.t_rel : -1;
            break;
        }
        // a worker may finalise two runs in one stage (W > 1: the super-cycle's last
        // slice goes with its own block): the second one gets a row of its own
        case OP_BIN: {
            auto* r = &row_for(st, op.worker);
            if ((*r)[4] >= 0) { out.push_back({st, -1, op.worker, -1, -1, -1, -1, -1}); r = &out.back(); }
            (*r)[4] = op.slice + 1;
            break;
        }
        case OP_SEND: {
            std::array<int32_t, 8>* r = nullptr;
            for (auto& q : out)   // the first row of this (stage, worker) with a free send field
                if (q[0] == st && q[2] == op.worker && q[5] < 0) { r = &q; break; }
            if (!r) { out.push_back({st, -1, op.worker, -1, -1, -1, -1, -1}); r = &out.back(); }
            (*r)[5] = op.slice + 1;
            break;
        }
        }
    }
    if (n_gpus == 1) {
        // single GPU: slices of the first super-cycle are loaded from storage at
        // stages 1..N_S; show them as receives like Table 1
        for (int j = 0; j < n_slices && n_cycles > 0; j++) {
            auto& r = row_for(j + 1, -1);
            r[1] = j + 1; r[6] = 0;
        }
    } else if (rank == 0) {
        for (int j = 0; j < n_slices && n_cycles > 0; j++) {
            auto& r = row_for(j + 1, -1);
            if (r[1] < 0) { r[1] = j + 1; r[6] = 0; }
        }
    }
    std::stable_sort(out.begin(), out.end(), [](const std::array<int32_t, 8>& x, const std::array<int32_t, 8>& y) {
        return x[0] != y[0] ? x[0] < y[0] : x[2] < y[2];
    });
    *n_rows = (int64_t)out.size();
    if (rows) {
        if (cap_rows < (int64_t)out.size()) return DSEA_EINVAL;
        for (size_t i = 0; i < out.size(); i++)
            for (int k = 0; k < 8; k++) rows[i * 8 + k] = out[i][k];
    }
    return DSEA_OK;
}

}  // extern "C"
