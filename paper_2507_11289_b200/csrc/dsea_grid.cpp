// dsea_grid.cpp -- C ABI and runtime of the stencil workload (include/dsea_grid.h):
// the second DSEA application.  The worker is the FTCS
// kernel of dsea_grid_kernels.cu (O_in = 1, O_out = 0, §3); everything else
// is the framework: the stage plan of dsea_plan.h (Table 1 generalised, P:146-195
// §3.3, shared with the MD engine), slot buffers per worker (§3.1), and the
// NVLink ring hop with arrival/release flags (§3.1, §3.4).
//
// Buffers (one context per GPU): the input buffer (N_S slots) and one output buffer
// per worker; a slot is the p x ny x nz doubles of one slice, so each buffer is also
// the whole field in x-major order and a block of slices is one contiguous range.
//  - FORCE (worker w, block): the stencil of the block's planes from w's input
//    buffer (neighbour planes from the adjacent slots) into w's output buffer;
//  - BIN (finalise; O_out = 0, so the slices are already final): the last worker
//    pushes them to the ring successor (copy engine + flag write), or, on a ring of
//    one, copies them back into the input buffer;
//  - PASS: a trailing partial super-cycle copies the block through (reading Q15).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dsea_grid.h"
#include "dsea_plan.h"

namespace dsea {
void ftcs_launch(const double* in, double* out, int x0, int x1, int nx, int ny, int nz, double r, bool pdl,
                 cudaStream_t s);
}
using namespace dsea;

namespace {
struct GridBlob {
    int32_t magic, rank, ns, pad;
    int64_t slot_bytes;
    cudaIpcMemHandle_t in, arr, rel;
};
constexpr int32_t GRID_MAGIC = 0x44534547;  // "DSEG"
}  // namespace

struct dsea_grid {
    dsea_grid_params p{};
    int ns = 0, pl = 0, W = 1, NG = 1, rank = 0, device = 0, mode = 0;
    size_t plane = 0, slot_elems = 0, slot_bytes = 0;
    Blocks bl;
    cudaStream_t cs = nullptr, hs = nullptr;   // compute, hop
    double* inb = nullptr;
    std::vector<double*> outb;
    // Ring flags: one monotone counter per direction instead of one flag per slot.
    // Slots arrive, and are released, in (super-cycle, slot) order, so the k-th
    // arrival (release) of slot s is event number (k-1) N_S + s + 1 of its stream:
    // the sender publishes the number of its last slot pushed, the receiver the
    // number of its last slot released -- one stream write / wait per block, not one
    // per slot (the per-slot flags cost ~40 us of stream memory operations per block,
    // more than a block's stencil pass).
    uint32_t* arr_dev = nullptr;               // [1] arrivals into my input buffer
    uint32_t* rel_dev = nullptr;               // [1] releases of my successor's slots
    double* succ_in = nullptr;                 // mapped successor input buffer
    uint32_t* succ_arr = nullptr;              // mapped successor arrival counter
    uint32_t* pred_rel = nullptr;              // mapped predecessor release counter
    bool peer = false;
    std::vector<uint32_t> push_k, exp_arr, rel_k;   // per slot: pushes made, arrivals expected, releases made
    uint32_t rel_init = 0;                     // 1 if the successor's slots start occupied (successor = rank 0)
    std::vector<cudaEvent_t> ev_hop;           // per block: last push of the run keyed by it
    std::vector<char> hop_rec;
    cudaEvent_t ev_cs = nullptr;
    bool timing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tpairs;
    dsea_grid_stats stats{};
    std::string msg;
};

namespace {
dsea_status gfail(dsea_grid* c, dsea_status s, const char* fmt, ...)
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

#define GTRY(c, expr)                                                                              \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return gfail(c, e_ == cudaErrorMemoryAllocation ? DSEA_ENOMEM : DSEA_ECUDA, "%s: %s", \
                         #expr, cudaGetErrorString(e_));                                           \
    } while (0)

bool pdl_enabled()
{
    const char* e = getenv("DSEA_PDL");
    return !(e && *e && atoi(e) == 0);
}

void stencil(dsea_grid* c, const double* in, double* out, int j, int n)
{
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (c->timing) {
        cudaEventCreate(&t0);
        cudaEventCreate(&t1);
        cudaEventRecord(t0, c->cs);
    }
    ftcs_launch(in, out, j * c->pl, (j + n) * c->pl, c->p.nx, c->p.ny, c->p.nz, c->p.r, pdl_enabled(), c->cs);
    if (c->timing) {
        cudaEventRecord(t1, c->cs);
        c->tpairs.push_back({t0, t1});
    }
    c->stats.kernel_launches++;
    c->stats.cell_steps += (int64_t)n * (int64_t)c->slot_elems;
}

dsea_status collect_timing(dsea_grid* c)
{
    for (auto& tp : c->tpairs) {
        float ms = 0;
        GTRY(c, cudaEventElapsedTime(&ms, tp.first, tp.second));
        c->stats.stencil_ms += ms;
        c->stats.stencil_launches++;
        cudaEventDestroy(tp.first);
        cudaEventDestroy(tp.second);
    }
    c->tpairs.clear();
    return DSEA_OK;
}

dsea_status run_fused(dsea_grid* c, int64_t n_steps)
{
    for (int64_t t = 0; t < n_steps; t++) {
        stencil(c, c->inb, c->outb[0], 0, c->ns);
        std::swap(c->inb, c->outb[0]);    // the field stays in the input buffer
    }
    return DSEA_OK;
}

dsea_status run_plan(dsea_grid* c, int64_t n_steps)
{
    const int ns = c->ns, W = c->W;
    const bool ring = c->NG > 1;
    const size_t sb = c->slot_bytes, se = c->slot_elems;
    const Plan P = build_plan(ns, c->NG, c->rank, W, n_steps, c->bl);
    auto in_of = [&](int w) { return w == 0 ? c->inb : c->outb[w - 1]; };
    auto ev_no = [&](uint32_t k, int s) { return (k - 1) * (uint32_t)ns + (uint32_t)s + 1; };
    auto release = [&](int f0, int f1) -> dsea_status {   // slots [f0, f1] read for the last time
        if (f1 < f0) return DSEA_OK;
        for (int sl = f0; sl <= f1; sl++) c->rel_k[sl]++;
        if (stream_write32(c->cs, c->pred_rel, ev_no(c->rel_k[f1], f1)))
            return gfail(c, DSEA_EPEER, "cuStreamWriteValue32 (release) failed");
        return DSEA_OK;
    };
    auto wait_arrival = [&](int s) -> dsea_status {        // the latest expected arrival of slot s
        if (stream_wait_geq32(c->cs, c->arr_dev, ev_no(c->exp_arr[s], s)))
            return gfail(c, DSEA_EPEER, "cuStreamWaitValue32 (arrival) failed");
        return DSEA_OK;
    };
    // push slots [m, m+n) of `src` to the successor on the hop stream (after the
    // compute-stream work so far): wait until it released their previous occupants,
    // copy over NVLink, publish the arrival number of the last slot
    auto push = [&](const double* src, int m, int n) -> dsea_status {
        GTRY(c, cudaEventRecord(c->ev_cs, c->cs));
        GTRY(c, cudaStreamWaitEvent(c->hs, c->ev_cs, 0));
        for (int sl = m; sl < m + n; sl++) c->push_k[sl]++;
        const uint32_t j = c->push_k[m + n - 1] - 1 + c->rel_init;   // release needed of the last slot
        if (j > 0 && stream_wait_geq32(c->hs, c->rel_dev, ev_no(j, m + n - 1)))
            return gfail(c, DSEA_EPEER, "cuStreamWaitValue32 (release) failed");
        GTRY(c, cudaMemcpyAsync(c->succ_in + (size_t)m * se, src, sb * n, cudaMemcpyDeviceToDevice, c->hs));
        if (stream_write32(c->hs, c->succ_arr, ev_no(c->push_k[m + n - 1], m + n - 1)))
            return gfail(c, DSEA_EPEER, "cuStreamWriteValue32 (arrival) failed");
        const int key = c->bl.of[m + n - 1];
        GTRY(c, cudaEventRecord(c->ev_hop[key], c->hs));
        c->hop_rec[key] = 1;
        c->stats.hop_bytes += (int64_t)sb * n;
        return DSEA_OK;
    };
    // pushes must leave in (super-cycle, slot) order for the counters (order_pushes)
    std::vector<Op> ops = P.ops;
    order_pushes(ops, W);
    for (const Op& op : ops) {
        switch (op.kind) {
        case OP_RECV:
            if (ring) c->exp_arr[op.slice]++;
            break;
        case OP_FORCE: {
            const int j = op.slice, n = op.count, w = op.worker;
            if (w == 0 && ring && !(c->rank == 0 && op.cycle == 0)) {
                dsea_status s = wait_arrival(std::min(j + n, ns - 1));   // right neighbour of the block
                if (s) return s;
            }
            if (ring && w == W - 1) {
                // the pushes that last read these output slots (runs keyed by the block of
                // their last slot: this block's and the next one's) must be done
                const int k1 = std::min(c->bl.of[j + n - 1] + 1, c->bl.n() - 1);
                for (int k = c->bl.of[j]; k <= k1; k++)
                    if (c->hop_rec[k]) GTRY(c, cudaStreamWaitEvent(c->cs, c->ev_hop[k], 0));
            }
            stencil(c, in_of(w), c->outb[w], j, n);
            if (w == 0 && ring) {
                dsea_status s = release(std::max(j - 1, 0), (j + n == ns) ? ns - 1 : j + n - 2);
                if (s) return s;
            }
            break;
        }
        case OP_PASS: {
            const int j = op.slice, n = op.count, w = op.worker;
            if (w == 0 && ring && !(c->rank == 0 && op.cycle == 0)) {
                dsea_status s = wait_arrival(j + n - 1);
                if (s) return s;
            }
            const double* src = in_of(w) + (size_t)j * se;
            if (ring && w == W - 1) {               // straight into the successor's slots
                dsea_status s = push(src, j, n);    // (on the hop stream: pushes stay in order)
                if (s) return s;
            } else {
                double* dst = (!ring && w == W - 1) ? c->inb : c->outb[w];
                if (dst + (size_t)j * se != src)
                    GTRY(c, cudaMemcpyAsync(dst + (size_t)j * se, src, sb * n, cudaMemcpyDeviceToDevice, c->cs));
            }
            if (w == 0 && ring) {
                dsea_status s = release(j, j + n - 1);
                if (s) return s;
            }
            break;
        }
        case OP_BIN: {
            const int m = op.slice, n = op.count, w = op.worker;
            if (w != W - 1) break;                  // O_out = 0: already final in outb[w]
            const double* src = c->outb[W - 1] + (size_t)m * se;
            if (!ring) {                            // ring of one: back into the input buffer
                GTRY(c, cudaMemcpyAsync(c->inb + (size_t)m * se, src, sb * n, cudaMemcpyDeviceToDevice, c->cs));
                break;
            }
            dsea_status s = push(src, m, n);
            if (s) return s;
            break;
        }
        default:                                    // OP_SEND: the push happened in BIN / PASS
            break;
        }
    }
    if (ring && c->rank == 0 && c->exp_arr[ns - 1] > 0) {   // the final super-cycle lands on rank 0 (Q22)
        dsea_status s = wait_arrival(ns - 1);
        if (s) return s;
    }
    return DSEA_OK;
}

void free_all(dsea_grid* c)
{
    if (c->device >= 0) cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    if (c->succ_in) cudaIpcCloseMemHandle(c->succ_in);
    if (c->succ_arr) cudaIpcCloseMemHandle(c->succ_arr);
    if (c->pred_rel) cudaIpcCloseMemHandle(c->pred_rel);
    c->succ_in = nullptr; c->succ_arr = nullptr; c->pred_rel = nullptr; c->peer = false;
    if (c->inb) cudaFree(c->inb);
    for (double* o : c->outb) if (o) cudaFree(o);
    c->inb = nullptr; c->outb.clear();
    if (c->arr_dev) cudaFree(c->arr_dev);
    if (c->rel_dev) cudaFree(c->rel_dev);
    c->arr_dev = c->rel_dev = nullptr;
    for (auto e : c->ev_hop) cudaEventDestroy(e);
    c->ev_hop.clear();
    if (c->ev_cs) cudaEventDestroy(c->ev_cs);
    if (c->cs) cudaStreamDestroy(c->cs);
    if (c->hs) cudaStreamDestroy(c->hs);
    c->ev_cs = nullptr; c->cs = c->hs = nullptr;
}
}  // namespace

extern "C" {

dsea_status dsea_grid_create(const dsea_grid_params* p, dsea_grid** out)
{
    if (!out) return DSEA_EINVAL;
    *out = nullptr;
    if (!p) return DSEA_EINVAL;
    dsea_grid* c = new (std::nothrow) dsea_grid();
    if (!c) return DSEA_ENOMEM;
    c->device = -1;
    auto bad = [&](dsea_status s) { free_all(c); delete c; return s; };
    if (p->nx < 3 || p->ny < 3 || p->nz < 3 || p->n_slices < 3 || p->nx % p->n_slices != 0 ||
        !(p->r > 0.0 && p->r <= 1.0 / 6.0) || p->n_gpus < 1 || p->rank < 0 || p->rank >= p->n_gpus ||
        p->workers_per_gpu < 1 || p->mode < 0 || p->mode > 2 || p->slices_per_stage < 0 ||
        p->slices_per_stage > p->n_slices || (p->mode == 1 && (p->n_gpus > 1 || p->workers_per_gpu > 1)))
        return bad(DSEA_EINVAL);
    c->p = *p;
    c->ns = p->n_slices;
    c->pl = p->nx / p->n_slices;
    c->W = p->workers_per_gpu;
    c->NG = p->n_gpus;
    c->rank = p->rank;
    c->plane = (size_t)p->ny * p->nz;
    c->slot_elems = (size_t)c->pl * c->plane;
    c->slot_bytes = c->slot_elems * sizeof(double);
    c->mode = p->mode == 0 ? ((c->NG == 1 && c->W == 1) ? 1 : 2) : p->mode;
    int B = p->slices_per_stage;
    if (B == 0) {
        // ~32M cells per launch (~80 us of HBM time) with >= N_GPU (2 + W) - 1 blocks
        const double cells = (double)p->nx * p->ny * p->nz;
        const int depth = c->NG > 1 ? c->NG * (2 + c->W) - 1 : 2 + c->W;
        const int nb = std::max((int)std::ceil(cells / 3.2e7), depth);
        B = std::max(1, (c->ns + nb - 1) / nb);
        while (B > 1 && (c->ns + B - 1) / B < depth) B--;
    }
    c->bl = make_blocks(c->ns, c->NG, B);
    if (c->mode == 2 && c->NG == 1) {
        const bool ok = B == 1 ? c->ns >= 2 + 2 * c->W : c->bl.n() >= 2 + c->W;
        if (!ok) return bad(DSEA_EINVAL);
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1 || p->device < 0 || p->device >= ndev) {
        cudaGetLastError();
        return bad(DSEA_ECUDA);
    }
    c->device = p->device;
    if (cudaSetDevice(c->device) != cudaSuccess) return bad(DSEA_ECUDA);
    const size_t bytes = c->slot_bytes * c->ns;
    if (cudaMalloc(&c->inb, bytes) != cudaSuccess) { cudaGetLastError(); return bad(DSEA_ENOMEM); }
    c->outb.assign(c->W, nullptr);
    for (int w = 0; w < c->W; w++)
        if (cudaMalloc(&c->outb[w], bytes) != cudaSuccess) { cudaGetLastError(); return bad(DSEA_ENOMEM); }
    if (cudaMalloc(&c->arr_dev, sizeof(uint32_t) * c->ns) != cudaSuccess ||
        cudaMalloc(&c->rel_dev, sizeof(uint32_t) * c->ns) != cudaSuccess) {
        cudaGetLastError();
        return bad(DSEA_ENOMEM);
    }
    if (cudaMemset(c->inb, 0, bytes) != cudaSuccess || cudaMemset(c->arr_dev, 0, sizeof(uint32_t) * c->ns) ||
        cudaMemset(c->rel_dev, 0, sizeof(uint32_t) * c->ns) ||
        cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->hs, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_cs, cudaEventDisableTiming) != cudaSuccess)
        return bad(DSEA_ECUDA);
    c->ev_hop.resize(c->bl.n());
    for (auto& e : c->ev_hop)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return bad(DSEA_ECUDA);
    c->hop_rec.assign(c->bl.n(), 0);
    c->push_k.assign(c->ns, 0u);
    c->exp_arr.assign(c->ns, 0u);
    c->rel_k.assign(c->ns, 0u);
    *out = c;
    return DSEA_OK;
}

dsea_status dsea_grid_set_field(dsea_grid* c, const double* u, int64_t n)
{
    if (!c) return DSEA_EINVAL;
    if (!u || n != (int64_t)c->p.nx * c->p.ny * c->p.nz) return gfail(c, DSEA_EINVAL, "need %lld cells",
                                                                      (long long)c->p.nx * c->p.ny * c->p.nz);
    if (c->rank != 0) return gfail(c, DSEA_ESTATE, "the field is loaded on rank 0 (P:93)");
    GTRY(c, cudaSetDevice(c->device));
    GTRY(c, cudaMemcpy(c->inb, u, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice));
    return DSEA_OK;
}

dsea_status dsea_grid_get_field(dsea_grid* c, double* u, int64_t n)
{
    if (!c) return DSEA_EINVAL;
    if (!u || n != (int64_t)c->p.nx * c->p.ny * c->p.nz) return gfail(c, DSEA_EINVAL, "need %lld cells",
                                                                      (long long)c->p.nx * c->p.ny * c->p.nz);
    if (c->rank != 0) return gfail(c, DSEA_ESTATE, "the field rests on rank 0 (Q22)");
    GTRY(c, cudaSetDevice(c->device));
    GTRY(c, cudaStreamSynchronize(c->cs));
    GTRY(c, cudaMemcpy(u, c->inb, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost));
    return DSEA_OK;
}

dsea_status dsea_grid_ring_export(dsea_grid* c, void* out, size_t cap, size_t* len)
{
    if (!c || !len) return DSEA_EINVAL;
    *len = sizeof(GridBlob);
    if (!out) return DSEA_OK;
    if (cap < sizeof(GridBlob)) return gfail(c, DSEA_EINVAL, "export buffer needs %zu bytes", sizeof(GridBlob));
    GTRY(c, cudaSetDevice(c->device));
    GridBlob b{};
    b.magic = GRID_MAGIC;
    b.rank = c->rank;
    b.ns = c->ns;
    b.slot_bytes = (int64_t)c->slot_bytes;
    GTRY(c, cudaIpcGetMemHandle(&b.in, c->inb));
    GTRY(c, cudaIpcGetMemHandle(&b.arr, c->arr_dev));
    GTRY(c, cudaIpcGetMemHandle(&b.rel, c->rel_dev));
    std::memcpy(out, &b, sizeof b);
    return DSEA_OK;
}

dsea_status dsea_grid_ring_connect_peer(dsea_grid* c, const void* blobs, size_t blob_bytes, int32_t n_blobs)
{
    if (!c) return DSEA_EINVAL;
    if (c->NG == 1) return DSEA_OK;
    if (!blobs || n_blobs != c->NG || blob_bytes != sizeof(GridBlob))
        return gfail(c, DSEA_EINVAL, "need %d blobs of %zu bytes", c->NG, sizeof(GridBlob));
    if (!stream_memops_available()) return gfail(c, DSEA_EPEER, "stream memory operations unavailable");
    GTRY(c, cudaSetDevice(c->device));
    const GridBlob* B = static_cast<const GridBlob*>(blobs);
    const int succ = (c->rank + 1) % c->NG, pred = (c->rank - 1 + c->NG) % c->NG;
    for (int r = 0; r < c->NG; r++)
        if (B[r].magic != GRID_MAGIC || B[r].rank != r || B[r].ns != c->ns ||
            B[r].slot_bytes != (int64_t)c->slot_bytes)
            return gfail(c, DSEA_EINVAL, "peer blob %d is not a dsea_grid_ring_export of rank %d", r, r);
    void* q = nullptr;
    GTRY(c, cudaIpcOpenMemHandle(&q, B[succ].in, cudaIpcMemLazyEnablePeerAccess));
    c->succ_in = static_cast<double*>(q);
    GTRY(c, cudaIpcOpenMemHandle(&q, B[succ].arr, cudaIpcMemLazyEnablePeerAccess));
    c->succ_arr = static_cast<uint32_t*>(q);
    GTRY(c, cudaIpcOpenMemHandle(&q, B[pred].rel, cudaIpcMemLazyEnablePeerAccess));
    c->pred_rel = static_cast<uint32_t*>(q);
    // release counts start at 1 for an initially empty slot, 0 for rank 0's resident field
    GTRY(c, cudaMemset(c->rel_dev, 0, sizeof(uint32_t)));
    GTRY(c, cudaMemset(c->arr_dev, 0, sizeof(uint32_t)));
    c->rel_init = succ == 0 ? 1u : 0u;
    c->push_k.assign(c->ns, 0u);
    c->exp_arr.assign(c->ns, 0u);
    c->rel_k.assign(c->ns, 0u);
    c->peer = true;
    return DSEA_OK;
}

dsea_status dsea_grid_ring_disconnect(dsea_grid* c)
{
    if (!c) return DSEA_EINVAL;
    GTRY(c, cudaSetDevice(c->device));
    GTRY(c, cudaDeviceSynchronize());
    if (c->succ_in) cudaIpcCloseMemHandle(c->succ_in);
    if (c->succ_arr) cudaIpcCloseMemHandle(c->succ_arr);
    if (c->pred_rel) cudaIpcCloseMemHandle(c->pred_rel);
    c->succ_in = nullptr; c->succ_arr = nullptr; c->pred_rel = nullptr;
    c->peer = false;
    return DSEA_OK;
}

dsea_status dsea_grid_step(dsea_grid* c, int64_t n_steps)
{
    if (!c || n_steps < 0) return DSEA_EINVAL;
    if (c->NG > 1 && !c->peer) return gfail(c, DSEA_ESTATE, "ring of %d GPUs not connected", c->NG);
    GTRY(c, cudaSetDevice(c->device));
    dsea_status s = c->mode == 1 ? run_fused(c, n_steps) : run_plan(c, n_steps);
    if (s) return s;
    GTRY(c, cudaStreamSynchronize(c->cs));
    GTRY(c, cudaStreamSynchronize(c->hs));
    GTRY(c, cudaGetLastError());
    return collect_timing(c);
}

dsea_status dsea_grid_set_timing(dsea_grid* c, int32_t enable)
{
    if (!c) return DSEA_EINVAL;
    c->timing = enable != 0;
    return DSEA_OK;
}

dsea_status dsea_grid_get_stats(dsea_grid* c, dsea_grid_stats* out)
{
    if (!c || !out) return DSEA_EINVAL;
    *out = c->stats;
    return DSEA_OK;
}

dsea_status dsea_grid_reset_stats(dsea_grid* c)
{
    if (!c) return DSEA_EINVAL;
    std::memset(&c->stats, 0, sizeof c->stats);
    return DSEA_OK;
}

const char* dsea_grid_last_error(const dsea_grid* c)
{
    return c ? c->msg.c_str() : "null context";
}

void dsea_grid_destroy(dsea_grid* c)
{
    if (!c) return;
    free_all(c);
    delete c;
}

}  // extern "C"
