// dsea_device.cuh -- device helpers shared by the sm_100a kernels of the DSEAmd hot
// path (dsea_kernels.cu: pipelined force kernel, bins, energies; dsea_force.cu: the
// tiled force kernel).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cmath>
#include <cstdlib>
#include "dsea_internal.h"
#include "../../include/dsea.h"

namespace dsea {

#define FULLMASK 0xffffffffu

// Programmatic dependent launch (PDL): kernels of the compute-stream chain (force ->
// bin scan -> place -> gather -> next force) are launched with programmatic stream
// serialisation, so a launch and its CTAs' prologue overlap the predecessor's tail.
// pdl_wait() blocks until the predecessor grid has completed and its memory is
// visible (a no-op without PDL); pdl_release() lets the successor launch early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void set_err(DevErr* e, int code, int slice, int atom, int aux) {
    if (atomicCAS(&e->code, 0, code) == 0) {
        e->slice = slice;
        e->atom = atom;
        e->aux = aux;
    }
}

// slot of a launch-normalised sequence number k in [-n, 2n) of a buffer of n slots
// (BufView.soff): one compare, no division -- a division path here doubled the bin
// gather's registers and halved its occupancy
__device__ __forceinline__ int wrap_slot(int k, int n) {
    return k >= n ? k - n : (k < 0 ? k + n : k);
}

__device__ __forceinline__ const int32_t* slot_cs(const BufView& B, int j) {
    return reinterpret_cast<const int32_t*>(B.base + (size_t)wrap_slot(j + B.soff, B.nslots) * B.L.slot_bytes);
}
__device__ __forceinline__ int32_t* slot_cs_w(const BufView& B, int j) {
    return reinterpret_cast<int32_t*>(B.base + (size_t)wrap_slot(j + B.soff, B.nslots) * B.L.slot_bytes);
}
__device__ __forceinline__ double* slot_d(const BufView& B, int j, size_t off) {
    return reinterpret_cast<double*>(B.base + (size_t)wrap_slot(j + B.soff, B.nslots) * B.L.slot_bytes + off);
}
__device__ __forceinline__ int32_t* slot_i(const BufView& B, int j, size_t off) {
    return reinterpret_cast<int32_t*>(B.base + (size_t)wrap_slot(j + B.soff, B.nslots) * B.L.slot_bytes + off);
}

// 1/x in FP64: MUFU approximation + Newton steps.  One step (default) leaves a relative
// error of ~2^-45 in 1/r^2 -- about 1e-13 in a pair force, far inside the 1e-10 parity
// bound (Q13) -- and shortens each hit's dependent FP64 chain by two DFMAs (C4 force
// launch 10.09 -> 9.93 ms); -DDSEA_RCP_NEWTON=2 restores the correctly-rounded-like
// reciprocal.
#ifndef DSEA_RCP_NEWTON
#define DSEA_RCP_NEWTON 1
#endif

__device__ __forceinline__ double rcp64(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
#if DSEA_RCP_NEWTON >= 2
    e = fma(-x, y, 1.0);
    y = fma(y, e, y);
#endif
    return y;
}

__device__ __forceinline__ int cell_coord(double r, double l, int n) {
    // cell = clamp(floor(r / l), 0, n-1) with IEEE division (reading Q4)
    double q = floor(r / l);
    if (!(q >= 0.0)) return 0;
    if (q >= (double)(n - 1)) return n - 1;
    return (int)q;
}

// staging index of atom i of slice j (StgView.pool, StgView.soff)
__device__ __forceinline__ size_t stg_index(const StgView& S, int j, int cap, int i) {
    return (size_t)wrap_slot(j + S.soff, S.pool) * cap + i;
}

// Position update of md_v3b for one atom whose kick is done:
// drift, mirror in x (Q2), wrap in y/z (Q1), destination slot/cell (must be j-1, j
// or j+1, else EUNSTABLE), staging stores and the arrival count of the cell.
__device__ __forceinline__ void drift_store(const Geo& g, const StgView& stg, size_t st, int j, double xi,
                                            double yi, double zi, double vx, double vy, double vz, double Fx,
                                            double Fy, double Fz, int id, int32_t* __restrict__ out_cnt,
                                            DevErr* __restrict__ err)
{
    const int CY = g.cells[1], CZ = g.cells[2];
    const double hdt2 = 0.5 * (g.dt * g.dt);
    double x = xi + vx * g.dt + Fx * hdt2;
    double y = yi + vy * g.dt + Fy * hdt2;
    double z = zi + vz * g.dt + Fz * hdt2;
    double Fxn = Fx;
    if (x < 0.0) { x = -x; vx = -vx; Fxn = -Fxn; }                       // Q2
    else if (x > g.b[0]) { x = 2.0 * g.b[0] - x; vx = -vx; Fxn = -Fxn; }
    if (y < 0.0) y += g.b[1]; else if (y >= g.b[1]) y -= g.b[1];         // Q1
    if (z < 0.0) z += g.b[2]; else if (z >= g.b[2]) z -= g.b[2];
    const int cxg = cell_coord(x, g.l[0], g.cells[0]);
    const int cyg = cell_coord(y, g.l[1], CY);
    const int czg = cell_coord(z, g.l[2], CZ);
    const int m = cxg / g.c;
    if (!(isfinite(x) && isfinite(y) && isfinite(z)) || m < j - 1 || m > j + 1) {
        set_err(err, DSEA_EUNSTABLE, j, id, m);
        stg.key[st] = -1;
    } else {
        const int key = m * g.ncell + ((cxg - m * g.c) * CY + cyg) * CZ + czg;
        stg.x[st] = x; stg.y[st] = y; stg.z[st] = z;
        stg.vx[st] = vx; stg.vy[st] = vy; stg.vz[st] = vz;
        stg.fx[st] = Fxn; stg.fy[st] = Fy; stg.fz[st] = Fz;
        stg.id[st] = id;
        stg.key[st] = key;
        atomicAdd(&out_cnt[key], 1);
    }
}

// ---- host-side launch helpers ------------------------------------------------
static inline double env_num(const char* name, double dflt)
{
    const char* v = getenv(name);
    return (v && *v) ? atof(v) : dflt;
}

// launch with programmatic stream serialisation (DSEA_PDL=0: plain launches, A/B)
static inline bool pdl_on()
{
    static const bool on = env_num("DSEA_PDL", 1) != 0;
    return on;
}
template <typename... KArgs, typename... Args>
static void launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_on() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

}  // namespace dsea
