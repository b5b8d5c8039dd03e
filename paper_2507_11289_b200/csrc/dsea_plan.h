// dsea_plan.h -- the stage plan shared by the MD engine (dsea_host.cpp) and the
// stencil engine (dsea_grid.cpp): Table 1 (§3.3) generalised to W workers
// per GPU, N_GPU GPUs in a ring and B slices per stage.  Workload-independent: a
// worker's FORCE op processes a block of slices reading their left/right neighbours
// (O_in = 1), BIN finalises slices whose contributions are complete, RECV/SEND move
// slices between ring neighbours.  Internal header (not part of the C ABI).
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace dsea {

enum OpKind { OP_RECV = 0, OP_FORCE, OP_PASS, OP_BIN, OP_SEND };

struct Op {
    int kind;
    int stage;
    int worker;
    int slice;      // first slice
    int count;      // number of consecutive slices
    int cycle;
    int64_t t_rel;  // timestep relative to the start of the call (FORCE only)
};

struct Plan {
    std::vector<Op> ops;
    int n_stages = 0;
};

struct Blocks {
    std::vector<int> first;   // nblk + 1 entries, first[nblk] = ns
    std::vector<int> of;      // block of each slice
    int d = 1;                // worker w+1 trails worker w by d stages
    int n() const { return (int)first.size() - 1; }
    int count(int c) const { return first[c + 1] - first[c]; }
};


Blocks make_blocks(int ns, int ng, int B);
bool plan_plateau(int ng, int W, const Blocks& bl);
int plan_gap(int ng, int W, const Blocks& bl);
Plan build_plan(int ns, int ng, int rank, int W, int64_t n_steps, const Blocks& bl);

// Pushes to the ring successor (the last worker's BIN and PASS ops) must leave in
// (super-cycle, slot) order for the monotone arrival/release counters.  The plan lists
// PASS(block 0 of cycle K) before BIN(last slice of cycle K-1) in the stage where the
// last worker starts passing a trailing partial super-cycle through; that BIN only
// pushes data finalised in an earlier stage, so it is moved first.  In place.
void order_pushes(std::vector<Op>& ops, int W);

// stream memory operations (cuStreamWaitValue32 >= / cuStreamWriteValue32 through
// the runtime's driver entry points): 0 on success
int stream_wait_geq32(cudaStream_t s, const uint32_t* addr, uint32_t v);
int stream_write32(cudaStream_t s, uint32_t* addr, uint32_t v);
bool stream_memops_available();

}  // namespace dsea
