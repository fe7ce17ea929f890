// Device-resident packed problem (one graph + cluster), shared by the
// simulator and rollout kernels.  Built once by fp_problem_create from the
// arrays the reference re-packs on every exec_time call
// (flowplace/simulate.py:194-237), plus the per-strategy task orders the
// event-driven core needs.
#pragma once

#include <cstdint>
#include <string>

#include "../../include/flowplace_b200.h"
#include "fp_layout.cuh"

namespace fp {

constexpr int kMaxDevices = 32;  // device masks are uint32

struct DevProblem {
    int n, d;
    int W;           // 32-bit words per n-bit bitset
    int R;           // resources: d exec + d*d links (diagonal links unused)
    int P;           // pool entries = R * SM (slot i of resource r at r*SM + i)
    int SM;          // max concurrent slots of any resource
    int n_nonentry;
    double comm_factor;
    const int *pred_ptr, *pred_idx, *succ_ptr, *succ_idx;
    const uint8_t *is_entry;
    const double *flops, *obytes, *rates, *bw;
    const double *tlev, *blev;
    const double *edur;    // [n][d]    flops[v] / rates[a]              (simulate.py duration)
    const double *tdur;    // [n][d][d] obytes[v] * cf / bw[a][b], 0 on the diagonal
    const int *slots;      // [R]
    const int *rank_pos;   // [3][n]  position of v in strategy order
    const int *rank_vert;  // [3][n]  vertex at position
    const int *krank;      // [3][n]  dense rank of the strategy key (0 for fifo)
};

void set_error(const std::string &msg);
// compact-path batched simulation (no workspace): fp_capi.cu
int sim_launch_compact(const fp_problem *p, const int32_t *assign, int B, int strategy,
                       double *makespan, int32_t *status, fp_event *trace, int trace_cap,
                       int32_t *trace_len, cudaStream_t stream);
// blocks of a persistent launch: occupancy x SMs, capped at blocks_needed
int persistent_blocks(const void *kern, int threads, int64_t smem, int64_t blocks_needed);

}  // namespace fp

struct fp_problem {
    fp::DevProblem dev;
    void *arena = nullptr;   // single cudaMalloc holding every array
    int device = 0;
    int64_t sim_smem = 0;
};
