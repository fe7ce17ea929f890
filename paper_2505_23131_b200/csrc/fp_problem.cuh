// Device-resident packed problem (one graph + cluster), shared by the
// simulator and rollout kernels.  Built once by fp_problem_create from the
// arrays the reference re-packs on every exec_time call
// (flowplace/simulate.py:194-237), plus the per-strategy task orders the
// event-driven core needs.
#pragma once

#include <cstdint>
#include <string>

#include "../../include/flowplace_b200.h"

namespace fp {

constexpr int kMaxDevices = 32;  // device masks are uint32

struct DevProblem {
    int n, d;
    int W;           // 32-bit words per n-bit bitset
    int R;           // resources: d exec + d*d links (diagonal links unused)
    int P;           // pool entries = sum of slots over used resources
    int n_nonentry;
    double comm_factor;
    const int *pred_ptr, *pred_idx, *succ_ptr, *succ_idx;
    const uint8_t *is_entry;
    const double *flops, *obytes, *rates, *bw;
    const double *tlev, *blev;
    const int *slots;      // [R]
    const int *pool_off;   // [R+1]
    const int *rank_pos;   // [3][n]  position of v in strategy order
    const int *rank_vert;  // [3][n]  vertex at position
    const int *krank;      // [3][n]  dense rank of the strategy key (0 for fifo)
};

// Shared-memory bytes for one episode's simulator state (see sim_carve).
__host__ __device__ inline int64_t sim_smem_bytes(int n, int d, int W, int R, int P) {
    (void)d;
    int64_t b = 0;
    b += 4LL * n * 3;             // rdy, missing, cons
    b += (n + 15) / 16 * 16;      // assign (uint8)
    b += 4LL * R * W;             // pending bitsets
    b += 4LL * R * 2;             // cnt, freec
    b = (b + 7) / 8 * 8;
    b += 8LL * P;                 // pool end times
    b += 8LL * P;                 // start-sort keys
    b += 4LL * P * 4;             // pool v, pool seq, sort idx, end list
    b += 16;                      // counters
    return (b + 15) / 16 * 16;
}

void set_error(const std::string &msg);

}  // namespace fp

struct fp_problem {
    fp::DevProblem dev;
    void *arena = nullptr;   // single cudaMalloc holding every array
    int device = 0;
    int64_t sim_smem = 0;
};
