// Shared-memory layout of one episode (byte offsets, computed identically on
// host and device).  Offsets index from the episode's slice of the dynamic
// shared buffer with plain pointer arithmetic, so every access compiles to
// LDS/STS (no generic-address round trips).
#pragma once

#include <cstdint>

namespace fp {

struct EpLayout {
    // SEL warp
    int cand, npl, clist, ce, cc, dsl, dse, order, flag;
    // PLC warp
    int tstart, tend, xd, stats, xn, rsum;
    // simulator (PLC warp after the rollout; also the sim-only kernel)
    int rdy, missing, cons, assign, bits, cnt, pend, pv, pseq, skey, sidx, elist, ctr;
    int bytes;
};

__host__ __device__ inline int fp_align(int x, int a) { return (x + a - 1) / a * a; }

// n vertices, W words per bitset, R resources, SM slots per resource.
// with_rollout = false gives the simulator-only layout.
// rsum_doubles: per-device running REINFORCE sums kept in smem (2*d*h, grad mode)
__host__ __device__ inline EpLayout make_layout(int n, int W, int R, int SM, bool with_rollout,
                                               int rsum_doubles = 0) {
    EpLayout L;
    int o = 0;
    auto take = [&](int bytes, int align) {
        o = fp_align(o, align);
        const int at = o;
        o += bytes;
        return at;
    };
    const int P = R * SM;
    if (with_rollout) {
        L.ce = take(8 * n, 16);
        L.cc = take(8 * n, 8);
        L.dsl = take(8 * n, 8);
        L.dse = take(8 * n, 8);
        L.tstart = take(8 * n, 8);
        L.tend = take(8 * n, 8);
        L.xd = take(8 * 32 * 5, 8);
        L.xn = take(8 * 32 * 5, 8);
        L.stats = take(8 * 16, 8);
        L.rsum = take(8 * rsum_doubles, 8);
        L.cand = take(4 * W, 4);
        L.npl = take(4 * n, 4);
        L.clist = take(4 * n, 4);
        L.order = take(4 * n, 4);
        L.flag = take(16, 16);
    } else {
        L.ce = L.cc = L.dsl = L.dse = L.tstart = L.tend = L.xd = L.xn = L.stats = L.rsum = 0;
        L.cand = L.npl = L.clist = L.order = L.flag = 0;
    }
    L.pend = take(8 * P, 8);
    L.skey = take(8 * P, 8);
    L.rdy = take(4 * n, 4);
    L.missing = take(4 * n, 4);
    L.cons = take(4 * n, 4);
    L.bits = take(4 * R * W, 4);
    L.cnt = take(4 * R, 4);
    L.pv = take(4 * P, 4);
    L.pseq = take(4 * P, 4);
    L.sidx = take(4 * P, 4);
    L.elist = take(4 * P, 4);
    L.ctr = take(16, 4);
    L.assign = take(n, 1);
    L.bytes = fp_align(o, 16);
    return L;
}

}  // namespace fp
