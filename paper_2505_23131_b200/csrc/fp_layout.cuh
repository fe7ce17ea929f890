// Per-episode state layout (byte offsets, computed identically on host and
// device).  Fields fall in two groups:
//   * n-sized arrays (timeline, candidate set, simulator ready/missing/pending
//     state) -- addressed from `nb`;
//   * small fixed-size scratch (device features, in-flight pool, hand-off
//     ring, counters) -- addressed from `sb`.
// Compact path (n <= ~1k): both groups live in the episode's shared-memory
// slice (nb == sb), every access an LDS/STS.  Wide path (large graphs): the
// n-sized group lives in a caller-provided HBM workspace slice per resident
// episode (L2-cached), the small group stays in shared memory.
#pragma once

#include <cstdint>

namespace fp {

constexpr int kRing = 128;        // SEL -> PLC vertex hand-off ring (wide path)
constexpr int kMaxTreeLevels = 6; // 32-ary candidate tree: n <= 32^6

struct EpLayout {
    // ---- n-sized group (nb) ----
    int ce, cc, dsl, dse, tstart, tend, cand, npl, clist, order;
    int rdy, missing, cons, assign, bits;
    int tm, tz, tc, tt;  // candidate tree nodes (wide rollout): max, scaled sum, count, teacher max
    // ---- small group (sb) ----
    int xd, xn, stats, rsum, flag, ring, simres;
    int cnt, pend, pv, pseq, skey, sidx, elist, ctr;
    int bytes;   // shared-memory bytes per episode
    int64_t gbytes;  // HBM workspace bytes per episode (wide), 0 for the compact path
    int wide;
    // hierarchical pending bitsets: words per resource = W + W1 + W2
    int W, W1, W2, BW;
    // candidate tree: levels 1..tl_n, level l has tl_cnt[l] nodes at tl_off[l]
    int tl_n;
    int tl_off[kMaxTreeLevels + 1];
    int tl_cnt[kMaxTreeLevels + 1];
};

__host__ __device__ inline int fp_align(int x, int a) { return (x + a - 1) / a * a; }
__host__ __device__ inline int64_t fp_align64(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// n vertices, W words per bitset, R resources, SM slots per resource.
// with_rollout = false gives the simulator-only layout.
// rsum_doubles: per-device running REINFORCE sums kept in smem (2*d*h, grad mode).
// wide: n-sized arrays in the HBM workspace, hierarchical bitsets, candidate tree.
__host__ __device__ inline EpLayout make_layout(int n, int W, int R, int SM, bool with_rollout,
                                               int rsum_doubles = 0, bool wide = false) {
    EpLayout L;
    L.wide = wide ? 1 : 0;
    L.W = W;
    L.W1 = wide ? (W + 31) / 32 : 0;
    L.W2 = wide ? (L.W1 + 31) / 32 : 0;
    L.BW = W + L.W1 + L.W2;
    // tree geometry (wide rollout only)
    L.tl_n = 0;
    int tree_nodes = 0;
    for (int l = 0; l <= kMaxTreeLevels; ++l) { L.tl_off[l] = 0; L.tl_cnt[l] = 0; }
    if (wide && with_rollout) {
        int c = n;
        while (L.tl_n < kMaxTreeLevels) {
            c = (c + 31) / 32;
            ++L.tl_n;
            L.tl_off[L.tl_n] = tree_nodes;
            L.tl_cnt[L.tl_n] = c;
            tree_nodes += c;
            if (c <= 1) break;
        }
    }
    int64_t og = 0;  // n-group cursor
    int os = 0;      // small-group cursor
    auto take_n = [&](int64_t bytes, int align) -> int {
        if (wide) {
            og = fp_align64(og, align);
            const int64_t at = og;
            og += bytes;
            return (int)at;
        }
        os = fp_align(os, align);
        const int at = os;
        os += (int)bytes;
        return at;
    };
    auto take_s = [&](int bytes, int align) {
        os = fp_align(os, align);
        const int at = os;
        os += bytes;
        return at;
    };
    const int P = R * SM;
    L.ce = L.cc = L.dsl = L.dse = L.tstart = L.tend = L.cand = L.npl = L.clist = L.order = 0;
    L.tm = L.tz = L.tc = L.tt = 0;
    L.xd = L.xn = L.stats = L.rsum = L.flag = L.ring = L.simres = 0;
    if (with_rollout) {
        if (!wide) {
            L.ce = take_n(8 * n, 16);
            L.cc = take_n(8 * n, 8);
            L.dsl = take_n(8 * n, 8);
            L.dse = take_n(8 * n, 8);
            L.clist = take_n(4 * n, 4);
            L.order = take_n(4 * n, 4);
        } else {
            L.tm = take_n(8LL * tree_nodes, 16);
            L.tz = take_n(8LL * tree_nodes, 8);
            L.tt = take_n(8LL * tree_nodes, 8);
            L.tc = take_n(4LL * tree_nodes, 4);
            L.ring = take_s(4 * kRing, 16);
        }
        L.tstart = take_n(8LL * n, 8);
        L.tend = take_n(8LL * n, 8);
        L.cand = take_n(4LL * W, 4);
        L.npl = take_n(4LL * n, 4);
        L.xd = take_s(8 * 32 * 5, 8);
        L.xn = take_s(8 * 32 * 5, 8);
        L.stats = take_s(8 * 16, 8);
        L.rsum = take_s(8 * rsum_doubles, 8);
        L.flag = take_s(16, 16);
        L.simres = take_s(16, 16);
    }
    L.pend = take_s(8 * P, 8);
    L.skey = take_s(8 * P, 8);
    L.rdy = take_n(4LL * n, 4);
    L.missing = take_n(4LL * n, 4);
    L.cons = take_n(4LL * n, 4);
    L.bits = take_n(4LL * R * L.BW, 4);
    L.cnt = take_s(4 * R, 4);
    L.pv = take_s(4 * P, 4);
    L.pseq = take_s(4 * P, 4);
    L.sidx = take_s(4 * P, 4);
    L.elist = take_s(4 * P, 4);
    L.ctr = take_s(16, 4);
    L.assign = take_n(n, 1);
    L.bytes = fp_align(os, 16);
    L.gbytes = wide ? fp_align64(og, 256) : 0;
    return L;
}

}  // namespace fp
