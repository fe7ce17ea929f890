// Batched SEL/PLC episodes fused with the WC simulator, episode state resident
// in shared memory, TWO warps per episode:
//
//   SEL warp (producer)  In per_episode mode the SEL logits are static per
//        snapshot and the candidate set depends only on the
//        vertices chosen so far — never on PLC decisions — so the whole vertex
//        order is one independent chain: candidate bitset -> ascending list ->
//        masked softmax over s[v] -> decision (Philox epsilon-mixture sample /
//        greedy / forced / critical-path teacher) -> mixture log-prob and
//        entropy (policy.py:186-204, 301-322) -> candidate update
//        (policy.py:384-389).  It publishes order[t] through shared memory.
//   PLC warp (consumer)  For v = order[t]: device features (lane = device,
//        policy.py:226-247 over timeline.py:30-45), column standardization with
//        the reference's sequential fp64 sums (policy.py:101-105; lane =
//        column), pre-activations A[v] + S_d + xn_d @ M + c (lane = hidden
//        column, fact 3), leaky, head2 via a transpose reduction, softmax over
//        devices, decision, log-prob / entropy, timeline commit
//        (timeline.py:47-58, bit-exact _rn fp64), S_d += G[v].
//   The two chains overlap; the episode's latency is the longer (PLC) chain.
//   After the last step the PLC warp runs sim_episode() on the assignment in
//   shared memory (fp_sim.cuh) — no round trip through HBM.
//
// Optional REINFORCE rows: d log-prob / d entropy w.r.t. the SEL logits
// (per-vertex smem accumulators, SEL warp) and the PLC pre-activations (per
// vertex A rows, running per-device sums R_d for the G rows, M / w2 / b2
// terms; PLC warp), consumed by the episode-reduction kernel (fp_train.cu).
#pragma once

#include <string>

#include "fp_common.cuh"
#include "fp_layout.cuh"
#include "fp_policy.cuh"
#include "fp_sim.cuh"

namespace fp {

__device__ __forceinline__ double lk(double x, double s) { return x > 0.0 ? x : s * x; }
__device__ __forceinline__ double lkd(double x, double s) { return x > 0.0 ? 1.0 : s; }

__device__ __forceinline__ void warp_argmax_first(double &v, int &i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(FP_FULL_MASK, v, o);
        const int oi = __shfl_xor_sync(FP_FULL_MASK, i, o);
        if (ov > v || (ov == v && oi < i)) { v = ov; i = oi; }
    }
}

__host__ __device__ inline int64_t grad_ep_stride(int n, int h, int d) {
    return ((2LL * n + 12LL * h + 2 + 2LL * d * h) + 3) / 4 * 4;
}

// REINFORCE decision records (compact GRAD rollouts), in the caller's
// grad_rows buffer, grad_rec_stride(d, W) doubles per (episode, step): the
// PLC warp's normalised device features xn[5d], logits[d] and (vertex,
// device) int2; the SEL warp's softmax max and normaliser over the
// candidates, the chosen vertex and the candidate bitset (W words).  The PLC warp also writes
// grad_ep[2n] = chain completed, [2n + 1] = epsilon.  fp_pg_reduce replays
// the records (plc_replay_kernel) -- the log-prob / entropy adjoints never
// run on the rollout's decision chains.
__host__ __device__ inline int grad_rec_stride(int d, int W) { return 6 * d + 4 + (W + 1) / 2; }

template <int MAXD>
struct PlcLog {  // log2(MAXD)
    static constexpr int v = MAXD <= 1 ? 0 : MAXD <= 2 ? 1 : MAXD <= 4 ? 2 : MAXD <= 8 ? 3 :
                             MAXD <= 16 ? 4 : 5;
};

// ---------------------------------------------------------------------------
// SEL warp
// ---------------------------------------------------------------------------
template <bool GRAD, bool LEAN = false>
__device__ __forceinline__ bool sel_chain(const DevProblem &PR, const DevPolicy &PO,
                                          const fp_rollout_args &A, uint8_t *base /* nb == sb */,
                                          const EpLayout &L, const double *s_sm, int ep,
                                          bool want_lp, bool want_amax) {
    const int lane = lane_id();
    const int n = PR.n, W = PR.W;
    uint32_t *cand = (uint32_t *)(base + L.cand);
    int *npl = (int *)(base + L.npl);
    int *clist = (int *)(base + L.clist);
    double *ce = (double *)(base + L.ce);
    double *cc = (double *)(base + L.cc);
    volatile int *order = (volatile int *)(base + L.order);
    const double eps = A.epsilon, ome = 1.0 - eps;
    const uint32_t k0 = (uint32_t)A.seed, k1 = (uint32_t)(A.seed >> 32);
    const uint32_t ctr_ep = A.episode_base + (uint32_t)ep;
    const int mode = LEAN ? FP_MODE_SAMPLE : A.mode;  // LEAN: sampling-only build
    const int32_t *frow = mode == FP_MODE_FORCED ? A.forced + (size_t)ep * n * 2 : nullptr;
    const int *__restrict__ pp = PR.pred_ptr;
    const int *__restrict__ sp = PR.succ_ptr;
    const int *__restrict__ si = PR.succ_idx;

#pragma unroll 1
    for (int w = lane; w < W; w += 32) cand[w] = 0u;
    __syncwarp();
#pragma unroll 1
    for (int v = lane; v < n; v += 32) {
        const int np = pp[v + 1] - pp[v];
        npl[v] = np;
        if (np == 0) atomicOr(&cand[v >> 5], 1u << (v & 31));
    }
    __syncwarp();

    FP_PHASE_DECL;
    FP_PHASE_BEGIN(ps);
    double dc1 = 0.0, dc2 = 0.0;  // draw cache (step_draw)
    const bool tie_rand = mode == FP_MODE_TEACHER && (A.flags & FP_FLAG_TIE_RANDOM);
    for (int step = 0; step < n; ++step) {
        double u1 = 0.0, u2 = 0.0;
        if (mode == FP_MODE_SAMPLE || tie_rand)
            step_draw(step, ctr_ep, 0u, k0, k1, dc1, dc2, u1, u2);
        // compact the candidate bitset into an ascending list
        const uint32_t cw = lane < W ? cand[lane] : 0u;
        const int pc = __popc(cw);
        const int incl = warp_inclusive_scan(pc);
        const int k = __shfl_sync(FP_FULL_MASK, incl, 31);
        if (k == 0) {  // cyclic graph: nothing is ever ready
            if (lane == 0) order[step] = -1;
            return false;
        }
        {
            int o = incl - pc;
            uint32_t m = cw;
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                clist[o++] = lane * 32 + b;
            }
        }
        __syncwarp();
        FP_PHASE_END(ps, 0);
        const bool fast = k <= 32;  // candidate i on lane i, values in registers
        int idx = -1;
        double e0 = 0.0, cum0 = 0.0, tot, mxr;
        int myv = -1;
        if (fast) {
            myv = lane < k ? clist[lane] : -1;
            const double sv = lane < k ? s_sm[myv] : -INFINITY;
            const double mx = warp_max_redux(sv);
            mxr = mx;
            e0 = lane < k ? exp(sv - mx) : 0.0;
            cum0 = warp_inclusive_scan(e0);
            tot = __shfl_sync(FP_FULL_MASK, cum0, 31);
            if (mode == FP_MODE_FORCED) {
                const unsigned hit = __ballot_sync(FP_FULL_MASK, lane < k && myv == frow[2 * step]);
                idx = hit ? __ffs(hit) - 1 : -1;
            } else if (mode == FP_MODE_TEACHER) {
                const double tv = lane < k ? PR.tlev[myv] : -INFINITY;
                const double bt = warp_max_redux(tv);
                unsigned top = __ballot_sync(FP_FULL_MASK, lane < k && tv == bt);
                if (tie_rand) {  // the r-th of the tied candidates, ascending id
                    const int cnt = __popc(top);
                    for (int r = min((int)(u1 * (double)cnt), cnt - 1); r > 0; --r) top &= top - 1;
                }
                idx = __ffs(top) - 1;
            } else if (mode == FP_MODE_SAMPLE) {
                if (u1 < eps) {
                    idx = min((int)(u2 * (double)k), k - 1);
                } else {
                    const unsigned hit = __ballot_sync(FP_FULL_MASK, lane < k && cum0 > u2 * tot);
                    idx = hit ? __ffs(hit) - 1 : k - 1;
                }
            }
        } else {
            double mx = -INFINITY;
#pragma unroll 1
            for (int i = lane; i < k; i += 32) mx = fmax(mx, s_sm[clist[i]]);
            mx = warp_max_redux(mx);
            double carry = 0.0;
#pragma unroll 1
            for (int b0 = 0; b0 < k; b0 += 32) {
                const int i = b0 + lane;
                const double e = i < k ? exp(s_sm[clist[i]] - mx) : 0.0;
                const double cum = warp_inclusive_scan(e) + carry;
                if (i < k) { ce[i] = e; cc[i] = cum; }
                carry = __shfl_sync(FP_FULL_MASK, cum, 31);
            }
            tot = carry;
            mxr = mx;
            __syncwarp();
            if (mode == FP_MODE_FORCED) {
                const int fv = frow[2 * step];
                for (int b0 = 0; b0 < k && idx < 0; b0 += 32) {
                    const unsigned hit =
                        __ballot_sync(FP_FULL_MASK, b0 + lane < k && clist[b0 + lane] == fv);
                    if (hit) idx = b0 + __ffs(hit) - 1;
                }
            } else if (mode == FP_MODE_TEACHER) {
                double bt = -INFINITY;
                for (int i = lane; i < k; i += 32) bt = fmax(bt, PR.tlev[clist[i]]);
                bt = warp_max_redux(bt);
                int r = 0;
                if (tie_rand) {
                    int cnt = 0;
                    for (int b0 = 0; b0 < k; b0 += 32)
                        cnt += __popc(__ballot_sync(
                            FP_FULL_MASK, b0 + lane < k && PR.tlev[clist[b0 + lane]] == bt));
                    r = min((int)(u1 * (double)cnt), cnt - 1);
                }
                for (int b0 = 0; b0 < k && idx < 0; b0 += 32) {
                    unsigned hit = __ballot_sync(
                        FP_FULL_MASK, b0 + lane < k && PR.tlev[clist[b0 + lane]] == bt);
                    const int c = __popc(hit);
                    if (r >= c) { r -= c; continue; }
                    for (; r > 0; --r) hit &= hit - 1;
                    idx = b0 + __ffs(hit) - 1;
                }
            } else if (mode == FP_MODE_SAMPLE) {
                if (u1 < eps) {
                    idx = min((int)(u2 * (double)k), k - 1);
                } else {
                    const double target = u2 * tot;
                    for (int b0 = 0; b0 < k && idx < 0; b0 += 32) {
                        const unsigned hit =
                            __ballot_sync(FP_FULL_MASK, b0 + lane < k && cc[b0 + lane] > target);
                        if (hit) idx = b0 + __ffs(hit) - 1;
                    }
                    if (idx < 0) idx = k - 1;
                }
            }
        }
        FP_PHASE_END(ps, 1);
        int amax = -1;
        if (want_amax || mode == FP_MODE_GREEDY) {
            // first maximum of p = e / tot (policy.py:309, 396)
            double bp = -1.0;
            int bi = 0x7fffffff;
            for (int i = lane; i < k; i += 32) {
                const double p = (fast ? e0 : ce[i]) / tot;
                if (p > bp) { bp = p; bi = i; }
            }
            warp_argmax_first(bp, bi);
            amax = bi;
            if (mode == FP_MODE_GREEDY) idx = amax;
        }
        if (idx < 0) {  // forced vertex is not a candidate
            if (lane == 0) order[step] = -2;
            return false;
        }
        const int v = clist[idx];
        // publish early: the PLC warp only needs the vertex (a single 32-bit
        // store replacing the -3 sentinel is the whole hand-off)
        if (lane == 0) order[step] = v;
        if constexpr (GRAD) {  // SEL part of the decision record (replayed by fp_pg_reduce)
            double *rec = A.grad_rows + ((size_t)ep * n + step) * grad_rec_stride(PR.d, W) +
                          6 * PR.d + 1;
            if (lane == 0) { rec[0] = mxr; rec[1] = tot; rec[2] = (double)v; }
            if (lane < W) ((uint32_t *)(rec + 3))[lane] = cw;
        }
        FP_PHASE_END(ps, 2);
        if (want_lp && fast) {
            // candidate i on lane i: p, mix, log(mix) once per lane; the
            // chosen candidate's terms by shuffle (the sums below are the
            // slow path's, same reduction tree)
            const double ek = eps / (double)k;
            double p = 0.0, mix = 0.0, lm = 0.0;
            if (lane < k) {
                p = e0 / tot;
                mix = __dadd_rn(__dmul_rn(p, ome), ek);
                lm = log(__dadd_rn(mix, 1e-30));
            }
            const double ent = -warp_sum(lane < k ? mix * lm : 0.0);
            const double lp = __shfl_sync(FP_FULL_MASK, lm, idx);
            if (lane == 0) {
                const size_t o = (size_t)ep * n + step;
                if (A.step_lp) A.step_lp[2 * o] = lp;
                if (A.step_ent) A.step_ent[2 * o] = ent;
            }
        } else if (want_lp) {
            const double ek = eps / (double)k;
            double entp = 0.0, lp = 0.0;
            for (int i = lane; i < k; i += 32) {
                const double p = (fast ? e0 : ce[i]) / tot;
                const double mix = __dadd_rn(__dmul_rn(p, ome), ek);
                const double lm = log(__dadd_rn(mix, 1e-30));
                entp += mix * lm;
                if (i == idx) lp = lm;
            }
            const double ent = -warp_sum(entp);
            lp = warp_sum(lp);  // exactly one lane non-zero
            if (lane == 0) {
                const size_t o = (size_t)ep * n + step;
                if (A.step_lp) A.step_lp[2 * o] = lp;
                if (A.step_ent) A.step_ent[2 * o] = ent;
            }
        }
        FP_PHASE_END(ps, 3);
        if (lane == 0) {
            const size_t o = (size_t)ep * n + step;
            if (A.step_vd) A.step_vd[2 * o] = v;
            if (A.step_argmax) A.step_argmax[2 * o] = clist[amax];
            if (A.step_ncand) A.step_ncand[o] = k;
            cand[v >> 5] &= ~(1u << (v & 31));
        }
        __syncwarp();
#pragma unroll 1
        for (int j = sp[v] + lane; j < sp[v + 1]; j += 32) {
            const int w = si[j];
            if (atomicSub(&npl[w], 1) == 1) atomicOr(&cand[w >> 5], 1u << (w & 31));
        }
        __syncwarp();
        FP_PHASE_END(ps, 4);
    }
    FP_PHASE_FLUSH(0);
    return true;
}

// ---------------------------------------------------------------------------
// SEL warp, wide path (graphs whose state lives in HBM)
//
// The compact chain re-compacts the candidate bitset every step (O(n/32)
// words) -- quadratic at 10k-100k ops.  Here the candidate set is a 32-ary
// tree over vertex ids whose node j at level l summarises leaves
// [j*32^l, (j+1)*32^l): m = max SEL logit of its candidates, z = sum of
// exp(s - m) over them (each node keeps its own max: SEL logits grow with
// the b/t path sums and span thousands of nats on 100k-op graphs, so no
// global shift keeps every sum in range), c = candidate count, t = max
// t-level (critical-path teacher).  A warp refreshes a node with one
// coalesced 32-child load, a REDUX max, one exp per lane and a butterfly sum;
// the ancestors touched by one step (the placed vertex and its newly ready
// successors) are refreshed once each, level by level.  Sampling descends
// by cumulative weight in ascending-id order -- the reference's
// searchsorted(cumsum(p), u * sum(p), 'right') (policy.py:313-316) -- and
// the uniform branch by count to the idx-th candidate in ascending order;
// the entropy (only when requested) is one pass over the candidates.
// ---------------------------------------------------------------------------
struct TreeRef {
    double *tm, *tz, *tt;
    int *tc;
    const uint32_t *cand;
    const double *s, *tlev;
    const EpLayout *L;
    int n;
    bool teacher;

    // child `i` of node j at level l (l == 1: leaf = vertex)
    __device__ __forceinline__ void child(int l, int j, double &m, double &z, double &t,
                                          int &c) const {
        const int ci = (j << 5) + lane_id();
        if (l == 1) {
            const bool ok = ci < n && ((cand[j] >> (ci & 31)) & 1u);
            m = ok ? s[ci] : -INFINITY;
            z = ok ? 1.0 : 0.0;
            c = ok ? 1 : 0;
            t = ok && teacher ? tlev[ci] : -INFINITY;
        } else {
            const bool ok = ci < L->tl_cnt[l - 1];
            const int idx = L->tl_off[l - 1] + ci;
            m = ok ? tm[idx] : -INFINITY;
            z = ok ? tz[idx] : 0.0;
            c = ok ? tc[idx] : 0;
            t = ok && teacher ? tt[idx] : -INFINITY;
        }
    }

    __device__ __forceinline__ void recompute(int l, int j) const {
        double m, z, t;
        int c;
        child(l, j, m, z, t, c);
        const double M = warp_max_redux(m);
        const double Z = warp_sum(c > 0 ? z * exp(m - M) : 0.0);
        const int C = __reduce_add_sync(FP_FULL_MASK, c);
        const double T = teacher ? warp_max_redux(t) : -INFINITY;
        if (lane_id() == 0) {
            const int idx = L->tl_off[l] + j;
            tm[idx] = M; tz[idx] = Z; tc[idx] = C;
            if (teacher) tt[idx] = T;
        }
        __syncwarp();
    }

    // leaves held by the lanes (-1: none) changed: refresh every distinct
    // ancestor once, bottom-up
    __device__ __forceinline__ void update_many(int leaf) const {
        for (int l = 1; l <= L->tl_n; ++l) {
            const int id = leaf >= 0 ? leaf >> (5 * l) : -1;
            const unsigned peers = __match_any_sync(FP_FULL_MASK, id);
            unsigned todo = __ballot_sync(FP_FULL_MASK, id >= 0 && lane_id() == __ffs(peers) - 1);
            while (todo) {
                const int src = __ffs(todo) - 1;
                todo &= todo - 1;
                recompute(l, __shfl_sync(FP_FULL_MASK, id, src));
            }
        }
    }

    __device__ __forceinline__ int root() const { return L->tl_off[L->tl_n]; }

    __device__ __forceinline__ void rebuild() const {
        for (int l = 1; l <= L->tl_n; ++l)
            for (int j = 0; j < L->tl_cnt[l]; ++j) recompute(l, j);
    }

    // first leaf whose inclusive cumulative weight exceeds target (root units)
    __device__ __forceinline__ int descend_weight(double target) const {
        int j = 0;
        double Mn = tm[root()];
        for (int l = L->tl_n; l >= 1; --l) {
            double m, z, t;
            int c;
            child(l, j, m, z, t, c);
            const double w = c > 0 ? z * exp(m - Mn) : 0.0;
            const double cum = warp_inclusive_scan(w);
            const unsigned nonempty = __ballot_sync(FP_FULL_MASK, c > 0);
            const unsigned hit = __ballot_sync(FP_FULL_MASK, c > 0 && cum > target);
            const int sel = hit ? __ffs(hit) - 1 : 31 - __clz(nonempty);
            const double prev = __shfl_sync(FP_FULL_MASK, cum - w, sel);
            const double ms = __shfl_sync(FP_FULL_MASK, m, sel);
            target = (target - prev) * exp(Mn - ms);  // into the child's units
            Mn = ms;
            j = (j << 5) + sel;
        }
        return j;
    }

    // the idx-th candidate (0-based) in ascending id order
    __device__ __forceinline__ int descend_count(int idx) const {
        int j = 0;
        for (int l = L->tl_n; l >= 1; --l) {
            double m, z, t;
            int c;
            child(l, j, m, z, t, c);
            const int cum = warp_inclusive_scan(c);
            const unsigned hit = __ballot_sync(FP_FULL_MASK, cum > idx);
            const int sel = __ffs(hit) - 1;
            idx -= __shfl_sync(FP_FULL_MASK, cum - c, sel);
            j = (j << 5) + sel;
        }
        return j;
    }

    // first candidate attaining the maximum logit (key 0) or t-level (key 1)
    __device__ __forceinline__ int descend_max(bool by_tlev) const {
        int j = 0;
        const double best = by_tlev ? tt[root()] : tm[root()];
        for (int l = L->tl_n; l >= 1; --l) {
            double m, z, t;
            int c;
            child(l, j, m, z, t, c);
            const double key = by_tlev ? t : m;
            const int sel = __ffs(__ballot_sync(FP_FULL_MASK, c > 0 && key == best)) - 1;
            j = (j << 5) + sel;
        }
        return j;
    }
};

__device__ __forceinline__ bool ring_publish(volatile int *ring, volatile int *dead, int step,
                                             int v) {
    int ok = 1;
    if (lane_id() == 0) {
        const int slot = step & (kRing - 1);
        while (ring[slot] != -3) {
            if (*dead) { ok = 0; break; }
        }
        if (ok) ring[slot] = v;
    }
    return __shfl_sync(FP_FULL_MASK, ok, 0) != 0;
}

template <bool LEAN = false>
__device__ __forceinline__ void sel_chain_wide(const DevProblem &PR, const DevPolicy &PO,
                                               const fp_rollout_args &A, uint8_t *nb,
                                               uint8_t *sb, const EpLayout &L, int ep,
                                               bool want_lp, bool want_amax) {
    const int lane = lane_id();
    const int n = PR.n, W = PR.W;
    uint32_t *cand = (uint32_t *)(nb + L.cand);
    int *npl = (int *)(nb + L.npl);
    volatile int *ring = (volatile int *)(sb + L.ring);
    volatile int *dead = (volatile int *)(sb + L.flag);
    const double eps = A.epsilon, ome = 1.0 - eps;
    const uint32_t k0 = (uint32_t)A.seed, k1 = (uint32_t)(A.seed >> 32);
    const uint32_t ctr_ep = A.episode_base + (uint32_t)ep;
    const int mode = LEAN ? FP_MODE_SAMPLE : A.mode;
    const int32_t *frow = mode == FP_MODE_FORCED ? A.forced + (size_t)ep * n * 2 : nullptr;
    const int *__restrict__ pp = PR.pred_ptr;
    const int *__restrict__ sp = PR.succ_ptr;
    const int *__restrict__ si = PR.succ_idx;
    const double *__restrict__ s = PO.s;
    TreeRef T{(double *)(nb + L.tm), (double *)(nb + L.tz), (double *)(nb + L.tt),
              (int *)(nb + L.tc), cand, s, PR.tlev, &L, n, mode == FP_MODE_TEACHER};

    for (int w = lane; w < W; w += 32) cand[w] = 0u;
    __syncwarp();
    for (int v = lane; v < n; v += 32) {
        const int np = pp[v + 1] - pp[v];
        npl[v] = np;
        if (np == 0) atomicOr(&cand[v >> 5], 1u << (v & 31));
    }
    __syncwarp();
    T.rebuild();

    const int rt = T.root();
    FP_PHASE_DECL;
    FP_PHASE_BEGIN(pw);
    double dc1 = 0.0, dc2 = 0.0;  // draw cache (step_draw)
    const bool tie_rand = mode == FP_MODE_TEACHER && (A.flags & FP_FLAG_TIE_RANDOM);
    for (int step = 0; step < n; ++step) {
        double u1 = 0.0, u2 = 0.0;
        if (mode == FP_MODE_SAMPLE || tie_rand)
            step_draw(step, ctr_ep, 0u, k0, k1, dc1, dc2, u1, u2);
        const int k = T.tc[rt];
        if (k == 0) {  // cyclic graph: nothing is ever ready
            ring_publish(ring, dead, step, -1);
            return;
        }
        const double Mr = T.tm[rt], Zr = T.tz[rt];  // p = exp(s - Mr) / Zr
        int v = -1;
        if (mode == FP_MODE_FORCED) {
            const int fv = frow[2 * step];
            if (fv >= 0 && fv < n && ((cand[fv >> 5] >> (fv & 31)) & 1u)) v = fv;
        } else if (mode == FP_MODE_TEACHER) {
            v = T.descend_max(true);
            if (tie_rand) {  // r-th tied candidate: one pass over the candidate bitset
                const double bt = T.tt[rt];
                int cnt = 0;
                for (int w = lane; w < W; w += 32) {
                    uint32_t m = cand[w];
                    while (m) {
                        const int u = (w << 5) + __ffs(m) - 1;
                        m &= m - 1;
                        cnt += PR.tlev[u] == bt;
                    }
                }
                cnt = __reduce_add_sync(FP_FULL_MASK, cnt);
                int r = min((int)(u1 * (double)cnt), cnt - 1);
                for (int w0 = 0; w0 < W; w0 += 32) {
                    const int w = w0 + lane;
                    uint32_t tied = 0;
                    if (w < W) {
                        uint32_t m = cand[w];
                        while (m) {
                            const int b = __ffs(m) - 1;
                            m &= m - 1;
                            if (PR.tlev[(w << 5) + b] == bt) tied |= 1u << b;
                        }
                    }
                    const int c = __popc(tied);
                    const int before = warp_inclusive_scan(c) - c;
                    const int total = __shfl_sync(FP_FULL_MASK, before + c, 31);
                    if (r >= total) { r -= total; continue; }
                    const unsigned own = __ballot_sync(FP_FULL_MASK, r >= before && r < before + c);
                    const int src = __ffs(own) - 1;
                    int pick = -1;
                    if (lane == src) {
                        uint32_t m = tied;
                        for (int q = r - before; q > 0; --q) m &= m - 1;
                        pick = (w << 5) + __ffs(m) - 1;
                    }
                    v = __shfl_sync(FP_FULL_MASK, pick, src);
                    break;
                }
            }
        } else if (mode == FP_MODE_SAMPLE) {
            v = u1 < eps ? T.descend_count(min((int)(u2 * (double)k), k - 1))
                         : T.descend_weight(u2 * Zr);
        }
        int amax = -1;
        if (want_amax || mode == FP_MODE_GREEDY) {
            amax = T.descend_max(false);
            if (mode == FP_MODE_GREEDY) v = amax;
        }
        if (v < 0) {  // forced vertex is not a candidate
            ring_publish(ring, dead, step, -2);
            return;
        }
        FP_PHASE_END(pw, 5);
        if (!ring_publish(ring, dead, step, v)) return;
        if (want_lp) {
            const double ek = eps / (double)k;
            const double p = exp(s[v] - Mr) / Zr;
            const double mix = __dadd_rn(__dmul_rn(p, ome), ek);
            const double lp = log(__dadd_rn(mix, 1e-30));
            double entp = 0.0;
            for (int w = lane; w < W; w += 32) {
                uint32_t m = cand[w];
                while (m) {
                    const int u = (w << 5) + __ffs(m) - 1;
                    m &= m - 1;
                    const double pu = exp(s[u] - Mr) / Zr;
                    const double mu = __dadd_rn(__dmul_rn(pu, ome), ek);
                    entp += mu * log(__dadd_rn(mu, 1e-30));
                }
            }
            const double ent = -warp_sum(entp);
            if (lane == 0) {
                const size_t o = (size_t)ep * n + step;
                if (A.step_lp) A.step_lp[2 * o] = lp;
                if (A.step_ent) A.step_ent[2 * o] = ent;
            }
        }
        if (lane == 0) {
            const size_t o = (size_t)ep * n + step;
            if (A.step_vd) A.step_vd[2 * o] = v;
            if (A.step_argmax) A.step_argmax[2 * o] = amax;
            if (A.step_ncand) A.step_ncand[o] = k;
            atomicAnd(&cand[v >> 5], ~(1u << (v & 31)));
        }
        __syncwarp();
        FP_PHASE_END(pw, 6);
        // successors whose last predecessor was just placed become candidates;
        // the changed leaves (v on lane 0 in the first round, then the new
        // candidates) refresh their ancestors once each
        {
            const int end_j = sp[v + 1];
            int base_j = sp[v];
            for (bool first = true;; first = false) {
                const int off = first ? 1 : 0;
                const int j = base_j + lane - off;
                int changed = -1;
                if (first && lane == 0) {
                    changed = v;
                } else if (j < end_j) {
                    const int w = si[j];
                    if (--npl[w] == 0) {
                        atomicOr(&cand[w >> 5], 1u << (w & 31));
                        changed = w;
                    }
                }
                __syncwarp();
                T.update_many(changed);
                base_j += 32 - off;
                if (base_j >= end_j) break;
            }
        }
        FP_PHASE_END(pw, 7);
    }
    FP_PHASE_FLUSH(0);
}

// ---------------------------------------------------------------------------
// PLC warp
// ---------------------------------------------------------------------------
// FULLD: the cluster has exactly MAXD devices and the hidden width is 32 * HPL,
// so every `d < D` / `lane < D` / `j < h` test folds away at compile time (the
// hot LEAN instantiations).
template <int MAXD, int HPL, bool GRAD, bool WIDE = false, bool LEAN = false, bool FULLD = false>
__device__ __forceinline__ int plc_chain(const DevProblem &PR, const DevPolicy &PO,
                                         const fp_rollout_args &A, uint8_t *nb, uint8_t *sb,
                                         const EpLayout &L, int ep, bool want_lp,
                                         bool want_amax) {
    static_assert(!(WIDE && GRAD), "REINFORCE rows are produced by the compact path only");
    const int lane = lane_id();
    const int n = PR.n, D = FULLD ? MAXD : PR.d, h = FULLD ? 32 * HPL : PO.h;
    constexpr int LOGD = PlcLog<MAXD>::v;
    double *tstart = (double *)(nb + L.tstart);
    double *tend = (double *)(nb + L.tend);
    double *xd = (double *)(sb + L.xd);
    double *xn = (double *)(sb + L.xn);
    double *stats = (double *)(sb + L.stats);
    const volatile int *order = (const volatile int *)(nb + L.order);
    volatile int *ring = (volatile int *)(sb + L.ring);
    volatile int *dead = (volatile int *)(sb + L.flag);
    uint8_t *dev = nb + L.assign;
    const double eps = A.epsilon, ome = 1.0 - eps, slope = PO.slope;
    const uint32_t k0 = (uint32_t)A.seed, k1 = (uint32_t)(A.seed >> 32);
    const uint32_t ctr_ep = A.episode_base + (uint32_t)ep;
    const int mode = LEAN ? FP_MODE_SAMPLE : A.mode;
    const int32_t *frow = mode == FP_MODE_FORCED ? A.forced + (size_t)ep * n * 2 : nullptr;
    const double *__restrict__ Atab = PO.A;
    const double *__restrict__ Gtab = PO.G;
    const int *__restrict__ pp = PR.pred_ptr;
    const int *__restrict__ pi = PR.pred_idx;
    const uint8_t *__restrict__ ent = PR.is_entry;
    const double *__restrict__ flops = PR.flops;
    const double *__restrict__ tdur = PR.tdur;
    const double *__restrict__ edur = PR.edur;
    const double b2p = PO.W(PR_PLC_H2_B)[0];
    double *rec_x = GRAD ? A.grad_rows : nullptr;  // decision records (GRAD)

#pragma unroll 1
    for (int v = lane; v < n; v += 32) { tstart[v] = 0.0; tend[v] = 0.0; dev[v] = 0xFF; }
    double avail = 0.0, aflops = 0.0;  // lane d < D
    double Mr[5][HPL], cr[HPL], w2r[HPL], Sd[MAXD][HPL];
    {
        const double *w2p = PO.W(PR_PLC_H2_W);
#pragma unroll
        for (int t = 0; t < HPL; ++t) {
            const int j = lane + 32 * t;
            const bool ok = j < h;
#pragma unroll
            for (int c = 0; c < 5; ++c) Mr[c][t] = ok ? PO.M[c * h + j] : 0.0;
            cr[t] = ok ? PO.c[j] : 0.0;
            w2r[t] = ok ? w2p[j] : 0.0;
#pragma unroll
            for (int d = 0; d < MAXD; ++d) Sd[d][t] = 0.0;
        }
    }
    __syncwarp();
    int status = FP_EP_OK;
    FP_PHASE_DECL;
    FP_PHASE_BEGIN(pp_);
    double dc1 = 0.0, dc2 = 0.0;  // draw cache (step_draw)
    for (int step = 0; step < n; ++step) {
        double u1 = 0.0, u2 = 0.0;
        if (mode == FP_MODE_SAMPLE) step_draw(step, ctr_ep, 1u, k0, k1, dc1, dc2, u1, u2);
        int v;
        if constexpr (WIDE) {
            // single-producer / single-consumer ring: the SEL warp refills a
            // slot only after this warp hands it back (-3)
            const int slot = step & (kRing - 1);
            while ((v = ring[slot]) == -3) { }
            __syncwarp();
            if (lane == 0) ring[slot] = -3;
        } else {
            while ((v = order[step]) == -3) { }
        }
        if (v < 0) { status = v == -1 ? FP_EP_DEADLOCK : FP_EP_BAD_ACTION; break; }
        FP_PHASE_END(pp_, 10);
        double Av[HPL], Gv[HPL];
#pragma unroll
        for (int t = 0; t < HPL; ++t) {
            const int j = lane + 32 * t;
            Av[t] = j < h ? Atab[(size_t)v * h + j] : 0.0;
            Gv[t] = j < h ? Gtab[(size_t)v * h + j] : 0.0;
        }
        // the commit's operands, loaded now (off the decision -> commit chain):
        // lane d holds v's duration on device d
        const double fl_v = flops[v];
        const bool ent_v = ent[v] != 0;
        const double edur_v = lane < D ? edur[v * D + lane] : 0.0;
        // ---- device features, lane = device (policy.py:240-246) ----
        double f4 = 0.0;
        if (lane < D) {
            double f2 = 0.0, f3 = 0.0;
            fp::NeuSum f1;
            bool any_local = false;
            const int p0 = pp[v], p1 = pp[v + 1];
            // two predecessors per trip: both load chains (index -> device ->
            // transfer time) in flight together, folded in predecessor order
#pragma unroll 1
            for (int j = p0; j < p1; j += 2) {
                const bool two = j + 1 < p1;
                const int pa = pi[j], pb = two ? pi[j + 1] : pa;
                const int da = dev[pa], db = dev[pb];
                const bool ea = ent[pa] != 0, eb = ent[pb] != 0;
                const double ta = tend[pa], tb = tend[pb];
                const double ra = tdur[(pa * D + da) * D + lane], rb = tdur[(pb * D + db) * D + lane];
                const double fa = flops[pa], fb = flops[pb];
                const double sa = tstart[pa], sbb = tstart[pb];
                // arrival = end + transfer (0.0 on the same device), timeline.py:30-35
                const double arra = ea ? 0.0 : __dadd_rn(ta, ra);
                f3 = j == p0 ? arra : fmax(f3, arra);
                if (da == lane) {
                    f1.add(fa);
                    f2 = any_local ? fmin(f2, sa) : sa;
                    any_local = true;
                }
                if (two) {
                    const double arrb = eb ? 0.0 : __dadd_rn(tb, rb);
                    f3 = fmax(f3, arrb);
                    if (db == lane) {
                        f1.add(fb);
                        f2 = any_local ? fmin(f2, sbb) : sbb;
                        any_local = true;
                    }
                }
            }
            f4 = fmax(avail, f3);
            double *xr = xd + lane * 5;
            xr[0] = aflops; xr[1] = f1.value(); xr[2] = f2; xr[3] = f3; xr[4] = f4;
        }
        __syncwarp();
        FP_PHASE_END(pp_, 11);
        // ---- column statistics: lane c < 5 sums over devices in order ----
        if (lane < 5) {
            double col[MAXD];
#pragma unroll
            for (int d = 0; d < MAXD; ++d) col[d] = d < D ? xd[d * 5 + lane] : 0.0;
            double sum = 0.0;
#pragma unroll
            for (int d = 0; d < MAXD; ++d)
                if (d < D) sum = __dadd_rn(sum, col[d]);
            // x / D == x * (1/D) exactly when D is a power of two (same real
            // value, one rounding): the reference's mean bit for bit
            const bool pow2 = (D & (D - 1)) == 0;
            const double invD = 1.0 / (double)D;
            const double mean = pow2 ? __dmul_rn(sum, invD) : __ddiv_rn(sum, (double)D);
            double sq = 0.0;
#pragma unroll
            for (int d = 0; d < MAXD; ++d)
                if (d < D) {
                    const double df = __dsub_rn(col[d], mean);
                    sq = __dadd_rn(sq, __dmul_rn(df, df));
                }
            const double var = pow2 ? __dmul_rn(sq, invD) : __ddiv_rn(sq, (double)D);
            stats[lane] = mean;
            // the reference's guard std < 1e-12 decided exactly on the variance
            // (sqrt_rn is monotone and sqrt_rn(v) < 1e-12 <=> v < 1e-24, checked
            // at the double boundary); the scaling is one rsqrt per column (within
            // ~1 ulp of 1 / sqrt_rn(var), a third of the sqrt + divide sequence)
            stats[5 + lane] = var < 1e-24 ? 1.0 : rsqrt(var);
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < (5 * MAXD + 31) / 32; ++t) {
            const int i = lane + 32 * t;
            if (i < 5 * D) {
                const int c = i % 5;
                xn[i] = __dmul_rn(__dsub_rn(xd[i], stats[c]), stats[5 + c]);
            }
        }
        __syncwarp();
        FP_PHASE_END(pp_, 12);
        // ---- pre-activations + head2 partial sums (lane = hidden column) ----
        double pre[MAXD][HPL];
        double part[MAXD];
#pragma unroll
        for (int d = 0; d < MAXD; ++d) {
            part[d] = 0.0;
#pragma unroll
            for (int t = 0; t < HPL; ++t) pre[d][t] = 0.0;
            if (d < D) {
                const double x0 = xn[d * 5], x1 = xn[d * 5 + 1], x2 = xn[d * 5 + 2],
                             x3 = xn[d * 5 + 3], x4 = xn[d * 5 + 4];
#pragma unroll
                for (int t = 0; t < HPL; ++t) {
                    double a = Av[t] + Sd[d][t] + cr[t];
                    a = fma(x0, Mr[0][t], a);
                    a = fma(x1, Mr[1][t], a);
                    a = fma(x2, Mr[2][t], a);
                    a = fma(x3, Mr[3][t], a);
                    a = fma(x4, Mr[4][t], a);
                    pre[d][t] = a;
                    part[d] = fma(lk(a, slope), w2r[t], part[d]);
                }
            }
        }
        // transpose reduction: after LOGD halving rounds lane l holds a partial
        // for device (l >> (5 - LOGD)) & (MAXD-1); the xor rounds finish it
        {
#pragma unroll
            for (int r = 0; r < LOGD; ++r) {
                const int o = 16 >> r;
                const bool upper = (lane & o) != 0;
                const int half = MAXD >> (r + 1);
#pragma unroll
                for (int i = 0; i < MAXD / 2; ++i) {
                    if (i < half) {
                        const double send = upper ? part[i] : part[i + half];
                        const double keep = upper ? part[i + half] : part[i];
                        part[i] = keep + __shfl_xor_sync(FP_FULL_MASK, send, o);
                    }
                }
            }
#pragma unroll
            for (int o = 16 >> LOGD; o > 0; o >>= 1)
                part[0] += __shfl_xor_sync(FP_FULL_MASK, part[0], o);
        }
        const double lgall = __shfl_sync(FP_FULL_MASK, part[0], (lane & (MAXD - 1)) << (5 - LOGD));
        FP_PHASE_END(pp_, 13);
        const double lg = lane < D ? lgall + b2p : -INFINITY;
        const double lmx = warp_max_redux(lg);
        const double ed = lane < D ? exp(lg - lmx) : 0.0;
        const double ecum = warp_scan_pow2<LOGD>(ed);
        const double etot = __shfl_sync(FP_FULL_MASK, ecum, D - 1);
        double pd = -1.0;  // only the log-prob / argmax consumers need p
        if ((want_lp || want_amax || mode == FP_MODE_GREEDY) && lane < D) pd = ed / etot;
        int amax = -1;
        if (want_amax || mode == FP_MODE_GREEDY) {
            double am = pd;
            int ai = lane < D ? lane : 0x7fffffff;
            warp_argmax_first(am, ai);
            amax = ai;
        }
        FP_PHASE_END(pp_, 14);
        int jdx;
        if (mode == FP_MODE_FORCED) {
            jdx = frow[2 * step + 1];
            if (jdx < 0 || jdx >= D) {
                status = FP_EP_BAD_ACTION;
                if (WIDE && lane == 0) *dead = 1;  // release a producer blocked on the ring
                break;
            }
        } else if (mode == FP_MODE_TEACHER) {
            // argmin earliest start, first device on ties (heuristics.py:85-91)
            const double tv = lane < D ? f4 : INFINITY;
            const double best = warp_min_redux(tv);
            jdx = __ffs(__ballot_sync(FP_FULL_MASK, lane < D && tv == best)) - 1;
        } else if (mode == FP_MODE_GREEDY) {
            jdx = amax;
        } else {
            if (u1 < eps) {
                jdx = min((int)(u2 * (double)D), D - 1);
            } else {
                const unsigned hit = __ballot_sync(FP_FULL_MASK, lane < D && ecum > u2 * etot);
                jdx = hit ? __ffs(hit) - 1 : D - 1;
            }
        }
        FP_PHASE_END(pp_, 15);
        if (want_lp) {
            const double ekd = eps / (double)D;
            double mixd = 0.0, lmd = 0.0;
            if (lane < D) {
                mixd = __dadd_rn(__dmul_rn(pd, ome), ekd);
                lmd = log(__dadd_rn(mixd, 1e-30));
            }
            const double entv = -warp_sum(lane < D ? mixd * lmd : 0.0);
            const double lp = __shfl_sync(FP_FULL_MASK, lmd, jdx);
            if (lane == 0) {
                const size_t o = (size_t)ep * n + step;
                if (A.step_lp) A.step_lp[2 * o + 1] = lp;
                if (A.step_ent) A.step_ent[2 * o + 1] = entv;
            }
        }
        if constexpr (GRAD) {  // decision record: the adjoints are formed by fp_pg_reduce
            double *rec = rec_x + ((size_t)ep * n + step) * grad_rec_stride(D, PR.W);
            for (int i = lane; i < 5 * D; i += 32) rec[i] = xn[i];
            if (lane < D) rec[5 * D + lane] = lg;
            if (lane == 0) *(int2 *)(rec + 6 * D) = make_int2(v, jdx);
        }
        FP_PHASE_END(pp_, 16);
        // ---- commit (timeline.py:47-58) ----
        if (lane == jdx) {
            aflops = __dadd_rn(aflops, fl_v);
            if (!ent_v) {
                const double en = __dadd_rn(f4, edur_v);
                tstart[v] = f4;
                tend[v] = en;
                avail = en;
            }
            dev[v] = (uint8_t)jdx;
            if constexpr (!WIDE) {  // release the placement to the overlapped simulator
                __threadfence_block();
                *(volatile int *)(sb + L.flag) = step + 1;
            }
            if (A.step_vd) A.step_vd[2 * ((size_t)ep * n + step) + 1] = jdx;
        }
        if (lane == 0 && A.step_argmax) A.step_argmax[2 * ((size_t)ep * n + step) + 1] = amax;
#pragma unroll
        for (int d = 0; d < MAXD; ++d)
            if (d == jdx)
#pragma unroll
                for (int t = 0; t < HPL; ++t) Sd[d][t] += Gv[t];
        __syncwarp();
        FP_PHASE_END(pp_, 17);
    }
    FP_PHASE_FLUSH(0);
    if constexpr (GRAD)
        if (lane == 0) {
            double *g = A.grad_ep + (size_t)ep * grad_ep_stride(n, h, D);
            g[2 * n] = status == FP_EP_OK ? 1.0 : 0.0;
            g[2 * n + 1] = eps;
        }
    return status;
}

// REINFORCE terms of the SEL decisions, off both decision chains: steps
// [t0, t1) of the recorded SEL decisions, run by a warp that would otherwise
// wait -- the PLC warp once its chain is done (the first ~70% of the steps)
// and the SEL warp once the simulation is done (the rest).  Per step the
// recorded candidate bitset is compacted to the ascending candidate list
// and, with the recorded softmax max / normaliser, the mixture's log-prob /
// entropy adjoints w.r.t. the SEL logits (policy.py:186-204, 301-322 in
// reverse) accumulate into dsl (dlp/ds) and dse (dent/ds) per vertex (lane
// = candidate, one update per candidate per step, steps in order).
__device__ __forceinline__ int sel_grad_split(int n) { return (7 * n) / 10; }

__device__ __forceinline__ void sel_grad_terms(const DevProblem &PR, const fp_rollout_args &A,
                                               const double *s_sm, int ep, int t0, int t1,
                                               int *cl, double *dsl, double *dse) {
    const int lane = lane_id();
    const int n = PR.n, D = PR.d, W = PR.W;
    const double eps = A.epsilon, ome = 1.0 - eps;
    const int rstride = grad_rec_stride(D, W);
    const double *rec = A.grad_rows + (size_t)ep * n * rstride;
#pragma unroll 1
    for (int v = lane; v < n; v += 32) { dsl[v] = 0.0; dse[v] = 0.0; }
    if (t0 >= t1) { __syncwarp(); return; }
    // step t's record fields, fetched one step ahead
    auto fetch = [&](int t, int &v, double &mx, double &tot, uint32_t &cw) {
        const double *r = rec + (size_t)t * rstride;
        mx = r[6 * D + 1];
        tot = r[6 * D + 2];
        v = (int)r[6 * D + 3];
        cw = lane < W ? ((const uint32_t *)(r + 6 * D + 4))[lane] : 0u;
    };
    int v, nv = 0;
    double mx, tot, nmx = 0.0, ntot = 0.0;
    uint32_t cw, ncw = 0u;
    fetch(t0, v, mx, tot, cw);
    __syncwarp();
#pragma unroll 1
    for (int t = t0; t < t1; ++t) {
        if (t + 1 < t1) fetch(t + 1, nv, nmx, ntot, ncw);
        const int pc = __popc(cw);
        const int incl = warp_inclusive_scan(pc);
        const int k = __shfl_sync(FP_FULL_MASK, incl, 31);
        {
            int o = incl - pc;
            uint32_t m = cw;
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                cl[o++] = lane * 32 + b;
            }
        }
        __syncwarp();
        const double ek = eps / (double)k;
        double p0 = 0.0, q0 = 0.0, acc = 0.0;
#pragma unroll 1
        for (int i = lane; i < k; i += 32) {
            const double p = exp(s_sm[cl[i]] - mx) / tot;
            const double mix = __dadd_rn(__dmul_rn(p, ome), ek);
            const double lm = log(__dadd_rn(mix, 1e-30));
            const double q = -ome * (lm + mix / __dadd_rn(mix, 1e-30));
            acc += q * p;
            if (i < 32) { p0 = p; q0 = q; }
        }
        const double qp = warp_sum(acc);
        const double pv = exp(s_sm[v] - mx) / tot;
        const double mv = __dadd_rn(__dmul_rn(pv, ome), ek);
        const double c1 = ome * pv / __dadd_rn(mv, 1e-30);
#pragma unroll 1
        for (int i = lane; i < k; i += 32) {
            double p = p0, q = q0;
            if (i >= 32) {
                p = exp(s_sm[cl[i]] - mx) / tot;
                const double mix = __dadd_rn(__dmul_rn(p, ome), ek);
                const double lm = log(__dadd_rn(mix, 1e-30));
                q = -ome * (lm + mix / __dadd_rn(mix, 1e-30));
            }
            const int u = cl[i];
            dsl[u] += c1 * ((u == v ? 1.0 : 0.0) - p);
            dse[u] += p * (q - qp);
        }
        __syncwarp();
        v = nv; mx = nmx; tot = ntot; cw = ncw;
    }
}

// Which warp of an episode's (SEL, PLC) pair runs the PLC chain, by hardware
// warp slot (%warpid; scheduler = slot % 4, see rollout_kernel).  All threads
// of the block call it (one barrier); slots: 2 x (pairs in the block).
__device__ __forceinline__ bool plc_role(unsigned *slots, int warp) {
    unsigned ws;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(ws));
    if (lane_id() == 0) slots[warp] = ws;
    __syncthreads();
    const unsigned s0 = slots[warp & ~1], s1 = slots[warp | 1];
    const bool p0 = (s0 & 1u) == ((s0 >> 2) & 1u), p1 = (s1 & 1u) == ((s1 >> 2) & 1u);
    return p0 != p1 ? ((warp & 1) ? p1 : p0) : (warp & 1) != 0;
}

// LEAN: the sampling-only instantiation (no forced / teacher / greedy modes,
// no per-step outputs, no traces) -- a smaller kernel for the throughput path
// (fewer instruction-fetch stalls with SEL, PLC and simulator code resident).
template <int MAXD, int HPL, bool GRAD, int EPB, bool SM1, bool LEAN = false, bool FULLD = false>
__global__ void __launch_bounds__(EPB * 64, 8 / EPB)
rollout_kernel(DevProblem PR, DevPolicy PO, fp_rollout_args A, EpLayout L) {
    extern __shared__ __align__(16) uint8_t smem[];
    constexpr int RPL = (MAXD + MAXD * MAXD + 31) / 32;
    const int lane = lane_id();
    const int warp = threadIdx.x >> 5;
    const int slot = warp >> 1;  // episode slot in the block
    // Role by hardware warp slot (%warpid; scheduler = slot % 4): blocks of
    // two warps take slot pairs (2b, 2b + 1), so "odd warp = PLC" would put
    // every latency-critical PLC warp on schedulers 1 and 3.  Choosing the
    // PLC warp by (slot & 1) == ((slot >> 2) & 1) spreads them over all four;
    // any other slot pattern falls back to warp 1 (both warps decide alike).
    __shared__ unsigned hw_slot[2 * EPB];
    FP_T0_DECL(t0_);
    const bool is_plc = plc_role(hw_slot, warp);
    const int ep = blockIdx.x * EPB + slot;
    const int n = PR.n;
    double *s_sm = (double *)smem;
    uint8_t *base = smem + fp_align(8 * n, 16) + (size_t)slot * L.bytes;
    volatile int *flag = (volatile int *)(base + L.flag);  // [0] placed, [1] PLC abort
    if (!is_plc) {
        volatile int *order = (volatile int *)(base + L.order);
#pragma unroll 1
        for (int t = lane; t < n; t += 32) order[t] = -3;  // hand-off sentinel
        if (lane == 0) { flag[0] = 0; flag[1] = 0; }
    }
    // (PDL) everything above overlaps the encoder's tail; its tables from here
    griddep_wait();
    // block-shared SEL logits (every episode of the batch uses one snapshot)
    for (int v = threadIdx.x; v < n; v += blockDim.x) s_sm[v] = PO.s[v];
    __syncthreads();
    if (ep >= A.B) return;
    const bool want_out = !LEAN && (A.step_lp != nullptr || A.step_ent != nullptr);
    const bool want_amax = !LEAN && A.step_argmax != nullptr;
    double *simres = (double *)(base + L.simres);  // makespan, status
    int status = FP_EP_OK;
    if (!is_plc) {
        // SEL warp: the vertex order, then -- while the PLC warp is still
        // placing -- the simulation, chasing the placement frontier
        const bool ok = sel_chain<GRAD, LEAN>(PR, PO, A, base, L, s_sm, ep, want_out, want_amax);
        FP_MARK(40, t0_);
        if constexpr (GRAD)  // no simulation to chase: the second part of the SEL terms now
            if (ok && !A.simulate)
                sel_grad_terms(PR, A, s_sm, ep, sel_grad_split(n), n, (int *)(base + L.clist),
                               (double *)(base + L.ce), (double *)(base + L.cc));
        if (ok && A.simulate) {
            const volatile int *order = (const volatile int *)(base + L.order);
            int *pos = (int *)(base + L.clist);     // SEL scratch, free now
            int *maxsucc = (int *)(base + L.npl);
#pragma unroll 1
            for (int i = lane; i < n; i += 32) pos[order[i]] = i;
            __syncwarp();
            int iw = -1;
#pragma unroll 1
            for (int v = lane; v < n; v += 32) {
                int m = -1;
#pragma unroll 1
                for (int j = PR.succ_ptr[v]; j < PR.succ_ptr[v + 1]; ++j) m = max(m, pos[PR.succ_idx[j]]);
                maxsucc[v] = m;
                if (!PR.is_entry[v]) {
                    bool all_entry = true;
#pragma unroll 1
                    for (int j = PR.pred_ptr[v]; j < PR.pred_ptr[v + 1]; ++j)
                        all_entry &= PR.is_entry[PR.pred_idx[j]] != 0;
                    if (all_entry) iw = max(iw, pos[v]);
                }
            }
            iw = __reduce_max_sync(FP_FULL_MASK, iw);
            __syncwarp();
            SimOut o = sim_episode<RPL, false, SM1, true, FULLD ? MAXD : 0, LEAN>(
                PR, base, base, L, A.strategy, nullptr,
                (!LEAN && A.trace) ? A.trace + (size_t)ep * A.trace_cap : nullptr, A.trace_cap,
                nullptr,
                SimSync{flag, flag + 1, maxsucc, iw});
            FP_MARK(42, t0_);
            // second part of the SEL terms (SEL / simulator scratch, free now)
            if constexpr (GRAD)
                if (o.status == FP_EP_OK && !flag[1])
                    sel_grad_terms(PR, A, s_sm, ep, sel_grad_split(n), n, (int *)(base + L.clist),
                                   (double *)(base + L.ce), (double *)(base + L.cc));
            if (lane == 0) {
                simres[0] = o.makespan;
                ((int *)simres)[2] = o.status;
                if (A.trace_len) A.trace_len[ep] = o.n_events;
            }
        }
    } else {
        status = plc_chain<MAXD, HPL, GRAD, false, LEAN, FULLD>(PR, PO, A, base, base, L, ep, want_out,
                                                         want_amax);
        FP_MARK(41, t0_);
        if (status != FP_EP_OK && lane == 0) flag[1] = 1;  // release a waiting simulator
        if constexpr (GRAD)  // first part of the SEL terms (cons: unused by the overlapped sim)
            if (status == FP_EP_OK)
                sel_grad_terms(PR, A, s_sm, ep, 0, sel_grad_split(n), (int *)(base + L.cons),
                               (double *)(base + L.dsl), (double *)(base + L.dse));
        const uint8_t *dev = base + L.assign;
#pragma unroll 1
        for (int v = lane; v < n; v += 32)
            A.assign[(size_t)ep * n + v] = dev[v] == 0xFF ? -1 : dev[v];
    }
    __syncthreads();
    if constexpr (GRAD)
        if (is_plc && status == FP_EP_OK &&
            (!A.simulate || ((const int *)simres)[2] == FP_EP_OK)) {  // the two parts of the SEL terms
            const double *dsl = (const double *)(base + L.dsl), *dse = (const double *)(base + L.dse);
            const double *dsl2 = (const double *)(base + L.ce), *dse2 = (const double *)(base + L.cc);
            double *g = A.grad_ep + (size_t)ep * grad_ep_stride(n, PO.h, PR.d);
#pragma unroll 1
            for (int u = lane; u < n; u += 32) {
                g[u] = dsl[u] + dsl2[u];
                g[n + u] = dse[u] + dse2[u];
            }
        }
    if (is_plc && lane == 0) {
        double mk = 0.0;
        if (status == FP_EP_OK && A.simulate) {
            mk = simres[0];
            status = ((const int *)simres)[2];
        }
        if (A.makespan) A.makespan[ep] = mk;
        A.status[ep] = status;
    }
}

// Stage-II REINFORCE replay (fp_pg_reduce), off the rollout's latency-bound
// decision chains: the rollout only records each PLC decision (normalised
// device features, logits, vertex / device; grad_rec_stride), and its idle
// warps fold the SEL decisions' terms into grad_ep (sel_grad_terms).
// plc_replay_kernel, one CTA of kChunkWarps warps per episode:
//   1. the placement order from the records (thread = step);
//   2. PLC adjoints (thread = step): the device softmax of the recorded
//      logits, the sampled mixture's log-prob / entropy adjoints
//      (policy.py:301-322 in reverse), folded with the episode's
//      coefficients: c_d = alpha_e dlp/dlogit_d + beta dent/dlogit_d;
//   3. PLC rows (warp = chunk of consecutive steps, lane = hidden column):
//      each chunk warp rebuilds S_d at its first step (prefix of the placed G
//      rows, in step order), then replays its steps: pre-activations from
//      (A, G, M, c) and xn, folded rows (dA row; the chunk-local running
//      per-device sum at placement, for dG) into a [B][n][2h] slab, and
//      chunk sums.  The chunk totals give, per chunk, final-sum-minus-
//      prefix tables, so dG needs no second pass over the episode.
// pg_rows_kernel contracts the slab over the episodes (a streaming pass,
// episode chunks in parallel, each in episode order; plus the SEL terms of
// grad_ep with alpha / beta) and pg_final_kernel sums the chunk partials in
// chunk order: bitwise deterministic, no atomics.
constexpr int kChunkWarps = 2;
constexpr int kPgChunks = 16;

__host__ __device__ inline int64_t pg_part_stride(int n, int h) {
    return 2LL * n * h + 6LL * h + 1 + n;  // dA | dG | dM dw2 db2 | ds
}

template <int MAXD, int HPL>
__global__ void __launch_bounds__(kChunkWarps * 32)
plc_replay_kernel(DevProblem PR, DevPolicy PO, const double *__restrict__ rec, int rstride,
                  const double *__restrict__ gep, int64_t gstride,
                  const double *__restrict__ alpha, double beta, int B, double *__restrict__ cbuf,
                  double *__restrict__ slab, double *__restrict__ tbuf, double *__restrict__ sbuf,
                  int *__restrict__ posbuf) {
    griddep_launch();
    griddep_wait();  // (PDL) predecessor complete before any access
    constexpr int K = kChunkWarps;
    __shared__ double stage[K][2][6 * MAXD];
    // dynamic: rtot[K][D][h] | rsm[K][6h+1] | vt[n] jt[n]
    extern __shared__ __align__(16) double dyn[];
    const int e = blockIdx.x;
    const int n = PR.n, D = PR.d, h = PO.h, W = PR.W;
    const double *ge = gep + (size_t)e * gstride;
    if (ge[2 * n] == 0.0) return;  // failed chain: no contribution (pg_rows skips it)
    const int lane = lane_id();
    const int wi = threadIdx.x >> 5;
    const int tid = threadIdx.x, nth = blockDim.x;
    FP_PHASE_DECL;
    FP_PHASE_BEGIN(rp_);
    double *rtot = dyn;
    double *rsm = rtot + (size_t)K * D * h;
    int *vt = (int *)(rsm + (size_t)K * (6 * h + 1)), *jt = vt + n;
    const double al = alpha[e];
    const double eps = ge[2 * n + 1], ome = 1.0 - eps, ekd = eps / (double)D;
    const double *recd = rec + (size_t)e * n * rstride;
    auto recp = [&](int t) { return recd + (size_t)t * rstride; };
    // ---- 1. placement order ----
    for (int t = tid; t < n; t += nth) {
        const int2 vj = *(const int2 *)(recp(t) + 6 * D);
        vt[t] = vj.x;
        jt[t] = vj.y;
        posbuf[(size_t)e * n + vj.x] = t;
    }
    __syncthreads();
    FP_PHASE_END(rp_, 25);
    // ---- 2. PLC adjoints (thread = step) ----
    double *cep = cbuf + (size_t)e * n * D;
    for (int t = tid; t < n; t += nth) {
        const double *r = recp(t);
        const double *lg = r + 5 * D;
        const int jdx = ((const int2 *)(r + 6 * D))->y;
        double mx = -INFINITY;
        for (int d = 0; d < D; ++d) mx = fmax(mx, lg[d]);
        double ed[MAXD], tot = 0.0;
#pragma unroll
        for (int d = 0; d < MAXD; ++d) {
            ed[d] = d < D ? exp(lg[d] - mx) : 0.0;
            tot += ed[d];
        }
        double pd[MAXD], q[MAXD], qp = 0.0, pj = 0.0, mj = 0.0;
#pragma unroll
        for (int d = 0; d < MAXD; ++d) {
            if (d >= D) { pd[d] = q[d] = 0.0; continue; }
            pd[d] = ed[d] / tot;
            const double mix = __dadd_rn(__dmul_rn(pd[d], ome), ekd);
            const double lm = log(__dadd_rn(mix, 1e-30));
            q[d] = -ome * (lm + mix / __dadd_rn(mix, 1e-30));
            qp += q[d] * pd[d];
            if (d == jdx) { pj = pd[d]; mj = mix; }
        }
        const double g0 = ome * pj / __dadd_rn(mj, 1e-30);
#pragma unroll
        for (int d = 0; d < MAXD; ++d)
            if (d < D)
                cep[(size_t)t * D + d] =
                    al * (g0 * ((d == jdx ? 1.0 : 0.0) - pd[d])) + beta * (pd[d] * (q[d] - qp));
    }
    __syncthreads();
    FP_PHASE_END(rp_, 26);
    // ---- 3. PLC rows, warp = chunk of steps, lane = hidden column ----
    const int L = (n + K - 1) / K;
    const int t0 = min(n, wi * L), t1 = min(n, t0 + L);
    const double slope = PO.slope;
    const double *__restrict__ Atab = PO.A;
    const double *__restrict__ Gtab = PO.G;
    double Mr[5][HPL], cr[HPL], w2r[HPL], Sd[MAXD][HPL], rc[MAXD][HPL], dM[5][HPL], dw[HPL];
    double db2 = 0.0;
    {
        const double *w2p = PO.W(PR_PLC_H2_W);
#pragma unroll
        for (int t = 0; t < HPL; ++t) {
            const int j = lane + 32 * t;
            const bool in = j < h;
#pragma unroll
            for (int c = 0; c < 5; ++c) { Mr[c][t] = in ? PO.M[c * h + j] : 0.0; dM[c][t] = 0.0; }
            cr[t] = in ? PO.c[j] : 0.0;
            w2r[t] = in ? w2p[j] : 0.0;
            dw[t] = 0.0;
#pragma unroll
            for (int d = 0; d < MAXD; ++d) Sd[d][t] = rc[d][t] = 0.0;
        }
    }
    // S_d at the chunk's first step: the placed G rows, in step order (rows
    // fetched four steps at a time)
#pragma unroll 1
    for (int tb = 0; tb < t0; tb += 4) {
        double g4[4][HPL];
        int j4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int t = tb + u;
            j4[u] = t < t0 ? jt[t] : -1;
            const int v = t < t0 ? vt[t] : 0;
#pragma unroll
            for (int q = 0; q < HPL; ++q) {
                const int j = lane + 32 * q;
                g4[u][q] = (t < t0 && j < h) ? Gtab[(size_t)v * h + j] : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int q = 0; q < HPL; ++q)
#pragma unroll
                for (int d = 0; d < MAXD; ++d)
                    if (d == j4[u]) Sd[d][q] += g4[u][q];
    }
    FP_PHASE_END(rp_, 29);
    const int RS = 6 * D;  // staged: xn[5D] | c[D]
    double *myslab = slab + (size_t)e * n * 2 * h;
    if (t0 < t1) {
        double *st0 = stage[wi][0];
        for (int i = lane; i < RS; i += 32)
            st0[i] = i < 5 * D ? recp(t0)[i] : cep[(size_t)t0 * D + i - 5 * D];
        int vv = vt[t0], jj = jt[t0];
        double Av[HPL], Gv[HPL];
#pragma unroll
        for (int q = 0; q < HPL; ++q) {
            const int j = lane + 32 * q;
            Av[q] = j < h ? Atab[(size_t)vv * h + j] : 0.0;
            Gv[q] = j < h ? Gtab[(size_t)vv * h + j] : 0.0;
        }
        __syncwarp();
#pragma unroll 1
        for (int step = t0; step < t1; ++step) {
            const double *x = stage[wi][(step - t0) & 1];
            const int v = vv, jdx = jj;
            // fetch the next record and vertex rows while this step is replayed
            double nx[(6 * MAXD + 31) / 32], nA[HPL], nG[HPL];
            if (step + 1 < t1) {
                const double *nr = recp(step + 1);
                const int nv = vt[step + 1];
#pragma unroll
                for (int k = 0; k < (6 * MAXD + 31) / 32; ++k) {
                    const int i = lane + 32 * k;
                    nx[k] = i < 5 * D ? nr[i] : i < RS ? cep[(size_t)(step + 1) * D + i - 5 * D] : 0.0;
                }
#pragma unroll
                for (int q = 0; q < HPL; ++q) {
                    const int j = lane + 32 * q;
                    nA[q] = j < h ? Atab[(size_t)nv * h + j] : 0.0;
                    nG[q] = j < h ? Gtab[(size_t)nv * h + j] : 0.0;
                }
            }
            double ar[HPL];
#pragma unroll
            for (int q = 0; q < HPL; ++q) ar[q] = 0.0;
#pragma unroll
            for (int d = 0; d < MAXD; ++d) {
                if (d >= D) continue;
                const double x0 = x[d * 5], x1 = x[d * 5 + 1], x2 = x[d * 5 + 2],
                             x3 = x[d * 5 + 3], x4 = x[d * 5 + 4];
                const double cd = x[5 * D + d];
                if (lane == 0) db2 += cd;
#pragma unroll
                for (int q = 0; q < HPL; ++q) {
                    double a = Av[q] + Sd[d][q] + cr[q];
                    a = fma(x0, Mr[0][q], a);
                    a = fma(x1, Mr[1][q], a);
                    a = fma(x2, Mr[2][q], a);
                    a = fma(x3, Mr[3][q], a);
                    a = fma(x4, Mr[4][q], a);
                    const double df = cd * w2r[q] * lkd(a, slope);
                    dw[q] = fma(cd, lk(a, slope), dw[q]);
                    ar[q] += df;
                    rc[d][q] += df;
                    dM[0][q] = fma(x0, df, dM[0][q]);
                    dM[1][q] = fma(x1, df, dM[1][q]);
                    dM[2][q] = fma(x2, df, dM[2][q]);
                    dM[3][q] = fma(x3, df, dM[3][q]);
                    dM[4][q] = fma(x4, df, dM[4][q]);
                }
            }
            double *row = myslab + (size_t)v * 2 * h;
#pragma unroll
            for (int q = 0; q < HPL; ++q) {
                const int j = lane + 32 * q;
                double sl = 0.0;
#pragma unroll
                for (int d = 0; d < MAXD; ++d)
                    if (d == jdx) { sl = rc[d][q]; Sd[d][q] += Gv[q]; }
                if (j < h) { row[j] = ar[q]; row[h + j] = sl; }
            }
            if (step + 1 < t1) {
                double *ns = stage[wi][(step + 1 - t0) & 1];
#pragma unroll
                for (int k = 0; k < (6 * MAXD + 31) / 32; ++k) {
                    const int i = lane + 32 * k;
                    if (i < RS) ns[i] = nx[k];
                }
#pragma unroll
                for (int q = 0; q < HPL; ++q) { Av[q] = nA[q]; Gv[q] = nG[q]; }
                vv = vt[step + 1];
                jj = jt[step + 1];
            }
            __syncwarp();
        }
    }
    // chunk totals / sums
    {
        double *Tw = rtot + (size_t)wi * D * h;
        double *sw = rsm + (size_t)wi * (6 * h + 1);
#pragma unroll
        for (int q = 0; q < HPL; ++q) {
            const int j = lane + 32 * q;
            if (j >= h) continue;
#pragma unroll
            for (int d = 0; d < MAXD; ++d)
                if (d < D) Tw[d * h + j] = rc[d][q];
#pragma unroll
            for (int c = 0; c < 5; ++c) sw[c * h + j] = dM[c][q];
            sw[5 * h + j] = dw[q];
        }
        if (lane == 0) sw[6 * h] = db2;
    }
    FP_PHASE_END(rp_, 30);
    __syncthreads();
    FP_PHASE_END(rp_, 31);
    FP_PHASE_FLUSH(0);
    // per chunk c: (final per-device sum) - (sum over the chunks before c)
    for (int i = tid; i < D * h; i += nth) {
        double tot = 0.0;
        for (int c = 0; c < K; ++c) tot += rtot[(size_t)c * D * h + i];
        double pre = 0.0;
        for (int c = 0; c < K; ++c) {
            tbuf[((size_t)e * K + c) * D * h + i] = tot - pre;
            pre += rtot[(size_t)c * D * h + i];
        }
    }
    for (int k = tid; k < 6 * h + 1; k += nth) {
        double acc = 0.0;
        for (int c = 0; c < K; ++c) acc += rsm[(size_t)c * (6 * h + 1) + k];
        sbuf[(size_t)e * (6 * h + 1) + k] = acc;
    }
}

// Episode contraction of the replay's slab: item = (v, j) of dA / dG, the
// small sums, and the SEL logits' terms ds[v]; episode chunk = blockIdx.y,
// episodes of a chunk in order.  dG[v] collects, per episode, the final
// per-device sum on v's device minus the running sum at v's placement
// (chunk table of v's step minus the chunk-local running sum).
static __global__ void pg_rows_kernel(DevPolicy P, int D, int B, int L,
                                      const double *__restrict__ slab,
                                      const double *__restrict__ tbuf,
                                      const double *__restrict__ sbuf,
                                      const int *__restrict__ posbuf,
                                      const double *__restrict__ gep, int64_t gstride,
                                      const int32_t *__restrict__ assign,
                                      const double *__restrict__ alpha, double beta,
                                      double *__restrict__ part) {
    griddep_launch();
    griddep_wait();  // (PDL) predecessor complete before any access
    const int n = P.n, h = P.h, nh = n * h;
    const int64_t PSt = pg_part_stride(n, h);
    const int item = blockIdx.x * blockDim.x + threadIdx.x;
    const int per = (B + kPgChunks - 1) / kPgChunks;
    const int e0 = blockIdx.y * per, e1 = min(B, e0 + per);
    double *pc = part + (size_t)blockIdx.y * PSt;
    if (item < nh) {
        const int v = item / h, j = item - v * h;
        double a = 0.0, g = 0.0;
#pragma unroll 4
        for (int e = e0; e < e1; ++e) {
            if (gep[(size_t)e * gstride + 2 * n] == 0.0) continue;  // failed chain
            const double *r = slab + ((size_t)e * n + v) * 2 * h;
            const int dv = assign[(size_t)e * n + v];
            const int c = posbuf[(size_t)e * n + v] / L;
            a += r[j];
            g += tbuf[(((size_t)e * kChunkWarps + c) * D + dv) * h + j] - r[h + j];
        }
        pc[item] = a;
        pc[nh + item] = g;
    } else if (item < nh + 6 * h + 1) {
        const int k = item - nh;
        double acc = 0.0;
        for (int e = e0; e < e1; ++e)
            if (gep[(size_t)e * gstride + 2 * n] != 0.0) acc += sbuf[(size_t)e * (6 * h + 1) + k];
        pc[nh + item] = acc;
    } else if (item < nh + 6 * h + 1 + n) {
        const int v = item - nh - 6 * h - 1;
        double acc = 0.0;
        for (int e = e0; e < e1; ++e)
        {
            const double *g = gep + (size_t)e * gstride;
            if (g[2 * n] != 0.0) acc += alpha[e] * g[v] + beta * g[n + v];
        }
        pc[nh + item] = acc;
    }
}

// chunk partials -> dA, dG, [dM | dw2 | db2], ds, summed in chunk order
static __global__ void pg_final_kernel(DevPolicy P, const double *__restrict__ part) {
    griddep_launch();
    griddep_wait();  // (PDL) predecessor complete before any access
    const int n = P.n, h = P.h, nh = n * h;
    const int64_t PSt = pg_part_stride(n, h);
    const int item = blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= PSt) return;
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < kPgChunks; ++c) acc += part[(size_t)c * PSt + item];
    if (item < nh) P.dA[item] = acc;
    else if (item < 2 * nh) P.dG[item - nh] = acc;
    else if (item < 2 * nh + 6 * h + 1) P.dsmall[h + (item - 2 * nh)] = acc;  // [dc | dM | dw2 | db2]
    else P.ds[item - 2 * nh - 6 * h - 1] = acc;
}

template <int MAXD, int HPL>
int launch_plc_replay(const fp_problem *p, const fp_policy *pol, const double *rec,
                      const double *gep, const int32_t *assign, const double *alpha, double beta,
                      int B, double *scratch, int64_t *scratch_bytes, cudaStream_t st) {
    constexpr int K = kChunkWarps;
    const DevProblem &PR = p->dev;
    const DevPolicy &PO = pol->dev;
    const int n = PR.n, D = PR.d, h = PO.h;
    const int64_t slab_d = (int64_t)B * n * 2 * h, t_d = (int64_t)B * K * D * h,
                  s_d = (int64_t)B * (6 * h + 1), PSt = pg_part_stride(n, h),
                  c_d = (int64_t)B * n * D, pos_d = ((int64_t)B * n + 1) / 2;
    if (scratch_bytes) {
        *scratch_bytes = (slab_d + t_d + s_d + c_d + pos_d + kPgChunks * PSt) * 8;
        return FP_OK;
    }
    double *slab = scratch, *tbuf = slab + slab_d, *sbuf = tbuf + t_d, *part = sbuf + s_d,
           *cbuf = part + kPgChunks * PSt;
    int *posbuf = (int *)(cbuf + c_d);
    const int64_t gstride = grad_ep_stride(n, h, D);
    const int64_t dyn = 8LL * ((int64_t)K * D * h + (int64_t)K * (6 * h + 1)) + 8LL * n;
    auto kern = plc_replay_kernel<MAXD, HPL>;
    cudaError_t e0 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)dyn);
    if (e0 != cudaSuccess) { set_error(cudaGetErrorString(e0)); return FP_ERR_CUDA; }
    launch_pdl(kern, dim3(B), dim3(K * 32), (size_t)dyn, st, PR, PO, rec, grad_rec_stride(D, PR.W),
               gep, gstride, alpha, beta, B, cbuf, slab, tbuf, sbuf, posbuf);
    const int items = n * h + 6 * h + 1 + n;
    launch_pdl(pg_rows_kernel, dim3((items + 127) / 128, kPgChunks), dim3(128), 0, st, PO, D, B,
               (n + K - 1) / K, (const double *)slab, (const double *)tbuf, (const double *)sbuf,
               (const int *)posbuf, gep, gstride, assign, alpha, beta, part);
    launch_pdl(pg_final_kernel, dim3((int)((PSt + 127) / 128)), dim3(128), 0, st, PO,
               (const double *)part);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FP_ERR_CUDA; }
    return FP_OK;
}

template <int MAXD, int HPL, bool GRAD>
int launch_rollout(const fp_problem *p, const fp_policy *pol, const fp_rollout_args &a,
                          cudaStream_t st) {
    constexpr int EPB = 1;
    const DevProblem &PR = p->dev;
    const EpLayout L = make_layout(PR.n, PR.W, PR.R, PR.SM, true, 0);
    const int64_t smem = fp_align(8 * PR.n, 16) + (int64_t)L.bytes * EPB;
    if (GRAD && (!a.grad_rows || !a.grad_ep)) {
        set_error("REINFORCE rollout needs grad_rows (decision records) and grad_ep");
        return FP_ERR_INVALID;
    }
    if (smem > 227 * 1024) {
        set_error("episode state exceeds shared memory for this graph size");
        return FP_ERR_UNSUPPORTED;
    }
    const bool lean = a.mode == FP_MODE_SAMPLE && !a.step_vd && !a.step_lp && !a.step_ent &&
                      !a.step_argmax && !a.step_ncand && !a.trace &&
                      !(a.flags & FP_FLAG_TIE_RANDOM);
    const bool full = PR.d == MAXD && pol->dev.h == 32 * HPL;
    auto kern = PR.SM == 1 ? (lean ? (full ? rollout_kernel<MAXD, HPL, GRAD, EPB, true, true, true>
                                                   : rollout_kernel<MAXD, HPL, GRAD, EPB, true, true>)
                                   : rollout_kernel<MAXD, HPL, GRAD, EPB, true>)
                           : rollout_kernel<MAXD, HPL, GRAD, EPB, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FP_ERR_CUDA; }
    const int grid = (a.B + EPB - 1) / EPB;
    e = launch_pdl(kern, dim3(grid), dim3(EPB * 64), (size_t)smem, st, PR, pol->dev, a, L);
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FP_ERR_CUDA; }
    return FP_OK;
}

// Wide path: persistent grid, one SEL + one PLC warp per resident episode,
// n-sized state in the HBM workspace slice of this block, small scratch and
// the hand-off ring in shared memory.  After the PLC chain the same warp
// scores the assignment with the hierarchical-bitset simulator.
template <int MAXD, int HPL, bool SM1, bool LEAN = false, bool FULLD = false>
__global__ void __launch_bounds__(64, 8)
rollout_wide_kernel(DevProblem PR, DevPolicy PO, fp_rollout_args A, EpLayout L) {
    extern __shared__ __align__(16) uint8_t smem[];
    constexpr int RPL = (MAXD + MAXD * MAXD + 31) / 32;
    const int lane = lane_id();
    __shared__ unsigned hw_slot[2];
    const bool is_plc = plc_role(hw_slot, threadIdx.x >> 5);  // spread over schedulers
    const int n = PR.n;
    uint8_t *sb = smem;
    uint8_t *nb = (uint8_t *)A.workspace + (size_t)blockIdx.x * L.gbytes;
    const bool want_lp = !LEAN && (A.step_lp != nullptr || A.step_ent != nullptr);
    const bool want_amax = !LEAN && A.step_argmax != nullptr;
    for (int ep = blockIdx.x; ep < A.B; ep += gridDim.x) {
        if (!is_plc) {
            volatile int *ring = (volatile int *)(sb + L.ring);
            for (int t = lane; t < kRing; t += 32) ring[t] = -3;
            if (lane == 0) *(volatile int *)(sb + L.flag) = 0;
        }
        __syncthreads();
        if (!is_plc) {
            sel_chain_wide<LEAN>(PR, PO, A, nb, sb, L, ep, want_lp, want_amax);
        } else {
            int status = plc_chain<MAXD, HPL, false, true, LEAN, FULLD>(PR, PO, A, nb, sb, L, ep,
                                                                 want_lp, want_amax);
            const uint8_t *dev = nb + L.assign;
            for (int v = lane; v < n; v += 32)
                A.assign[(size_t)ep * n + v] = dev[v] == 0xFF ? -1 : dev[v];
            double mk = 0.0;
            if (status == FP_EP_OK && A.simulate) {
                __syncwarp();
                SimOut o = sim_episode<RPL, true, SM1, false, FULLD ? MAXD : 0, LEAN>(
                    PR, nb, sb, L, A.strategy, nullptr,
                    (!LEAN && A.trace) ? A.trace + (size_t)ep * A.trace_cap : nullptr,
                    A.trace_cap, nullptr);
                status = o.status;
                mk = o.makespan;
                if (lane == 0 && A.trace_len) A.trace_len[ep] = o.n_events;
            }
            if (lane == 0) {
                if (A.makespan) A.makespan[ep] = mk;
                A.status[ep] = status;
            }
        }
        __syncthreads();
    }
}

template <int MAXD, int HPL>
int launch_rollout_wide(const fp_problem *p, const fp_policy *pol,
                               const fp_rollout_args &a, int64_t *ws_needed, cudaStream_t st) {
    const DevProblem &PR = p->dev;
    const EpLayout L = make_layout(PR.n, PR.W, PR.R, PR.SM, true, 0, true);
    const int64_t smem = L.bytes;
    if (smem > 227 * 1024) {
        set_error("episode scratch exceeds shared memory (too many devices / slots)");
        return FP_ERR_UNSUPPORTED;
    }
    const bool lean = a.mode == FP_MODE_SAMPLE && !a.step_vd && !a.step_lp && !a.step_ent &&
                      !a.step_argmax && !a.step_ncand && !a.trace && !(a.flags & FP_FLAG_TIE_RANDOM);
    const bool full = PR.d == MAXD && pol->dev.h == 32 * HPL;
    auto kern = PR.SM == 1 ? (lean ? (full ? rollout_wide_kernel<MAXD, HPL, true, true, true>
                                           : rollout_wide_kernel<MAXD, HPL, true, true>)
                                   : rollout_wide_kernel<MAXD, HPL, true>)
                           : rollout_wide_kernel<MAXD, HPL, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FP_ERR_CUDA; }
    const int grid = persistent_blocks((const void *)kern, 64, smem, a.B);
    const int64_t need = (int64_t)grid * L.gbytes;
    if (ws_needed) { *ws_needed = need; return FP_OK; }
    if (!a.workspace || a.workspace_bytes < need) {
        set_error("workspace too small for the wide rollout (see fp_rollout_workspace_size)");
        return FP_ERR_INVALID;
    }
    kern<<<grid, 64, smem, st>>>(PR, pol->dev, a, L);
    e = cudaGetLastError();
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FP_ERR_CUDA; }
    return FP_OK;
}

}  // namespace fp
