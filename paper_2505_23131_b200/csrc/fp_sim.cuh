// Event-driven work-conserving simulator, one warp per episode.
//
// Semantics: flowplace/_simcore.pyx:39-248 (== _simpy.py:35-161), re-derived
// for a batched GPU core:
//   * The reference restarts an O(n*d) scan after every task start
//     (_simcore.pyx:107-202).  Starting a task only consumes a slot, so the
//     sequence of starts at one instant equals ONE pass over the startable
//     tasks in enumeration order (fifo: transfers by (v, dst), then execs by
//     v; depth/breadth: stable by level key).  Tasks on different resources
//     never compete, so each resource starts its first `free` pending tasks
//     in that order: pending tasks live in per-resource bitsets indexed by
//     the vertex's position in the strategy order, popped with find-first-set.
//   * Pending sets change only at completions: an exec of v on a makes the
//     transfers (v, a->dst) for every consumer device dst != a pending
//     (_simcore.pyx:115-126); readiness of (v, dev) decrements missing[w] of
//     successors w placed on dev, and missing[w] == 0 makes exec w pending
//     (_simcore.pyx:147-159).
//   * Completions: every in-flight record whose end == tmin exactly, in start
//     order (_simcore.pyx:209-232); the loop stops when the last exec retires.
//   * Durations are the reference's fp64 expressions with explicit _rn
//     intrinsics (no FMA contraction): flops/rate, (bytes*cf)/bw (:183,:189),
//     then * jitter factor when a table is given.
// Event order in the optional trace is the reference's: starts of an instant
// sorted by the global enumeration key, completions by start sequence.
#pragma once

#include "fp_common.cuh"
#include "fp_problem.cuh"

namespace fp {

struct SimSmem {
    uint32_t *rdy;      // [n] device mask where v's output is materialised
    int *missing;       // [n] preds not ready on assign[v]
    uint32_t *cons;     // [n] devices hosting v's successors
    uint8_t *assign;    // [n]
    uint32_t *bits;     // [R][W] pending tasks per resource (strategy-order bit index)
    int *cnt;           // [R] pending count
    int *freec;         // [R] free slots
    double *pend;       // [P] in-flight end time
    uint64_t *skey;     // [P] start-sort keys
    int *pv;            // [P] in-flight vertex (-1 empty)
    int *pseq;          // [P] start sequence number
    int *sidx;          // [P] started pool entries / retiring vertices (this instant)
    int *elist;         // [P] retiring pool entries
    int *ctr;           // [4] counters
};

__device__ __forceinline__ SimSmem sim_carve(uint8_t *base, const DevProblem &P) {
    SimSmem s;
    const int n = P.n;
    uint8_t *p = base;
    s.rdy = (uint32_t *)p; p += 4 * n;
    s.missing = (int *)p; p += 4 * n;
    s.cons = (uint32_t *)p; p += 4 * n;
    s.assign = p; p += (n + 15) / 16 * 16;
    s.bits = (uint32_t *)p; p += 4 * P.R * P.W;
    s.cnt = (int *)p; p += 4 * P.R;
    s.freec = (int *)p; p += 4 * P.R;
    p = (uint8_t *)(((uintptr_t)p + 7) & ~(uintptr_t)7);
    s.pend = (double *)p; p += 8 * P.P;
    s.skey = (uint64_t *)p; p += 8 * P.P;
    s.pv = (int *)p; p += 4 * P.P;
    s.pseq = (int *)p; p += 4 * P.P;
    s.sidx = (int *)p; p += 4 * P.P;
    s.elist = (int *)p; p += 4 * P.P;
    s.ctr = (int *)p;
    return s;
}

struct SimOut {
    double makespan;
    int status;
    int n_events;
};

__device__ __forceinline__ void sim_push(const SimSmem &S, const DevProblem &P, int r, int pos) {
    atomicOr(&S.bits[r * P.W + (pos >> 5)], 1u << (pos & 31));
    atomicAdd(&S.cnt[r], 1);
}

// Global enumeration key of a started task (see header comment).
__device__ __forceinline__ uint64_t sim_task_key(int krank, int kind, int v, int b) {
    return ((uint64_t)krank << 40) | ((uint64_t)(kind == 0 ? 1 : 0) << 39) |
           ((uint64_t)v << 8) | (uint64_t)(b & 0xff);
}

// Runs one episode.  S.assign must hold the assignment (written by the caller
// and made visible with __syncwarp).  All 32 lanes must call.
static __device__ SimOut sim_episode(const DevProblem &P, const SimSmem &S, int strategy,
                              const double *__restrict__ jit, fp_event *__restrict__ trace,
                              int trace_cap, uint8_t *__restrict__ blocked) {
    const int lane = lane_id();
    const int n = P.n, d = P.d, W = P.W, R = P.R;
    const uint32_t dmask = d >= 32 ? 0xffffffffu : ((1u << d) - 1u);
    const int *rpos = P.rank_pos + strategy * n;
    const int *rvert = P.rank_vert + strategy * n;
    const int *krk = P.krank + strategy * n;

    // ---- init (_simcore.pyx:71-105) ----
    for (int v = lane; v < n; v += 32) {
        const bool entry = P.is_entry[v];
        S.rdy[v] = entry ? dmask : 0u;
        uint32_t c = 0;
        for (int j = P.succ_ptr[v]; j < P.succ_ptr[v + 1]; ++j) c |= 1u << S.assign[P.succ_idx[j]];
        S.cons[v] = c;
        int miss = 0;
        for (int j = P.pred_ptr[v]; j < P.pred_ptr[v + 1]; ++j) miss += !P.is_entry[P.pred_idx[j]];
        S.missing[v] = miss;
    }
    for (int i = lane; i < R * W; i += 32) S.bits[i] = 0u;
    for (int r = lane; r < R; r += 32) { S.cnt[r] = 0; S.freec[r] = P.slots[r]; }
    for (int i = lane; i < P.P; i += 32) S.pv[i] = -1;
    __syncwarp();
    for (int v = lane; v < n; v += 32)
        if (!P.is_entry[v] && S.missing[v] == 0) sim_push(S, P, S.assign[v], rpos[v]);
    __syncwarp();

    SimOut out{0.0, FP_EP_OK, 0};
    int remaining = P.n_nonentry;
    double t = 0.0;
    int seq = 0;
    const bool tracing = trace != nullptr;

    while (remaining > 0) {
        // ---------------- start phase: each lane serves its resources ----------
        int nstart = 0;  // per-lane count (for deadlock detection)
        if (tracing && lane == 0) S.ctr[0] = 0;
        __syncwarp();
        for (int r = lane; r < R; r += 32) {
            int fr = S.freec[r];
            int c = S.cnt[r];
            if (fr <= 0 || c <= 0) continue;
            uint32_t *wb = S.bits + r * W;
            int w = 0;
            const int po = P.pool_off[r], pe = P.pool_off[r + 1];
            int slot = po;
            while (fr > 0 && c > 0) {
                uint32_t word = wb[w];
                while (word == 0u) word = wb[++w];
                const int b = __ffs(word) - 1;
                wb[w] = word & ~(1u << b);
                const int v = rvert[(w << 5) + b];
                double dur;
                int ta, tb, kind;
                if (r < d) {
                    kind = 0; ta = r; tb = -1;
                    dur = __ddiv_rn(P.flops[v], P.rates[r]);
                    if (jit) dur = __dmul_rn(dur, jit[v * d + r]);
                } else {
                    kind = 1; ta = (r - d) / d; tb = (r - d) % d;
                    dur = __ddiv_rn(__dmul_rn(P.obytes[v], P.comm_factor), P.bw[ta * d + tb]);
                    if (jit) dur = __dmul_rn(dur, jit[n * d + (v * d + ta) * d + tb]);
                }
                while (S.pv[slot] >= 0) ++slot;
                S.pend[slot] = __dadd_rn(t, dur);
                S.pv[slot] = v;
                if (tracing) {
                    const int k = atomicAdd(&S.ctr[0], 1);
                    S.skey[k] = sim_task_key(krk[v], kind, v, tb);
                    S.sidx[k] = slot;
                }
                --fr; --c; ++nstart;
                (void)pe; (void)ta;
            }
            S.freec[r] = fr;
            S.cnt[r] = c;
        }
        __syncwarp();
        if (tracing) {
            // order this instant's starts by the global enumeration key
            const int k = S.ctr[0];
            for (int i = lane; i < k; i += 32) {
                const uint64_t key = S.skey[i];
                int rank = 0;
                for (int j = 0; j < k; ++j) rank += S.skey[j] < key;
                const int slot = S.sidx[i];
                S.pseq[slot] = seq + rank;
                const int pos = out.n_events + rank;
                if (pos < trace_cap) {
                    // recover (kind, a, b) from the slot's resource
                    int r = 0;
                    while (P.pool_off[r + 1] <= slot) ++r;
                    fp_event e;
                    e.time = t; e.v = S.pv[slot]; e.etype = 0;
                    if (r < d) { e.kind = 0; e.a = (int8_t)r; e.b = -1; }
                    else { e.kind = 1; e.a = (int8_t)((r - d) / d); e.b = (int8_t)((r - d) % d); }
                    trace[pos] = e;
                }
            }
            seq += k;
            out.n_events += k;
            __syncwarp();
        }

        // ---------------- wait phase: earliest completion ----------------------
        double lmin = __longlong_as_double(0x7ff0000000000000LL);  // +inf
        int live = 0;
        for (int r = lane; r < R; r += 32)
            for (int s = P.pool_off[r]; s < P.pool_off[r + 1]; ++s)
                if (S.pv[s] >= 0) { lmin = fmin(lmin, S.pend[s]); ++live; }
        live = warp_sum(live);
        if (live == 0) {
            out.status = FP_EP_DEADLOCK;
            out.makespan = t;
            if (blocked)
                for (int v = lane; v < n; v += 32)
                    blocked[v] = !P.is_entry[v] && !((S.rdy[v] >> S.assign[v]) & 1u);
            return out;
        }
        const double tmin = warp_min(lmin);
        if (tracing && lane == 0) S.ctr[1] = 0;
        __syncwarp();
        int done_exec = 0;
        for (int r = lane; r < R; r += 32) {
            for (int s = P.pool_off[r]; s < P.pool_off[r + 1]; ++s) {
                const int v = S.pv[s];
                if (v < 0 || S.pend[s] != tmin) continue;
                S.pv[s] = -1;
                S.freec[r] += 1;
                if (tracing) {
                    const int k = atomicAdd(&S.ctr[1], 1);
                    S.elist[k] = s;
                    S.sidx[k] = v;  // start list is consumed; reuse for the vertex
                }
                int dev;
                if (r < d) {
                    dev = r;
                    atomicOr(&S.rdy[v], 1u << r);
                    ++done_exec;
                    uint32_t m = S.cons[v] & ~(1u << r);
                    const int pos = rpos[v];
                    while (m) {
                        const int dst = __ffs(m) - 1;
                        m &= m - 1;
                        sim_push(S, P, d + r * d + dst, pos);
                    }
                } else {
                    dev = (r - d) % d;
                    atomicOr(&S.rdy[v], 1u << dev);
                }
                for (int j = P.succ_ptr[v]; j < P.succ_ptr[v + 1]; ++j) {
                    const int w = P.succ_idx[j];
                    if (S.assign[w] == dev && atomicSub(&S.missing[w], 1) == 1)
                        sim_push(S, P, dev, rpos[w]);
                }
            }
        }
        remaining -= warp_sum(done_exec);
        __syncwarp();
        if (tracing) {
            const int k = S.ctr[1];
            for (int i = lane; i < k; i += 32) {
                const int slot = S.elist[i];
                const int sq = S.pseq[slot];
                int rank = 0;
                for (int j = 0; j < k; ++j) rank += S.pseq[S.elist[j]] < sq;
                const int pos = out.n_events + rank;
                if (pos < trace_cap) {
                    int r = 0;
                    while (P.pool_off[r + 1] <= slot) ++r;
                    fp_event e;
                    e.time = tmin; e.etype = 1;
                    e.v = S.sidx[i];
                    if (r < d) { e.kind = 0; e.a = (int8_t)r; e.b = -1; }
                    else { e.kind = 1; e.a = (int8_t)((r - d) / d); e.b = (int8_t)((r - d) % d); }
                    trace[pos] = e;
                }
            }
            out.n_events += k;
            __syncwarp();
        }
        t = tmin;
    }
    out.makespan = t;
    if (tracing && out.n_events > trace_cap) out.status = FP_EP_TRACE_OVERFLOW;
    return out;
}

}  // namespace fp
