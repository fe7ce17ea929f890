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
//   * Durations are the reference's fp64 expressions flops/rate and
//     (bytes*cf)/bw (:183,:189), evaluated once per problem on the host
//     (P.edur / P.tdur), then * jitter factor when a table is given.
// Lane l owns resources l, l+32, ... (RPL per lane): their free-slot counts
// live in registers and their in-flight slots (r*SM + i) are only touched by
// that lane; pending bitsets / counts are shared (atomic pushes).
// Event order in the optional trace is the reference's: starts of an instant
// sorted by the global enumeration key, completions by start sequence.
#pragma once

#include "fp_common.cuh"
#include "fp_problem.cuh"

namespace fp {

__device__ __forceinline__ uint64_t sim_task_key(int krank, int kind, int v, int b) {
    return ((uint64_t)krank << 40) | ((uint64_t)(kind == 0 ? 1 : 0) << 39) |
           ((uint64_t)v << 8) | (uint64_t)(b & 0xff);
}

struct SimOut {
    double makespan;
    int status;
    int n_events;
};

// Pending set of one resource: bit `pos` = the task whose vertex sits at
// position pos of the strategy order.  Compact path: one flat bitset scanned
// from word 0 (n <= ~1k).  Wide path (HIER): three levels -- L0 words, an L1
// word per 32 L0 words, an L2 word per 32 L1 words -- so pushes and pops
// are O(1) words plus an L2 scan of n/32768 words.  Pushes happen only in
// the completion phase (any lane, atomicOr), pops only in the start phase by
// the lane owning the resource, so the two never race.
template <bool HIER>
__device__ __forceinline__ void pend_push(uint32_t *b, const EpLayout &L, int pos) {
    const int w = pos >> 5;
    atomicOr(&b[w], 1u << (pos & 31));
    if constexpr (HIER) {
        atomicOr(&b[L.W + (w >> 5)], 1u << (w & 31));
        atomicOr(&b[L.W + L.W1 + (w >> 10)], 1u << ((w >> 5) & 31));
    }
}

template <bool HIER>
__device__ __forceinline__ int pend_pop_hier(uint32_t *b, const EpLayout &L) {
    uint32_t *b1 = b + L.W, *b2 = b1 + L.W1;
    int w2 = 0;
    uint32_t x2;
    while ((x2 = b2[w2]) == 0u) ++w2;
    const int w1 = (w2 << 5) + __ffs(x2) - 1;
    uint32_t x1 = b1[w1];
    const int w = (w1 << 5) + __ffs(x1) - 1;
    uint32_t x = b[w];
    const int bit = __ffs(x) - 1;
    x &= ~(1u << bit);
    b[w] = x;
    if (x == 0u) {
        x1 &= ~(1u << (w & 31));
        b1[w1] = x1;
        if (x1 == 0u) b2[w2] = x2 & ~(1u << (w1 & 31));
    }
    return (w << 5) + bit;
}

// nb: this episode's n-sized state (shared memory, or its HBM workspace slice
// on the wide path); sb: its small shared-memory scratch.  nb + L.assign must
// hold the assignment (made visible with __syncwarp).  All 32 lanes must call.
// Overlap with the placement chain (OVL): the simulator may run while the
// PLC warp is still placing vertices (in the SEL order).  A task only needs
// the devices of vertices it touches: starting a pending task needs nothing
// new, and retiring (exec or transfer of) v needs the devices of all of v's
// successors (consumer devices, readiness of w on A_w).  So before retiring
// the tasks of an instant the simulator waits until the placement counter
// passes the largest SEL position among their successors (maxsucc[v]), and
// before seeding the initially pending execs until it passes the last of
// them (initwait).  Any vertex that becomes startable is the successor of a
// retired task (or initially pending), so every pending task is placed.
struct SimSync {
    const volatile int *placed;  // vertices placed so far (PLC warp, release)
    const volatile int *abort;   // PLC chain failed: stop waiting
    const int *maxsucc;          // [n] max SEL position over successors, -1 if none
    int initwait;                // max SEL position over the initially pending execs
};

__device__ __forceinline__ bool sim_wait_placed(const SimSync &S, int need) {
    int ok = 1;
    if (need >= 0 && lane_id() == 0) {
        // back off (a PLC step is ~1-3 us): the spin's loads and branches
        // would otherwise take issue slots from the placing warps
        unsigned ns = 64;
        while (*S.placed <= need) {
            if (*S.abort) { ok = 0; break; }
            __nanosleep(ns);
            ns = min(ns * 2u, 512u);
        }
        __threadfence_block();  // acquire: the devices written before the counter
    }
    ok = __shfl_sync(FP_FULL_MASK, ok, 0);
    __syncwarp();
    return ok != 0;
}

// FD > 0: the cluster's device count as a compile-time constant (resources,
// link decompositions and loop bounds fold); SM1 likewise fixes one slot.
// PLAIN: no trace, no jitter table, no blocked-task output (the fused
// sampling rollout) -- those branches compile away.
template <int RPL, bool HIER = false, bool SM1 = false, bool OVL = false, int FD = 0,
          bool PLAIN = false>
__device__ __forceinline__ SimOut sim_episode(const DevProblem &P, uint8_t *nb, uint8_t *sb,
                                              const EpLayout &L, int strategy,
                                              const double *__restrict__ jit,
                                              fp_event *__restrict__ trace, int trace_cap,
                                              uint8_t *__restrict__ blocked,
                                              SimSync sync = SimSync{nullptr, nullptr, nullptr, -1}) {
    const int lane = lane_id();
    const int n = P.n, d = FD ? FD : P.d, R = FD ? FD + FD * FD : P.R, SM = SM1 ? 1 : P.SM,
              BW = L.BW;
    uint32_t *rdy = (uint32_t *)(nb + L.rdy);
    uint32_t *cons = (uint32_t *)(nb + L.cons);
    int *missing = (int *)(nb + L.missing);
    const uint8_t *assign = nb + L.assign;
    uint32_t *bits = (uint32_t *)(nb + L.bits);
    int *cnt = (int *)(sb + L.cnt);
    double *pend = (double *)(sb + L.pend);
    int *pv = (int *)(sb + L.pv);
    int *pseq = (int *)(sb + L.pseq);
    uint64_t *skey = (uint64_t *)(sb + L.skey);
    int *sidx = (int *)(sb + L.sidx);
    int *elist = (int *)(sb + L.elist);
    int *ctr = (int *)(sb + L.ctr);
    const uint32_t dmask = d >= 32 ? 0xffffffffu : ((1u << d) - 1u);
    const int *__restrict__ rpos = P.rank_pos + strategy * n;
    const int *__restrict__ rvert = P.rank_vert + strategy * n;
    const int *__restrict__ krk = P.krank + strategy * n;
    const int *__restrict__ sp = P.succ_ptr;
    const int *__restrict__ si = P.succ_idx;
    const uint8_t *__restrict__ ent = P.is_entry;
    const double *__restrict__ edur = P.edur;
    const double *__restrict__ tdur = P.tdur;

    // ---- init (_simcore.pyx:71-105); cold loops kept rolled (code size) ----
#pragma unroll 1
    for (int v = lane; v < n; v += 32) {
        const bool e = ent[v];
        rdy[v] = e ? dmask : 0u;
        if constexpr (!OVL) {  // consumer devices (_simcore.pyx:84-97), all placed
            uint32_t c = 0;
#pragma unroll 1
            for (int j = sp[v]; j < sp[v + 1]; ++j) c |= 1u << assign[si[j]];
            cons[v] = c;
        }
        int miss = 0;
#pragma unroll 1
        for (int j = P.pred_ptr[v]; j < P.pred_ptr[v + 1]; ++j) miss += !ent[P.pred_idx[j]];
        missing[v] = miss;
    }
#pragma unroll 1
    for (int i = lane; i < R * BW; i += 32) bits[i] = 0u;
    // SM1: every resource has at most one slot (the reference's default
    // cluster), so each resource's in-flight task lives in its owning lane's
    // registers (ipv / iend) instead of the shared-memory pool; the pool is
    // only mirrored for the trace sort.
    int fr[RPL];
    int ipv[SM1 ? RPL : 1];
    double iend[SM1 ? RPL : 1];
    int rsrc[RPL], rdst[RPL];  // link r >= d: (src, dst) = divmod(r - d, d), once per episode
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
        const int r = lane + 32 * q;
        rsrc[q] = r < d ? r : (r - d) / d;
        rdst[q] = r < d ? r : (r - d) - rsrc[q] * d;
    }
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
        const int r = lane + 32 * q;
        fr[q] = r < R ? P.slots[r] : 0;
        if constexpr (SM1) { ipv[q] = -1; iend[q] = 0.0; }
        if (r < R) {
            cnt[r] = 0;
            if constexpr (!SM1)
                for (int i = 0; i < SM; ++i) pv[r * SM + i] = -1;
        }
    }
    __syncwarp();
    if constexpr (OVL)
        if (!sim_wait_placed(sync, sync.initwait)) return SimOut{0.0, FP_EP_BAD_ACTION, 0};
    for (int v = lane; v < n; v += 32)
        if (!ent[v] && missing[v] == 0) {
            pend_push<HIER>(bits + assign[v] * BW, L, rpos[v]);
            atomicAdd(&cnt[assign[v]], 1);
        }
    __syncwarp();

    SimOut out{0.0, FP_EP_OK, 0};
    FP_PHASE_DECL;
    FP_PHASE_BEGIN(pq_);
    int remaining = P.n_nonentry;
    double t = 0.0;
    int seq = 0;
    const bool tracing = !PLAIN && trace != nullptr;
    if constexpr (PLAIN) { jit = nullptr; blocked = nullptr; }

    while (remaining > 0) {
        // ---------------- start phase: each lane serves its resources --------
        if (tracing && lane == 0) ctr[0] = 0;
        __syncwarp();
        int live = 0;
        double lmin = __longlong_as_double(0x7ff0000000000000LL);  // +inf
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
            const int r = lane + 32 * q;
            if (r >= R) continue;
            if (fr[q] > 0) {
                int c = cnt[r];
                if (c > 0) {
                    uint32_t *wb = bits + r * BW;
                    int w = 0;
                    int slot = r * SM;
                    int f = fr[q];
                    while (f > 0 && c > 0) {
                        int pos;
                        if constexpr (HIER) {
                            pos = pend_pop_hier<HIER>(wb, L);
                        } else {
                            uint32_t word = wb[w];
                            while (word == 0u) word = wb[++w];
                            const int b = __ffs(word) - 1;
                            wb[w] = word & ~(1u << b);
                            pos = (w << 5) + b;
                        }
                        const int v = rvert[pos];
                        double dur;
                        int kind, tb;
                        if (r < d) {
                            kind = 0; tb = -1;
                            dur = edur[v * d + r];
                            if (jit) dur = __dmul_rn(dur, jit[v * d + r]);
                        } else {
                            const int ta = rsrc[q];
                            kind = 1; tb = rdst[q];
                            dur = tdur[(v * d + ta) * d + tb];
                            if (jit) dur = __dmul_rn(dur, jit[n * d + (v * d + ta) * d + tb]);
                        }
                        const double end = __dadd_rn(t, dur);
                        if constexpr (SM1) {
                            ipv[q] = v;
                            iend[q] = end;
                            if (tracing) { pend[slot] = end; pv[slot] = v; }
                        } else {
                            while (pv[slot] >= 0) ++slot;
                            pend[slot] = end;
                            pv[slot] = v;
                        }
                        if (tracing) {
                            const int k = atomicAdd(&ctr[0], 1);
                            skey[k] = sim_task_key(krk[v], kind, v, tb);
                            sidx[k] = slot;
                        }
                        --f;
                        --c;
                    }
                    fr[q] = f;
                    cnt[r] = c;
                }
            }
            // in-flight tasks of this resource (the wait phase's min)
            if constexpr (SM1) {
                if (ipv[q] >= 0) { lmin = fmin(lmin, iend[q]); ++live; }
            } else {
                for (int i = 0; i < SM; ++i) {
                    const int s = r * SM + i;
                    if (pv[s] >= 0) { lmin = fmin(lmin, pend[s]); ++live; }
                }
            }
        }
        __syncwarp();
        FP_PHASE_END(pq_, 21);
        if (tracing) {
            const int k = ctr[0];
            for (int i = lane; i < k; i += 32) {
                const uint64_t key = skey[i];
                int rank = 0;
                for (int j = 0; j < k; ++j) rank += skey[j] < key;
                const int slot = sidx[i];
                pseq[slot] = seq + rank;
                const int pos = out.n_events + rank;
                if (pos < trace_cap) {
                    const int r = slot / SM;
                    fp_event e;
                    e.time = t; e.v = pv[slot]; e.etype = 0;
                    if (r < d) { e.kind = 0; e.a = (int8_t)r; e.b = -1; }
                    else { e.kind = 1; e.a = (int8_t)((r - d) / d); e.b = (int8_t)((r - d) % d); }
                    trace[pos] = e;
                }
            }
            seq += k;
            out.n_events += k;
            __syncwarp();
        }

        // ---------------- wait phase: earliest completion -----------------
        if (__reduce_add_sync(FP_FULL_MASK, live) == 0) {
            out.status = FP_EP_DEADLOCK;
            out.makespan = t;
            if (blocked)
                for (int v = lane; v < n; v += 32)
                    blocked[v] = !ent[v] && !((rdy[v] >> assign[v]) & 1u);
            return out;
        }
        const double tmin = warp_min_redux(lmin);
        FP_PHASE_END(pq_, 23);
        if (tracing && lane == 0) ctr[1] = 0;
        __syncwarp();
        if constexpr (OVL) {  // the retiring tasks' successors must be placed
            int need = -1;
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
                const int r = lane + 32 * q;
                if (r >= R) continue;
                for (int i = 0; i < (SM1 ? 1 : SM); ++i) {
                    const int v = SM1 ? ipv[q] : pv[r * SM + i];
                    const double e = SM1 ? iend[q] : pend[r * SM + i];
                    if (v >= 0 && e == tmin) need = max(need, sync.maxsucc[v]);
                }
            }
            need = __reduce_max_sync(FP_FULL_MASK, need);
            if (!sim_wait_placed(sync, need)) return SimOut{0.0, FP_EP_BAD_ACTION, 0};
            FP_PHASE_END(pq_, 22);
        }
        int done_exec = 0;
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
            const int r = lane + 32 * q;
            if (r >= R) continue;
            for (int i = 0; i < (SM1 ? 1 : SM); ++i) {
                const int s = r * SM + i;
                int v;
                if constexpr (SM1) {
                    v = ipv[q];
                    if (v < 0 || iend[q] != tmin) continue;
                    ipv[q] = -1;
                } else {
                    v = pv[s];
                    if (v < 0 || pend[s] != tmin) continue;
                    pv[s] = -1;
                }
                fr[q] += 1;
                if (tracing) {
                    const int k = atomicAdd(&ctr[1], 1);
                    elist[k] = s;
                    sidx[k] = v;  // start list is consumed; reuse for the vertex
                }
                int dev;
                if (r < d) {
                    dev = r;
                    atomicOr(&rdy[v], 1u << r);
                    ++done_exec;
                    // consumer devices of v (_simcore.pyx:84-97); overlapped: only
                    // known now that every successor is placed
                    uint32_t m = 0u;
                    if constexpr (OVL) {
                        const int j1 = sp[v + 1];
#pragma unroll 1
                        for (int j = sp[v]; j < j1; j += 2) {  // two successors per trip
                            const int wa = si[j], wb = j + 1 < j1 ? si[j + 1] : wa;
                            m |= (1u << assign[wa]) | (1u << assign[wb]);
                        }
                    } else {
                        m = cons[v];
                    }
                    m &= ~(1u << r);
                    const int pos = rpos[v];
                    while (m) {
                        const int dst = __ffs(m) - 1;
                        m &= m - 1;
                        const int rr = d + r * d + dst;
                        pend_push<HIER>(bits + rr * BW, L, pos);
                        atomicAdd(&cnt[rr], 1);
                    }
                } else {
                    dev = rdst[q];
                    atomicOr(&rdy[v], 1u << dev);
                }
#pragma unroll 1
                for (int j = sp[v], j1 = sp[v + 1]; j < j1; j += 2) {
                    // two successors per trip: index and device loads in flight
                    // together, processed in successor order
                    const bool two = j + 1 < j1;
                    const int wa = si[j], wb = two ? si[j + 1] : wa;
                    const bool ha = assign[wa] == dev, hb = two && assign[wb] == dev;
                    if (ha && atomicSub(&missing[wa], 1) == 1) {
                        pend_push<HIER>(bits + dev * BW, L, rpos[wa]);
                        atomicAdd(&cnt[dev], 1);
                    }
                    if (hb && atomicSub(&missing[wb], 1) == 1) {
                        pend_push<HIER>(bits + dev * BW, L, rpos[wb]);
                        atomicAdd(&cnt[dev], 1);
                    }
                }
            }
        }
        remaining -= __reduce_add_sync(FP_FULL_MASK, done_exec);
        __syncwarp();
        FP_PHASE_END(pq_, 24);
        if (tracing) {
            const int k = ctr[1];
            for (int i = lane; i < k; i += 32) {
                const int slot = elist[i];
                const int sq = pseq[slot];
                int rank = 0;
                for (int j = 0; j < k; ++j) rank += pseq[elist[j]] < sq;
                const int pos = out.n_events + rank;
                if (pos < trace_cap) {
                    const int r = slot / SM;
                    fp_event e;
                    e.time = tmin; e.etype = 1; e.v = sidx[i];
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
    FP_PHASE_FLUSH(0);
    return out;
}

}  // namespace fp
