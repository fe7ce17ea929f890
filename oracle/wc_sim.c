/*
 * ORACLE — test infrastructure only.  Nothing in the product path links or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg load it.
 *
 * Plain-C restatement of the reference work-conserving simulator core,
 * flowplace/_simcore.pyx:39-248 (== flowplace/_simpy.py:35-161), keeping its
 * O(n) rescan-and-start-one loop so it is an independent check of the CUDA
 * core's event-driven formulation (per-resource pending queues, one ordered
 * pass per instant).  Parity pinned against event streams dumped from the
 * reference itself (tests/golden/sim_cases.json, tests/test_oracle.py).
 *
 *   jitter            _simcore.pyx:15-36   (libm log/cos/exp/sqrt, as the reference)
 *   consumer devices  _simcore.pyx:84-97
 *   transfer scan     _simcore.pyx:115-145
 *   exec scan         _simcore.pyx:146-175
 *   task start        _simcore.pyx:177-202
 *   deadlock          _simcore.pyx:204-207
 *   completion batch  _simcore.pyx:209-232
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    double time;
    int32_t v;
    int8_t kind;   /* 0 exec, 1 transfer */
    int8_t etype;  /* 0 beg, 1 end */
    int8_t a;      /* exec device / transfer src */
    int8_t b;      /* transfer dst, -1 for exec */
} oracle_event;

static uint64_t o_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double oracle_jitter_factor(uint64_t seed, int kind, int a, int b, int c, double sigma) {
    uint64_t h = o_mix64(seed ^ 0xD1B54A32D192ED03ULL);
    h = o_mix64(h ^ (uint64_t)(int64_t)(kind + 1));
    h = o_mix64(h ^ (uint64_t)(int64_t)(a + 1));
    h = o_mix64(h ^ (uint64_t)(int64_t)(b + 2));
    h = o_mix64(h ^ (uint64_t)(int64_t)(c + 2));
    const double s53 = ldexp(1.0, -53);
    double u1 = ((double)(h >> 11) + 0.5) * s53;
    h = o_mix64(h);
    double u2 = ((double)(h >> 11) + 0.5) * s53;
    double z = sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
    return exp(sigma * z);
}

typedef struct { double end; int kind, v, a, b; } flight;

/* Returns 0 ok, 1 deadlock (dl_time / blocked filled), 2 event overflow,
 * 3 allocation failure.  ev may be NULL (makespan only). */
int oracle_run_packed(int n, int d,
                      const int32_t *pred_indptr, const int32_t *pred_indices,
                      const int32_t *succ_indptr, const int32_t *succ_indices,
                      const uint8_t *is_entry, const double *flops, const double *obytes,
                      const int32_t *assign, const double *rates, const double *bw,
                      const int32_t *eslots, const int32_t *tslots,
                      const double *tlev, const double *blev,
                      int strategy, double comm_factor, double sigma, int64_t seed,
                      double *makespan, oracle_event *ev, int64_t ev_cap, int64_t *n_ev,
                      double *dl_time, uint8_t *blocked) {
    const size_t nd = (size_t)n * (size_t)d;
    uint8_t *ready = calloc(nd ? nd : 1, 1);
    uint8_t *ex_started = calloc(n ? n : 1, 1);
    uint8_t *tr_started = calloc(nd ? nd : 1, 1);
    int *dev_free = malloc(sizeof(int) * (d ? d : 1));
    int *link_free = malloc(sizeof(int) * (d * d ? d * d : 1));
    int *cons_ptr = malloc(sizeof(int) * (n + 1));
    int *cons_dev = malloc(sizeof(int) * (nd ? nd : 1));
    flight *fl = malloc(sizeof(flight) * (nd + n + 1));
    int rc = 0;
    int64_t ne = 0;
    if (!ready || !ex_started || !tr_started || !dev_free || !link_free || !cons_ptr ||
        !cons_dev || !fl) { rc = 3; goto done; }

    for (int v = 0; v < n; ++v)
        if (is_entry[v]) memset(ready + (size_t)v * d, 1, d);
    for (int k = 0; k < d; ++k) dev_free[k] = eslots[k];
    for (int k = 0; k < d * d; ++k) link_free[k] = tslots[k];

    /* ascending unique devices hosting v's successors */
    cons_ptr[0] = 0;
    for (int v = 0, w = 0; v < n; ++v) {
        uint64_t seen = 0;  /* d <= 64 */
        for (int j = succ_indptr[v]; j < succ_indptr[v + 1]; ++j)
            seen |= 1ULL << assign[succ_indices[j]];
        for (int k = 0; k < d; ++k)
            if (seen >> k & 1ULL) cons_dev[w++] = k;
        cons_ptr[v + 1] = w;
    }

    int left = 0;
    for (int v = 0; v < n; ++v) left += !is_entry[v];
    double now = 0.0;
    int inflight = 0;

    while (left > 0) {
        /* ---- pick: transfers by (v, dst), then execs by v ---- */
        int found = 0, bk = 0, bv = 0, ba = 0, bb = 0;
        double bkey = 0.0;
        for (int v = 0; v < n && !(strategy == 0 && found); ++v) {
            if (cons_ptr[v + 1] == cons_ptr[v]) continue;
            int src = assign[v];
            if (!ready[(size_t)v * d + src]) continue;
            for (int j = cons_ptr[v]; j < cons_ptr[v + 1]; ++j) {
                int dst = cons_dev[j];
                size_t at = (size_t)v * d + dst;
                if (ready[at] || tr_started[at] || link_free[src * d + dst] <= 0) continue;
                double key = strategy == 1 ? tlev[v] : (strategy == 2 ? blev[v] : 0.0);
                if (strategy == 0 || !found || (strategy == 1 && key > bkey) ||
                    (strategy == 2 && key < bkey)) {
                    found = 1; bkey = key; bk = 1; bv = v; ba = src; bb = dst;
                    if (strategy == 0) break;
                }
            }
        }
        if (!(strategy == 0 && found)) {
            for (int v = 0; v < n; ++v) {
                if (is_entry[v] || ex_started[v]) continue;
                int dev = assign[v];
                if (dev_free[dev] <= 0) continue;
                int ok = 1;
                for (int j = pred_indptr[v]; j < pred_indptr[v + 1] && ok; ++j)
                    ok = ready[(size_t)pred_indices[j] * d + dev];
                if (!ok) continue;
                double key = strategy == 1 ? tlev[v] : (strategy == 2 ? blev[v] : 0.0);
                if (strategy == 0 || !found || (strategy == 1 && key > bkey) ||
                    (strategy == 2 && key < bkey)) {
                    found = 1; bkey = key; bk = 0; bv = v; ba = dev; bb = -1;
                    if (strategy == 0) break;
                }
            }
        }

        if (found) {
            double dur;
            if (bk == 0) {
                dur = flops[bv] / rates[ba];
                if (sigma > 0.0) dur *= oracle_jitter_factor((uint64_t)seed, 0, bv, ba, 0, sigma);
                dev_free[ba] -= 1;
                ex_started[bv] = 1;
            } else {
                dur = obytes[bv] * comm_factor / bw[ba * d + bb];
                if (sigma > 0.0) dur *= oracle_jitter_factor((uint64_t)seed, 1, bv, ba, bb, sigma);
                link_free[ba * d + bb] -= 1;
                tr_started[(size_t)bv * d + bb] = 1;
            }
            if (ev) {
                if (ne >= ev_cap) { rc = 2; goto done; }
                ev[ne] = (oracle_event){now, bv, (int8_t)bk, 0, (int8_t)ba, (int8_t)bb};
            }
            ++ne;
            fl[inflight++] = (flight){now + dur, bk, bv, ba, bb};
            continue;
        }

        if (inflight == 0) {
            if (dl_time) *dl_time = now;
            if (blocked)
                for (int v = 0; v < n; ++v)
                    blocked[v] = !is_entry[v] && !ready[(size_t)v * d + assign[v]];
            rc = 1;
            goto done;
        }

        /* ---- advance to the earliest completion; retire every record that
         *      ends exactly then, in start order ---- */
        double tmin = fl[0].end;
        for (int i = 1; i < inflight; ++i)
            if (fl[i].end < tmin) tmin = fl[i].end;
        int keep = 0;
        for (int i = 0; i < inflight; ++i) {
            flight f = fl[i];
            if (f.end != tmin) { fl[keep++] = f; continue; }
            if (f.kind == 0) {
                dev_free[f.a] += 1;
                ready[(size_t)f.v * d + f.a] = 1;
                --left;
            } else {
                link_free[f.a * d + f.b] += 1;
                ready[(size_t)f.v * d + f.b] = 1;
            }
            if (ev) {
                if (ne >= ev_cap) { rc = 2; goto done; }
                ev[ne] = (oracle_event){tmin, f.v, (int8_t)f.kind, 1, (int8_t)f.a, (int8_t)f.b};
            }
            ++ne;
        }
        inflight = keep;
        now = tmin;
    }
    *makespan = now;

done:
    if (n_ev) *n_ev = ne;
    free(ready); free(ex_started); free(tr_started); free(dev_free); free(link_free);
    free(cons_ptr); free(cons_dev); free(fl);
    return rc;
}

/* Makespans of B assignments of one graph (no trace, no jitter): the CPU
 * baseline's simulator leg.  status[b] as oracle_run_packed. */
void oracle_sim_batch(int n, int d,
                      const int32_t *pred_indptr, const int32_t *pred_indices,
                      const int32_t *succ_indptr, const int32_t *succ_indices,
                      const uint8_t *is_entry, const double *flops, const double *obytes,
                      const int32_t *assign_bn, int B, const double *rates, const double *bw,
                      const int32_t *eslots, const int32_t *tslots,
                      const double *tlev, const double *blev,
                      int strategy, double comm_factor, double *makespan, int32_t *status) {
    for (int b = 0; b < B; ++b) {
        double mk = 0.0;
        status[b] = oracle_run_packed(n, d, pred_indptr, pred_indices, succ_indptr, succ_indices,
                                      is_entry, flops, obytes, assign_bn + (size_t)b * n, rates,
                                      bw, eslots, tslots, tlev, blev, strategy, comm_factor, 0.0,
                                      0, &mk, NULL, 0, NULL, NULL, NULL);
        makespan[b] = mk;
    }
}
