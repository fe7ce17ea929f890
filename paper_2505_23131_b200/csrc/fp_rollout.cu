// Batched SEL/PLC episodes fused with the WC simulator: one warp per episode,
// episode state resident in shared memory, several episodes per CTA.
//
// Per step (flowplace/policy.py:352-399), all warp-synchronous:
//  SEL  candidate bitset -> compacted ascending list; masked softmax over the
//       static logits s[v] (per_episode mode: SURVEY §0 fact 1); decision by
//       mode (Philox epsilon-mixture sample / greedy / forced / CP teacher);
//       mixture log-prob + entropy (policy.py:301-322).
//  PLC  device features for the chosen vertex (lane = device; policy.py:226-247
//       over timeline.py:30-45), column standardization with the reference's
//       sequential fp64 sums (policy.py:101-105), pre-activations
//       A[v] + S_d + xn_d @ M + c (lane = hidden column; fact 3), leaky,
//       head2, softmax over devices, decision, log-prob, entropy.
//  commit timeline (timeline.py:47-58) with _rn intrinsics (bit-exact fp64),
//       S_d += G[v], candidate update (policy.py:384-389).
//  REINFORCE rows (optional): d log-prob / d entropy w.r.t. the SEL logits
//       (accumulated per vertex in smem) and the PLC pre-activations
//       (per-vertex A rows, running per-device sums R_d for the G rows, and
//       the M / w2 / b2 terms), written for the episode-reduction kernel.
// After the last step the same warp runs sim_episode() on the assignment
// held in shared memory (fp_sim.cuh): no round trip through HBM.
#include <string>

#include "fp_common.cuh"
#include "fp_policy.cuh"
#include "fp_sim.cuh"

namespace fp {

__device__ __forceinline__ double lk(double x, double s) { return x > 0.0 ? x : s * x; }
__device__ __forceinline__ double lkd(double x, double s) { return x > 0.0 ? 1.0 : s; }

struct RollSmem {
    uint32_t *cand;  // [W]
    int *npl;        // [n] predecessors not yet placed
    double *tstart, *tend;  // [n] timeline
    int *clist;      // [n] compacted candidates
    double *ce, *cc; // [n] exp / cumulative per candidate index
    double *xd, *xn; // [32*5]
    double *dsl, *dse;  // [n] SEL gradient accumulators (lp / entropy parts)
};

__host__ __device__ inline int64_t roll_smem_bytes(int n, int W) {
    int64_t b = 4LL * W;
    b = (b + 7) / 8 * 8;
    b += 4LL * n;
    b = (b + 7) / 8 * 8;
    b += 8LL * n * 2 + 4LL * n;
    b = (b + 7) / 8 * 8;
    b += 8LL * n * 2 + 8LL * 32 * 5 * 2 + 8LL * n * 2;
    return (b + 15) / 16 * 16;
}

__device__ __forceinline__ RollSmem roll_carve(uint8_t *p, int n, int W) {
    RollSmem r;
    auto al = [](uint8_t *q) { return (uint8_t *)(((uintptr_t)q + 7) & ~(uintptr_t)7); };
    r.cand = (uint32_t *)p; p = al(p + 4 * W);
    r.npl = (int *)p; p = al(p + 4 * n);
    r.tstart = (double *)p; p += 8 * n;
    r.tend = (double *)p; p += 8 * n;
    r.clist = (int *)p; p = al(p + 4 * n);
    r.ce = (double *)p; p += 8 * n;
    r.cc = (double *)p; p += 8 * n;
    r.xd = (double *)p; p += 8 * 32 * 5;
    r.xn = (double *)p; p += 8 * 32 * 5;
    r.dsl = (double *)p; p += 8 * n;
    r.dse = (double *)p;
    return r;
}

// (value, index) reductions: first maximum / first minimum across lanes
__device__ __forceinline__ void warp_argmax_first(double &v, int &i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(FP_FULL_MASK, v, o);
        const int oi = __shfl_xor_sync(FP_FULL_MASK, i, o);
        if (ov > v || (ov == v && oi < i)) { v = ov; i = oi; }
    }
}
__device__ __forceinline__ void warp_argmin_first(double &v, int &i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(FP_FULL_MASK, v, o);
        const int oi = __shfl_xor_sync(FP_FULL_MASK, i, o);
        if (ov < v || (ov == v && oi < i)) { v = ov; i = oi; }
    }
}

__host__ __device__ inline int64_t grad_ep_stride(int n, int h, int d) {
    return ((2LL * n + 12LL * h + 2 + 2LL * d * h) + 3) / 4 * 4;
}

template <int MAXD, int HPL, bool GRAD, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1)
rollout_kernel(DevProblem PR, DevPolicy PO, fp_rollout_args A, int64_t per_ep, int64_t roll_bytes) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = lane_id();
    const int warp = threadIdx.x >> 5;
    const int ep = blockIdx.x * WARPS + warp;
    if (ep >= A.B) return;
    const int n = PR.n, D = PR.d, W = PR.W, h = PO.h;
    uint8_t *base = smem + (size_t)warp * per_ep;
    RollSmem R = roll_carve(base, n, W);
    SimSmem S = sim_carve(base + roll_bytes, PR);
    uint8_t *dev = S.assign;
    const double eps = A.epsilon, ome = 1.0 - eps, slope = PO.slope;
    const uint32_t k0 = (uint32_t)A.seed, k1 = (uint32_t)(A.seed >> 32);
    const uint32_t ctr_ep = A.episode_base + (uint32_t)ep;
    const double *__restrict__ slog = PO.s;
    const double *__restrict__ Atab = PO.A;
    const double *__restrict__ Gtab = PO.G;
    const double *w2p = PO.W(PR_PLC_H2_W);
    const double b2p = PO.W(PR_PLC_H2_B)[0];
    const bool forced = A.mode == FP_MODE_FORCED, teacher = A.mode == FP_MODE_TEACHER,
               greedy = A.mode == FP_MODE_GREEDY;
    const int32_t *frow = forced ? A.forced + (size_t)ep * n * 2 : nullptr;

    // ---- init ----
    for (int w = lane; w < W; w += 32) R.cand[w] = 0u;
    __syncwarp();
    for (int v = lane; v < n; v += 32) {
        const int np = PR.pred_ptr[v + 1] - PR.pred_ptr[v];
        R.npl[v] = np;
        R.tstart[v] = 0.0;
        R.tend[v] = 0.0;
        dev[v] = 0xFF;
        if constexpr (GRAD) { R.dsl[v] = 0.0; R.dse[v] = 0.0; }
        if (np == 0) atomicOr(&R.cand[v >> 5], 1u << (v & 31));
    }
    double avail = 0.0, aflops = 0.0;  // lane d < D
    double Mr[5][HPL], cr[HPL], w2r[HPL];
    double Sd[MAXD][HPL];
    double Rl[GRAD ? MAXD : 1][HPL], Re[GRAD ? MAXD : 1][HPL];
    double dMl[GRAD ? 5 : 1][HPL], dMe[GRAD ? 5 : 1][HPL], dwl[HPL], dwe[HPL];
    double db2l = 0.0, db2e = 0.0;
#pragma unroll
    for (int t = 0; t < HPL; ++t) {
        const int j = lane + 32 * t;
        const bool ok = j < h;
#pragma unroll
        for (int c = 0; c < 5; ++c) Mr[c][t] = ok ? PO.M[c * h + j] : 0.0;
        cr[t] = ok ? PO.c[j] : 0.0;
        w2r[t] = ok ? w2p[j] : 0.0;
        dwl[t] = dwe[t] = 0.0;
#pragma unroll
        for (int d = 0; d < MAXD; ++d) Sd[d][t] = 0.0;
        if constexpr (GRAD) {
#pragma unroll
            for (int d = 0; d < MAXD; ++d) Rl[d][t] = Re[d][t] = 0.0;
#pragma unroll
            for (int c = 0; c < 5; ++c) dMl[c][t] = dMe[c][t] = 0.0;
        }
    }
    int status = FP_EP_OK;
    __syncwarp();

    for (int step = 0; step < n; ++step) {
        // ================= SEL =================
        const uint32_t cw = lane < W ? R.cand[lane] : 0u;
        const int pc = __popc(cw);
        const int incl = warp_inclusive_scan(pc);
        const int k = __shfl_sync(FP_FULL_MASK, incl, 31);
        {
            int o = incl - pc;
            uint32_t m = cw;
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                R.clist[o++] = lane * 32 + b;
            }
        }
        __syncwarp();
        if (k == 0) { status = FP_EP_DEADLOCK; break; }  // cyclic graph
        double mx = -INFINITY;
        for (int i = lane; i < k; i += 32) mx = fmax(mx, slog[R.clist[i]]);
        mx = warp_max(mx);
        double carry = 0.0;
        for (int b0 = 0; b0 < k; b0 += 32) {
            const int i = b0 + lane;
            const double e = i < k ? exp(slog[R.clist[i]] - mx) : 0.0;
            const double cum = warp_inclusive_scan(e) + carry;
            if (i < k) { R.ce[i] = e; R.cc[i] = cum; }
            carry = __shfl_sync(FP_FULL_MASK, cum, 31);
        }
        const double tot = carry;
        __syncwarp();
        // greedy argmax of p (first maximum)
        double bp = -1.0;
        int bi = 0x7fffffff;
        for (int i = lane; i < k; i += 32) {
            const double p = R.ce[i] / tot;
            if (p > bp) { bp = p; bi = i; }
        }
        warp_argmax_first(bp, bi);
        const int amax_sel = bi;
        int idx = -1;
        if (forced) {
            const int fv = frow[2 * step];
            for (int b0 = 0; b0 < k && idx < 0; b0 += 32) {
                const int i = b0 + lane;
                const unsigned hit = __ballot_sync(FP_FULL_MASK, i < k && R.clist[i] == fv);
                if (hit) idx = b0 + __ffs(hit) - 1;
            }
            if (idx < 0) { status = FP_EP_BAD_ACTION; break; }
        } else if (teacher) {
            double bt = -INFINITY;
            for (int i = lane; i < k; i += 32) bt = fmax(bt, PR.tlev[R.clist[i]]);
            bt = warp_max(bt);
            for (int b0 = 0; b0 < k && idx < 0; b0 += 32) {
                const int i = b0 + lane;
                const unsigned hit = __ballot_sync(FP_FULL_MASK, i < k && PR.tlev[R.clist[i]] == bt);
                if (hit) idx = b0 + __ffs(hit) - 1;
            }
        } else if (greedy) {
            idx = amax_sel;
        } else {
            double u1, u2;
            uniform2(philox4x32_10(U4{ctr_ep, (uint32_t)step, 0u, 0u}, k0, k1), u1, u2);
            if (u1 < eps) {
                idx = min((int)(u2 * (double)k), k - 1);
            } else {
                const double target = u2 * tot;
                for (int b0 = 0; b0 < k && idx < 0; b0 += 32) {
                    const int i = b0 + lane;
                    const unsigned hit = __ballot_sync(FP_FULL_MASK, i < k && R.cc[i] > target);
                    if (hit) idx = b0 + __ffs(hit) - 1;
                }
                if (idx < 0) idx = k - 1;
            }
        }
        // mixture log-prob / entropy (+ gradients w.r.t. the logits)
        const double ek = eps / (double)k;
        double entp = 0.0, lp_sel = 0.0, pidx = 0.0, midx = 0.0, qp = 0.0;
        for (int i = lane; i < k; i += 32) {
            const double p = R.ce[i] / tot;
            const double mix = __dadd_rn(__dmul_rn(p, ome), ek);
            const double lm = log(__dadd_rn(mix, 1e-30));
            entp += mix * lm;
            if (i == idx) { lp_sel = lm; pidx = p; midx = mix; }
            if constexpr (GRAD) qp += -ome * (lm + mix / __dadd_rn(mix, 1e-30)) * p;
        }
        const double ent_sel = -warp_sum(entp);
        lp_sel = warp_sum(lp_sel);  // exactly one lane is non-zero
        const int v = R.clist[idx];
        if constexpr (GRAD) {
            pidx = warp_sum(pidx);
            midx = warp_sum(midx);
            qp = warp_sum(qp);
            const double c1 = ome * pidx / __dadd_rn(midx, 1e-30);
            for (int i = lane; i < k; i += 32) {
                const double p = R.ce[i] / tot;
                const double mix = __dadd_rn(__dmul_rn(p, ome), ek);
                const double lm = log(__dadd_rn(mix, 1e-30));
                const double q = -ome * (lm + mix / __dadd_rn(mix, 1e-30));
                const int u = R.clist[i];
                R.dsl[u] += c1 * ((i == idx ? 1.0 : 0.0) - p);
                R.dse[u] += p * (q - qp);
            }
        }

        // ================= PLC =================
        double Av[HPL], Gv[HPL];
#pragma unroll
        for (int t = 0; t < HPL; ++t) {
            const int j = lane + 32 * t;
            Av[t] = j < h ? Atab[(size_t)v * h + j] : 0.0;
            Gv[t] = j < h ? Gtab[(size_t)v * h + j] : 0.0;
        }
        // device features, lane = device (policy.py:240-246)
        double f0 = 0.0, f1 = 0.0, f2 = 0.0, f3 = 0.0, f4 = 0.0;
        if (lane < D) {
            f0 = aflops;
            bool any_local = false;
            for (int j = PR.pred_ptr[v]; j < PR.pred_ptr[v + 1]; ++j) {
                const int p = PR.pred_idx[j];
                const int dp = dev[p];
                double arr = 0.0;
                if (!PR.is_entry[p]) {
                    arr = R.tend[p];
                    if (dp != lane)
                        arr = __dadd_rn(arr, __ddiv_rn(__dmul_rn(PR.obytes[p], PR.comm_factor),
                                                       PR.bw[dp * D + lane]));
                }
                f3 = j == PR.pred_ptr[v] ? arr : fmax(f3, arr);
                if (dp == lane) {
                    f1 = __dadd_rn(f1, PR.flops[p]);
                    f2 = any_local ? fmin(f2, R.tstart[p]) : R.tstart[p];
                    any_local = true;
                }
            }
            f4 = fmax(avail, f3);
            double *xr = R.xd + lane * 5;
            xr[0] = f0; xr[1] = f1; xr[2] = f2; xr[3] = f3; xr[4] = f4;
        }
        __syncwarp();
        {
            // column mean / population std, sequential over devices (numpy axis-0)
            double mean[5], sd[5];
#pragma unroll
            for (int c = 0; c < 5; ++c) {
                double sum = 0.0;
                for (int d = 0; d < D; ++d) sum = __dadd_rn(sum, R.xd[d * 5 + c]);
                mean[c] = __ddiv_rn(sum, (double)D);
                double sq = 0.0;
                for (int d = 0; d < D; ++d) {
                    const double df = __dsub_rn(R.xd[d * 5 + c], mean[c]);
                    sq = __dadd_rn(sq, __dmul_rn(df, df));
                }
                const double s = __dsqrt_rn(__ddiv_rn(sq, (double)D));
                sd[c] = s < 1e-12 ? 1.0 : s;
            }
            if (lane < D)
#pragma unroll
                for (int c = 0; c < 5; ++c)
                    R.xn[lane * 5 + c] = __ddiv_rn(__dsub_rn(R.xd[lane * 5 + c], mean[c]), sd[c]);
        }
        __syncwarp();
        double pre[MAXD][HPL];
        double part[MAXD];
#pragma unroll
        for (int d = 0; d < MAXD; ++d) {
            part[d] = 0.0;
            if (d < D) {
                const double x0 = R.xn[d * 5], x1 = R.xn[d * 5 + 1], x2 = R.xn[d * 5 + 2],
                             x3 = R.xn[d * 5 + 3], x4 = R.xn[d * 5 + 4];
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
            } else {
#pragma unroll
                for (int t = 0; t < HPL; ++t) pre[d][t] = 0.0;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int d = 0; d < MAXD; ++d) part[d] += __shfl_xor_sync(FP_FULL_MASK, part[d], o);
        // lane d owns device d
        double lg = -INFINITY;
#pragma unroll
        for (int d = 0; d < MAXD; ++d)
            if (d == lane && d < D) lg = part[d] + b2p;
        const double lmx = warp_max(lane < D ? lg : -INFINITY);
        const double ed = lane < D ? exp(lg - lmx) : 0.0;
        const double ecum = warp_inclusive_scan(ed);
        const double etot = __shfl_sync(FP_FULL_MASK, ecum, 31);
        const double pd = lane < D ? ed / etot : -1.0;
        double am = pd;
        int ai = lane < D ? lane : 0x7fffffff;
        warp_argmax_first(am, ai);
        const int amax_plc = ai;
        int jdx;
        if (forced) {
            jdx = frow[2 * step + 1];
            if (jdx < 0 || jdx >= D) { status = FP_EP_BAD_ACTION; break; }
        } else if (teacher) {
            double tv = lane < D ? f4 : INFINITY;
            int ti = lane < D ? lane : 0x7fffffff;
            warp_argmin_first(tv, ti);
            jdx = ti;
        } else if (greedy) {
            jdx = amax_plc;
        } else {
            double u1, u2;
            uniform2(philox4x32_10(U4{ctr_ep, (uint32_t)step, 1u, 0u}, k0, k1), u1, u2);
            if (u1 < eps) {
                jdx = min((int)(u2 * (double)D), D - 1);
            } else {
                const unsigned hit = __ballot_sync(FP_FULL_MASK, lane < D && ecum > u2 * etot);
                jdx = hit ? __ffs(hit) - 1 : D - 1;
            }
        }
        const double ekd = eps / (double)D;
        double mixd = 0.0, lmd = 0.0;
        if (lane < D) {
            mixd = __dadd_rn(__dmul_rn(pd, ome), ekd);
            lmd = log(__dadd_rn(mixd, 1e-30));
        }
        const double ent_plc = -warp_sum(lane < D ? mixd * lmd : 0.0);
        const double lp_plc = __shfl_sync(FP_FULL_MASK, lmd, jdx);

        if constexpr (GRAD) {
            const double pj = __shfl_sync(FP_FULL_MASK, pd, jdx);
            const double mj = __shfl_sync(FP_FULL_MASK, mixd, jdx);
            const double q = lane < D ? -ome * (lmd + mixd / __dadd_rn(mixd, 1e-30)) : 0.0;
            const double qpd = warp_sum(lane < D ? q * pd : 0.0);
            const double gl = lane < D ? ome * pj / __dadd_rn(mj, 1e-30) *
                                             ((lane == jdx ? 1.0 : 0.0) - pd) : 0.0;
            const double ge = lane < D ? pd * (q - qpd) : 0.0;
            double arl[HPL], are[HPL];
#pragma unroll
            for (int t = 0; t < HPL; ++t) arl[t] = are[t] = 0.0;
#pragma unroll
            for (int d = 0; d < MAXD; ++d) {
                if (d >= D) continue;
                const double gld = __shfl_sync(FP_FULL_MASK, gl, d);
                const double ged = __shfl_sync(FP_FULL_MASK, ge, d);
                if (lane == 0) { db2l += gld; db2e += ged; }
                const double x0 = R.xn[d * 5], x1 = R.xn[d * 5 + 1], x2 = R.xn[d * 5 + 2],
                             x3 = R.xn[d * 5 + 3], x4 = R.xn[d * 5 + 4];
#pragma unroll
                for (int t = 0; t < HPL; ++t) {
                    const double dl = gld * w2r[t] * lkd(pre[d][t], slope);
                    const double de = ged * w2r[t] * lkd(pre[d][t], slope);
                    const double lv = lk(pre[d][t], slope);
                    dwl[t] = fma(gld, lv, dwl[t]);
                    dwe[t] = fma(ged, lv, dwe[t]);
                    arl[t] += dl;
                    are[t] += de;
                    Rl[d][t] += dl;
                    Re[d][t] += de;
                    dMl[0][t] = fma(x0, dl, dMl[0][t]); dMe[0][t] = fma(x0, de, dMe[0][t]);
                    dMl[1][t] = fma(x1, dl, dMl[1][t]); dMe[1][t] = fma(x1, de, dMe[1][t]);
                    dMl[2][t] = fma(x2, dl, dMl[2][t]); dMe[2][t] = fma(x2, de, dMe[2][t]);
                    dMl[3][t] = fma(x3, dl, dMl[3][t]); dMe[3][t] = fma(x3, de, dMe[3][t]);
                    dMl[4][t] = fma(x4, dl, dMl[4][t]); dMe[4][t] = fma(x4, de, dMe[4][t]);
                }
            }
            double *row = A.grad_rows + ((size_t)ep * n + v) * 4 * h;
#pragma unroll
            for (int t = 0; t < HPL; ++t) {
                const int j = lane + 32 * t;
                if (j >= h) continue;
                row[j] = arl[t];
                row[h + j] = are[t];
#pragma unroll
                for (int d = 0; d < MAXD; ++d)
                    if (d == jdx) { row[2 * h + j] = Rl[d][t]; row[3 * h + j] = Re[d][t]; }
            }
        }

        // ================= commit =================
        if (lane == jdx) {
            aflops = __dadd_rn(aflops, PR.flops[v]);
            if (!PR.is_entry[v]) {
                const double st = f4;
                const double en = __dadd_rn(st, __ddiv_rn(PR.flops[v], PR.rates[jdx]));
                R.tstart[v] = st;
                R.tend[v] = en;
                avail = en;
            }
        }
#pragma unroll
        for (int d = 0; d < MAXD; ++d)
            if (d == jdx)
#pragma unroll
                for (int t = 0; t < HPL; ++t) Sd[d][t] += Gv[t];
        if (lane == 0) {
            dev[v] = (uint8_t)jdx;
            R.cand[v >> 5] &= ~(1u << (v & 31));
            const size_t o = (size_t)ep * n + step;
            if (A.step_vd) { A.step_vd[2 * o] = v; A.step_vd[2 * o + 1] = jdx; }
            if (A.step_lp) { A.step_lp[2 * o] = lp_sel; A.step_lp[2 * o + 1] = lp_plc; }
            if (A.step_ent) { A.step_ent[2 * o] = ent_sel; A.step_ent[2 * o + 1] = ent_plc; }
            if (A.step_argmax) {
                A.step_argmax[2 * o] = R.clist[amax_sel];
                A.step_argmax[2 * o + 1] = amax_plc;
            }
            if (A.step_ncand) A.step_ncand[o] = k;
        }
        __syncwarp();
        for (int j = PR.succ_ptr[v] + lane; j < PR.succ_ptr[v + 1]; j += 32) {
            const int w = PR.succ_idx[j];
            if (atomicSub(&R.npl[w], 1) == 1) atomicOr(&R.cand[w >> 5], 1u << (w & 31));
        }
        __syncwarp();
    }

    // ---- episode outputs ----
    for (int v = lane; v < n; v += 32) A.assign[(size_t)ep * n + v] = dev[v] == 0xFF ? -1 : dev[v];
    if constexpr (GRAD) if (status == FP_EP_OK) {
        double *g = A.grad_ep + (size_t)ep * grad_ep_stride(n, h, D);
        for (int v = lane; v < n; v += 32) { g[v] = R.dsl[v]; g[n + v] = R.dse[v]; }
        double *q = g + 2 * n;
#pragma unroll
        for (int t = 0; t < HPL; ++t) {
            const int j = lane + 32 * t;
            if (j >= h) continue;
#pragma unroll
            for (int c = 0; c < 5; ++c) { q[c * h + j] = dMl[c][t]; q[5 * h + c * h + j] = dMe[c][t]; }
            q[10 * h + j] = dwl[t];
            q[11 * h + j] = dwe[t];
#pragma unroll
            for (int d = 0; d < MAXD; ++d)
                if (d < D) {
                    q[12 * h + 2 + d * h + j] = Rl[d][t];
                    q[12 * h + 2 + D * h + d * h + j] = Re[d][t];
                }
        }
        if (lane == 0) { q[12 * h] = db2l; q[12 * h + 1] = db2e; }
    }
    double mk = 0.0;
    if (status == FP_EP_OK && A.simulate) {
        __syncwarp();
        SimOut o = sim_episode(PR, S, A.strategy, nullptr,
                               A.trace ? A.trace + (size_t)ep * A.trace_cap : nullptr, A.trace_cap,
                               nullptr);
        status = o.status;
        mk = o.makespan;
        if (lane == 0 && A.trace_len) A.trace_len[ep] = o.n_events;
    }
    if (lane == 0) {
        if (A.makespan) A.makespan[ep] = mk;
        if (A.status) A.status[ep] = status;
    }
}

template <int MAXD, int HPL, bool GRAD>
static int launch_rollout(const fp_problem *p, const fp_policy *pol, const fp_rollout_args &a,
                          cudaStream_t st) {
    constexpr int WARPS = 4;
    const DevProblem &PR = p->dev;
    const int64_t rb = roll_smem_bytes(PR.n, PR.W);
    const int64_t per = (rb + p->sim_smem + 15) / 16 * 16;
    const int64_t smem = per * WARPS;
    if (smem > 227 * 1024) {
        set_error("episode state exceeds shared memory for this graph size");
        return FP_ERR_UNSUPPORTED;
    }
    auto kern = rollout_kernel<MAXD, HPL, GRAD, WARPS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FP_ERR_CUDA; }
    const int grid = (a.B + WARPS - 1) / WARPS;
    kern<<<grid, WARPS * 32, smem, st>>>(PR, pol->dev, a, per, rb);
    e = cudaGetLastError();
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FP_ERR_CUDA; }
    return FP_OK;
}

template <int MAXD, int HPL>
static int dispatch_grad(const fp_problem *p, const fp_policy *pol, const fp_rollout_args &a,
                         cudaStream_t st) {
    return a.grad_rows ? launch_rollout<MAXD, HPL, true>(p, pol, a, st)
                       : launch_rollout<MAXD, HPL, false>(p, pol, a, st);
}

}  // namespace fp

using namespace fp;

extern "C" {

int fp_grad_ep_stride(const fp_policy *pol, int32_t d, int64_t *stride) {
    if (!pol || !stride) { set_error("null argument"); return FP_ERR_INVALID; }
    *stride = grad_ep_stride(pol->dev.n, pol->dev.h, d);
    return FP_OK;
}

int fp_rollout_batch(const fp_problem *p, const fp_policy *pol, const fp_rollout_args *args,
                     void *stream) {
    if (!p || !pol || !args || !args->assign || !args->status) {
        set_error("null argument");
        return FP_ERR_INVALID;
    }
    const fp_rollout_args &a = *args;
    if (a.B <= 0) return FP_OK;
    if (p->dev.n > 1024) { set_error("rollout kernel supports n <= 1024"); return FP_ERR_UNSUPPORTED; }
    if (a.mode == FP_MODE_FORCED && !a.forced) { set_error("FORCED mode needs actions"); return FP_ERR_INVALID; }
    if (a.mode < 0 || a.mode > 3) { set_error("unknown mode"); return FP_ERR_INVALID; }
    if (a.grad_rows && !a.grad_ep) { set_error("grad_rows needs grad_ep"); return FP_ERR_INVALID; }
    if (a.simulate && !a.makespan) { set_error("simulate needs makespan"); return FP_ERR_INVALID; }
    cudaStream_t st = (cudaStream_t)stream;
    const int D = p->dev.d, h = pol->dev.h;
    if (h <= 32) {
        if (D <= 4) return dispatch_grad<4, 1>(p, pol, a, st);
        if (D <= 8) return dispatch_grad<8, 1>(p, pol, a, st);
        if (D <= 16) return dispatch_grad<16, 1>(p, pol, a, st);
        return dispatch_grad<32, 1>(p, pol, a, st);
    }
    if (D <= 8) return dispatch_grad<8, 2>(p, pol, a, st);
    if (D <= 16) return dispatch_grad<16, 2>(p, pol, a, st);
    return dispatch_grad<32, 2>(p, pol, a, st);
}

}  // extern "C"
