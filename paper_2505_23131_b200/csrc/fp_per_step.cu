// per_step message passing (reference policy.py:353-371, mp_mode="per_step";
// Appendix I of the paper): both encoders re-run before EVERY decision with
// the dynamic input columns dyn[v] = (1, (d+1)/D) of the vertices placed so
// far, so SEL logits and the PLC tables change every step and nothing can be
// precomputed per snapshot.  This is the genuinely batched GNN workload: the
// B episodes advance in lockstep, and each step is
//
//   1. one encode of all B x n rows (gnn_proj0 with the per-episode dyn
//      columns, then K x (aggregation + DMMA node MLPs) -- the same kernels
//      as the per-snapshot encoder, run over a B*n-row batch);
//   2. ps_step_kernel, one 4-warp block per episode: SEL logits of the
//      current candidates from this step's H_sel (path sums over the explicit
//      b/t path lists, head1 as a lane-per-column mat-vec; candidates spread
//      over the warps), masked softmax + decision, then the PLC step on this step's A / G rows
//      (h_d = sum of G over the vertices placed on d, recomputed because G
//      changed), device features, standardisation, softmax over devices,
//      decision, timeline commit -- the per_episode kernels' math, with the
//      episode state in the workspace between launches.
//
// After n steps the assignments are scored by the compact simulator.  With
// grad_rows the step kernel also records each decision (normalised device
// features, vertex / device, candidate bitset) for fp_pg_reduce_per_step,
// which backpropagates through every step's encode (end of this file).
#include <vector>

#include "fp_rollout.cuh"

namespace fp {

constexpr int kPsWarps = 4;

struct PsState {
    int *dev;        // [B*n] device of each vertex, -1 unplaced (also the dyn columns)
    int *npl;        // [B*n] unplaced predecessors
    uint32_t *cand;  // [B][W] candidate bitsets
    int *order;      // [B*n] placement order
    double *tstart, *tend;   // [B*n] timeline
    double *avail, *aflops;  // [B][32]
    int *stat;       // [B] FP_EP_* (non-zero: episode stopped)
};

struct PsLayout {
    int64_t dev, npl, cand, order, tstart, tend, avail, aflops, stat;
    int64_t H[2][kMaxRounds + 1], Pm[2][kMaxRounds], Qm[2][kMaxRounds], AG[2][kMaxRounds];
    int64_t Zs, A, G;
    int64_t X;  // bf16 encoder planes (tc mode), 0 bytes otherwise
    int64_t bytes;
};

static PsLayout ps_layout(int n, int B, int h, int K, int n_enc, int W, bool tc) {
    PsLayout L{};
    int64_t o = 0;
    const int64_t R = (int64_t)n * B;
    auto take = [&](int64_t bytes) {
        o = (o + 255) / 256 * 256;
        const int64_t at = o;
        o += std::max<int64_t>(bytes, 8);
        return at;
    };
    L.dev = take(4 * R); L.npl = take(4 * R); L.cand = take(4LL * B * W); L.order = take(4 * R);
    L.tstart = take(8 * R); L.tend = take(8 * R);
    L.avail = take(8LL * B * 32); L.aflops = take(8LL * B * 32);
    L.stat = take(4LL * B);
    for (int e = 0; e < n_enc; ++e) {
        L.H[e][0] = take(8 * R * 7);
        for (int k = 0; k < K; ++k) {
            L.H[e][k + 1] = take(8 * R * h);
            L.Pm[e][k] = take(8 * R * h);
            L.Qm[e][k] = take(8 * R * h);
            L.AG[e][k] = take(8 * R * h);
        }
    }
    L.Zs = take(8 * R * h); L.A = take(8 * R * h); L.G = take(8 * R * h);
    L.X = tc ? take(tc_plane_bytes(R, K, n_enc)) : 0;
    L.bytes = (o + 255) / 256 * 256;
    return L;
}

__global__ void ps_init_kernel(DevProblem PR, PsState S, int B) {
    const int lane = lane_id();
    const int ep = blockIdx.x * kPsWarps + (threadIdx.x >> 5);
    if (ep >= B) return;
    const int n = PR.n, W = PR.W;
    const size_t base = (size_t)ep * n;
    for (int w = lane; w < W; w += 32) S.cand[(size_t)ep * W + w] = 0u;
    if (lane < 32) { S.avail[ep * 32 + lane] = 0.0; S.aflops[ep * 32 + lane] = 0.0; }
    __syncwarp();
    for (int v = lane; v < n; v += 32) {
        const int np = PR.pred_ptr[v + 1] - PR.pred_ptr[v];
        S.dev[base + v] = -1;
        S.npl[base + v] = np;
        S.tstart[base + v] = 0.0;
        S.tend[base + v] = 0.0;
        if (np == 0) atomicOr(&S.cand[(size_t)ep * W + (v >> 5)], 1u << (v & 31));
    }
    if (lane == 0) S.stat[ep] = FP_EP_OK;
}

// One decision step (SEL then PLC) of every live episode: one block of
// kPsWarps warps per episode.  All warps compute candidate logits (candidate
// i on warp i mod kPsWarps: path sums + head1 mat-vec), warp 0 then runs the
// softmax / decision and the PLC step.
template <int MAXD, int HPL>
__global__ void __launch_bounds__(kPsWarps * 32)
ps_step_kernel(DevProblem PR, DevPolicy PO, DevPolicy PB, fp_rollout_args A, PsState S,
               int step) {
    constexpr int LOGD = PlcLog<MAXD>::v;
    __shared__ double xd_sm[32 * 5], xn_sm[32 * 5], st_sm[16];
    __shared__ double cs[1024];
    __shared__ int cid[1024];
    __shared__ int k_sm;
    __shared__ uint32_t cw_sm[32];  // this step's candidate bitset (REINFORCE record)
    __shared__ double sd_part[kPsWarps - 1][MAXD * HPL <= 16 ? MAXD : 1][MAXD * HPL <= 16 ? 32 * HPL : 1];
    const int lane = lane_id(), warp = threadIdx.x >> 5;
    const int ep = blockIdx.x;
    griddep_wait();  // (PDL) this step's encode complete
    if (ep >= A.B || S.stat[ep] != FP_EP_OK) return;  // block-uniform
    const int n = PR.n, W = PR.W, D = PR.d, h = PO.h;
    const size_t base = (size_t)ep * n;
    const double eps = A.epsilon, ome = 1.0 - eps, slope = PO.slope;
    const uint32_t k0 = (uint32_t)A.seed, k1 = (uint32_t)(A.seed >> 32);
    const uint32_t ctr_ep = A.episode_base + (uint32_t)ep;
    const int mode = A.mode;
    const bool want_lp = A.step_lp != nullptr || A.step_ent != nullptr;
    const bool want_amax = A.step_argmax != nullptr;
    const size_t o = base + step;
    const double *Hs = PB.H[0][PO.K];
    uint32_t *cand = S.cand + (size_t)ep * W;

    // ---------------- SEL: logits of the current candidates ----------------
    if (warp == 0) {
        const uint32_t cw = lane < W ? cand[lane] : 0u;
        const int pc = __popc(cw);
        const int incl = warp_inclusive_scan(pc);
        int q = incl - pc;
        uint32_t m = cw;
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            cid[q++] = lane * 32 + b;
        }
        cw_sm[lane] = cw;
        if (lane == 31) k_sm = incl;
    }
    __syncthreads();
    const int k = k_sm;
    if (k == 0) {
        if (threadIdx.x == 0) S.stat[ep] = FP_EP_DEADLOCK;
        return;
    }
    const double *w1 = PO.W(PR_SEL_H1_W), *b1 = PO.W(PR_SEL_H1_B), *w2 = PO.W(PR_SEL_H2_W);
    const double b2 = PO.W(PR_SEL_H2_B)[0];
    // Candidates in groups of PSG per warp (candidates i0 + c * kPsWarps): each
    // head-1 weight w1[.][j] is loaded once per group and feeds PSG independent
    // FMA chains (the per-candidate chain order is unchanged, so every logit
    // is the one-candidate loop's); the group's embedding loads are in flight
    // together.  (One candidate per trip was bound by the w1 loads on its
    // 128-long dependent chain: 48% of the kernel's stall samples.)
    constexpr int PSG = 4;
    for (int i0 = warp; i0 < k; i0 += kPsWarps * PSG) {
        double em[PSG][4][HPL];
#pragma unroll
        for (int c = 0; c < PSG; ++c) {
            const int i = i0 + c * kPsWarps;
            const int v = i < k ? cid[i] : -1;
#pragma unroll
            for (int t = 0; t < HPL; ++t) {
                const int j = lane + 32 * t;
                em[c][0][t] = em[c][1][t] = em[c][2][t] = em[c][3][t] = 0.0;
                if (j >= h || v < 0) continue;
                em[c][0][t] = Hs[(base + v) * h + j];
                double hb = 0.0, ht = 0.0;
#pragma unroll 4
                for (int q = PO.bp_ptr[v]; q < PO.bp_ptr[v + 1]; ++q) hb += Hs[(base + PO.bp_idx[q]) * h + j];
#pragma unroll 4
                for (int q = PO.tp_ptr[v]; q < PO.tp_ptr[v + 1]; ++q) ht += Hs[(base + PO.tp_idx[q]) * h + j];
                em[c][1][t] = hb;
                em[c][2][t] = ht;
                em[c][3][t] = PB.Zs[(base + v) * h + j];
            }
        }
        double acc[PSG][HPL];
#pragma unroll
        for (int c = 0; c < PSG; ++c)
#pragma unroll
            for (int t = 0; t < HPL; ++t) acc[c][t] = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll 4
            for (int ii = 0; ii < h; ++ii) {
                double w[HPL];
#pragma unroll
                for (int t = 0; t < HPL; ++t) {
                    const int j = lane + 32 * t;
                    w[t] = j < h ? w1[(b * h + ii) * h + j] : 0.0;
                }
#pragma unroll
                for (int c = 0; c < PSG; ++c) {
                    double ev = 0.0;
#pragma unroll
                    for (int t = 0; t < HPL; ++t) {
                        const double x = __shfl_sync(FP_FULL_MASK, em[c][b][t], ii & 31);
                        if ((ii >> 5) == t) ev = x;
                    }
#pragma unroll
                    for (int t = 0; t < HPL; ++t) {
                        const int j = lane + 32 * t;
                        if (j < h) acc[c][t] = fma(ev, w[t], acc[c][t]);
                    }
                }
            }
#pragma unroll
        for (int c = 0; c < PSG; ++c) {
            const int i = i0 + c * kPsWarps;
            double part = 0.0;
#pragma unroll
            for (int t = 0; t < HPL; ++t) {
                const int j = lane + 32 * t;
                if (j < h) part = fma(lk(acc[c][t] + b1[j], slope), w2[j], part);
            }
            part = warp_sum(part);
            if (lane == 0 && i < k) cs[i] = part + b2;
        }
    }
    // h_d partial sums: h_d = sum of this step's G rows over the vertices
    // placed on d (before this step) -- independent of this step's choices,
    // so every warp takes a contiguous quarter of the placement order
    constexpr bool SPLIT = MAXD * HPL <= 16;
    double Sd[MAXD][HPL];
#pragma unroll
    for (int d = 0; d < MAXD; ++d)
#pragma unroll
        for (int t = 0; t < HPL; ++t) Sd[d][t] = 0.0;
    {
        const int nw = SPLIT ? kPsWarps : 1;
        const int chunk = (step + nw - 1) / nw;
        const int i_lo = SPLIT ? warp * chunk : 0, i_hi = SPLIT ? min(step, i_lo + chunk) : step;
        if (SPLIT || warp == 0)
            for (int i0 = i_lo; i0 < i_hi; i0 += 32) {
                // 32 placed vertices at a time: lane i loads (u, d_u), then the G
                // rows are summed in placement order (independent loads in flight)
                const int cnt = min(32, i_hi - i0);
                const int my_u = lane < cnt ? S.order[base + i0 + lane] : 0;
                const int my_d = lane < cnt ? S.dev[base + my_u] : -1;
#pragma unroll 4
                for (int i = 0; i < cnt; ++i) {
                    const int u = __shfl_sync(FP_FULL_MASK, my_u, i);
                    const int du = __shfl_sync(FP_FULL_MASK, my_d, i);
#pragma unroll
                    for (int t = 0; t < HPL; ++t) {
                        const int j = lane + 32 * t;
                        const double g = j < h ? PB.G[(base + u) * h + j] : 0.0;
#pragma unroll
                        for (int d = 0; d < MAXD; ++d)
                            if (d == du) Sd[d][t] += g;
                    }
                }
            }
        if constexpr (SPLIT) {
            if (warp != 0)
#pragma unroll
                for (int d = 0; d < MAXD; ++d)
#pragma unroll
                    for (int t = 0; t < HPL; ++t)
                        sd_part[warp - 1][d][lane + 32 * t] = Sd[d][t];
        }
    }
    __syncthreads();
    if (warp != 0) return;
    if constexpr (SPLIT)  // fixed order: warp 0's quarter, then warps 1, 2, 3
#pragma unroll
        for (int w = 0; w < kPsWarps - 1; ++w)
#pragma unroll
            for (int d = 0; d < MAXD; ++d)
#pragma unroll
                for (int t = 0; t < HPL; ++t) Sd[d][t] += sd_part[w][d][lane + 32 * t];
    // masked softmax over the candidates in ascending-id order (policy.py:204)
    double mx = -INFINITY;
    for (int i = lane; i < k; i += 32) mx = fmax(mx, cs[i]);
    mx = warp_max_redux(mx);
    double tot = 0.0;
    {
        double carry = 0.0;
        for (int b0 = 0; b0 < k; b0 += 32) {
            const int i = b0 + lane;
            const double e = i < k ? exp(cs[i] - mx) : 0.0;
            const double cum = warp_inclusive_scan(e) + carry;
            carry = __shfl_sync(FP_FULL_MASK, cum, 31);
        }
        tot = carry;
    }
    int idx = -1;
    double su1 = 0.0, su2 = 0.0;
    if (mode == FP_MODE_SAMPLE)
        uniform2(philox4x32_10(U4{ctr_ep, (uint32_t)step, 0u, 0u}, k0, k1), su1, su2);
    if (mode == FP_MODE_FORCED) {
        const int fv = A.forced[2 * o];
        for (int b0 = 0; b0 < k && idx < 0; b0 += 32) {
            const unsigned hit = __ballot_sync(FP_FULL_MASK, b0 + lane < k && cid[b0 + lane] == fv);
            if (hit) idx = b0 + __ffs(hit) - 1;
        }
    } else if (mode == FP_MODE_TEACHER) {
        double bt = -INFINITY;
        for (int i = lane; i < k; i += 32) bt = fmax(bt, PR.tlev[cid[i]]);
        bt = warp_max_redux(bt);
        for (int b0 = 0; b0 < k && idx < 0; b0 += 32) {
            const unsigned hit =
                __ballot_sync(FP_FULL_MASK, b0 + lane < k && PR.tlev[cid[b0 + lane]] == bt);
            if (hit) idx = b0 + __ffs(hit) - 1;
        }
    } else if (mode == FP_MODE_SAMPLE) {
        if (su1 < eps) {
            idx = min((int)(su2 * (double)k), k - 1);
        } else {
            const double target = su2 * tot;
            double carry = 0.0;
            for (int b0 = 0; b0 < k && idx < 0; b0 += 32) {
                const int i = b0 + lane;
                const double e = i < k ? exp(cs[i] - mx) : 0.0;
                const double cum = warp_inclusive_scan(e) + carry;
                const unsigned hit = __ballot_sync(FP_FULL_MASK, i < k && cum > target);
                if (hit) idx = b0 + __ffs(hit) - 1;
                carry = __shfl_sync(FP_FULL_MASK, cum, 31);
            }
            if (idx < 0) idx = k - 1;
        }
    }
    int amax = -1;
    if (want_amax || mode == FP_MODE_GREEDY) {
        double bp = -1.0;
        int bi = 0x7fffffff;
        for (int i = lane; i < k; i += 32) {
            const double p = exp(cs[i] - mx) / tot;
            if (p > bp) { bp = p; bi = i; }
        }
        warp_argmax_first(bp, bi);
        amax = bi;
        if (mode == FP_MODE_GREEDY) idx = amax;
    }
    if (idx < 0) {
        if (lane == 0) S.stat[ep] = FP_EP_BAD_ACTION;
        return;
    }
    const int v = cid[idx];
    if (want_lp) {
        const double ek = eps / (double)k;
        double entp = 0.0, lp = 0.0;
        for (int i = lane; i < k; i += 32) {
            const double p = exp(cs[i] - mx) / tot;
            const double mix = __dadd_rn(__dmul_rn(p, ome), ek);
            const double lm = log(__dadd_rn(mix, 1e-30));
            entp += mix * lm;
            if (i == idx) lp = lm;
        }
        const double ent = -warp_sum(entp);
        lp = warp_sum(lp);
        if (lane == 0) {
            if (A.step_lp) A.step_lp[2 * o] = lp;
            if (A.step_ent) A.step_ent[2 * o] = ent;
        }
    }
    if (lane == 0) {
        if (A.step_vd) A.step_vd[2 * o] = v;
        if (A.step_argmax) A.step_argmax[2 * o] = cid[amax];
        if (A.step_ncand) A.step_ncand[o] = k;
        cand[v >> 5] &= ~(1u << (v & 31));
    }
    __syncwarp();
    for (int j = PR.succ_ptr[v] + lane; j < PR.succ_ptr[v + 1]; j += 32) {
        const int w = PR.succ_idx[j];
        if (atomicSub(&S.npl[base + w], 1) == 1) atomicOr(&cand[w >> 5], 1u << (w & 31));
    }

    // ---------------- PLC ----------------
    double *xd = xd_sm, *xn = xn_sm, *stats = st_sm;
    const int *pp = PR.pred_ptr, *pi = PR.pred_idx;
    const uint8_t *ent = PR.is_entry;
    double f4 = 0.0;
    if (lane < D) {
        double f2 = 0.0, f3 = 0.0;
        fp::NeuSum f1s;
        bool any_local = false;
        for (int j = pp[v]; j < pp[v + 1]; ++j) {
            const int p = pi[j];
            const int dp = S.dev[base + p];
            const double arr =
                ent[p] ? 0.0 : __dadd_rn(S.tend[base + p], PR.tdur[(p * D + dp) * D + lane]);
            f3 = j == pp[v] ? arr : fmax(f3, arr);
            if (dp == lane) {
                f1s.add(PR.flops[p]);
                f2 = any_local ? fmin(f2, S.tstart[base + p]) : S.tstart[base + p];
                any_local = true;
            }
        }
        f4 = fmax(S.avail[ep * 32 + lane], f3);
        double *xr = xd + lane * 5;
        xr[0] = S.aflops[ep * 32 + lane]; xr[1] = f1s.value(); xr[2] = f2; xr[3] = f3; xr[4] = f4;
    }
    __syncwarp();
    if (lane < 5) {
        double sum = 0.0;
        for (int d = 0; d < D; ++d) sum = __dadd_rn(sum, xd[d * 5 + lane]);
        const bool pow2 = (D & (D - 1)) == 0;
        const double invD = 1.0 / (double)D;
        const double mean = pow2 ? __dmul_rn(sum, invD) : __ddiv_rn(sum, (double)D);
        double sq = 0.0;
        for (int d = 0; d < D; ++d) {
            const double df = __dsub_rn(xd[d * 5 + lane], mean);
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
    for (int i = lane; i < 5 * D; i += 32) {
        const int c = i % 5;
        xn[i] = __dmul_rn(__dsub_rn(xd[i], stats[c]), stats[5 + c]);
    }
    __syncwarp();
    const double *w2p = PO.W(PR_PLC_H2_W);
    const double b2p = PO.W(PR_PLC_H2_B)[0];
    double part[MAXD];
#pragma unroll
    for (int d = 0; d < MAXD; ++d) {
        part[d] = 0.0;
        if (d < D) {
#pragma unroll
            for (int t = 0; t < HPL; ++t) {
                const int j = lane + 32 * t;
                if (j >= h) continue;
                double a = PB.A[(base + v) * h + j] + Sd[d][t] + PO.c[j];
#pragma unroll
                for (int c = 0; c < 5; ++c) a = fma(xn[d * 5 + c], PO.M[c * h + j], a);
                part[d] = fma(lk(a, slope), w2p[j], part[d]);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < LOGD; ++r) {
        const int off = 16 >> r;
        const bool upper = (lane & off) != 0;
        const int half = MAXD >> (r + 1);
#pragma unroll
        for (int i = 0; i < MAXD / 2; ++i) {
            if (i < half) {
                const double send = upper ? part[i] : part[i + half];
                const double keep = upper ? part[i + half] : part[i];
                part[i] = keep + __shfl_xor_sync(FP_FULL_MASK, send, off);
            }
        }
    }
#pragma unroll
    for (int off = 16 >> LOGD; off > 0; off >>= 1) part[0] += __shfl_xor_sync(FP_FULL_MASK, part[0], off);
    const double lgall = __shfl_sync(FP_FULL_MASK, part[0], (lane & (MAXD - 1)) << (5 - LOGD));
    const double lg = lane < D ? lgall + b2p : -INFINITY;
    const double lmx = warp_max_redux(lg);
    const double ed = lane < D ? exp(lg - lmx) : 0.0;
    const double ecum = warp_scan_pow2<LOGD>(ed);
    const double etot = __shfl_sync(FP_FULL_MASK, ecum, D - 1);
    const double pd = lane < D ? ed / etot : -1.0;
    int pam = -1;
    if (want_amax || mode == FP_MODE_GREEDY) {
        double am = pd;
        int ai = lane < D ? lane : 0x7fffffff;
        warp_argmax_first(am, ai);
        pam = ai;
    }
    int jdx;
    if (mode == FP_MODE_FORCED) {
        jdx = A.forced[2 * o + 1];
        if (jdx < 0 || jdx >= D) {
            if (lane == 0) S.stat[ep] = FP_EP_BAD_ACTION;
            return;
        }
    } else if (mode == FP_MODE_TEACHER) {
        const double tv = lane < D ? f4 : INFINITY;
        const double best = warp_min_redux(tv);
        jdx = __ffs(__ballot_sync(FP_FULL_MASK, lane < D && tv == best)) - 1;
    } else if (mode == FP_MODE_GREEDY) {
        jdx = pam;
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
            if (A.step_lp) A.step_lp[2 * o + 1] = lp;
            if (A.step_ent) A.step_ent[2 * o + 1] = entv;
        }
    }
    // commit (timeline.py:47-58) + the dyn columns of the next encode
    if (lane == jdx) {
        S.aflops[ep * 32 + jdx] = __dadd_rn(S.aflops[ep * 32 + jdx], PR.flops[v]);
        if (!ent[v]) {
            const double en = __dadd_rn(f4, PR.edur[v * D + jdx]);
            S.tstart[base + v] = f4;
            S.tend[base + v] = en;
            S.avail[ep * 32 + jdx] = en;
        }
        S.dev[base + v] = jdx;
        S.order[base + step] = v;
        if (A.step_vd) A.step_vd[2 * o + 1] = jdx;
    }
    if (lane == 0 && A.step_argmax) A.step_argmax[2 * o + 1] = pam;
    if (A.grad_rows) {  // REINFORCE record (replayed by fp_pg_reduce_per_step)
        double *rec = A.grad_rows + o * grad_rec_stride(D, W);
        for (int i = lane; i < 5 * D; i += 32) rec[i] = xn[i];
        if (lane == 0) { *(int2 *)(rec + 6 * D) = make_int2(v, jdx); rec[6 * D + 3] = (double)v; }
        if (lane < W) ((uint32_t *)(rec + 6 * D + 4))[lane] = cw_sm[lane];
    }
}

// assignments out (unplaced -> 0 for the simulator, fixed up afterwards)
__global__ void ps_finish_kernel(PsState S, fp_rollout_args A, int n, int fixup, int64_t gstride) {
    const int64_t total = (int64_t)A.B * n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int ep = (int)(i / n);
        const int d = S.dev[i];
        if (!fixup) {
            A.assign[i] = d < 0 ? 0 : d;
        } else if (S.stat[ep] != FP_EP_OK) {
            A.assign[i] = d;
            if (i % n == 0) {
                A.status[ep] = S.stat[ep];
                if (A.makespan) A.makespan[ep] = 0.0;
            }
        }
        if (fixup && A.grad_ep && i % n == 0) {  // replay header: chain completed, epsilon
            double *g = A.grad_ep + (size_t)ep * gstride;
            g[2 * n] = S.stat[ep] == FP_EP_OK ? 1.0 : 0.0;
            g[2 * n + 1] = A.epsilon;
        }
    }
}

template <int MAXD, int HPL>
static void ps_launch_step(const fp_problem *p, const fp_policy *pol, const DevPolicy &PB,
                           const fp_rollout_args &a, const PsState &S, int step,
                           cudaStream_t st) {
    launch_pdl(ps_step_kernel<MAXD, HPL>, dim3(a.B), dim3(kPsWarps * 32), 0, st, p->dev, pol->dev, PB, a,
               S, step);
}

int per_step_rollout(const fp_problem *p, const fp_policy *pol, const fp_rollout_args &a,
                     int64_t *ws_needed, cudaStream_t st) {
    const DevProblem &PR = p->dev;
    const DevPolicy &PO = pol->dev;
    if (PO.forest || PR.n > 1024) {
        set_error("per_step message passing supports graphs up to 1024 ops");
        return FP_ERR_UNSUPPORTED;
    }

    if (PO.h % 8 != 0 || PO.h > 64) {
        set_error("per_step message passing needs hidden in {8, 16, 32, 64}");
        return FP_ERR_UNSUPPORTED;
    }
    const int n = PR.n, B = a.B;
    const PsLayout L = ps_layout(n, B, PO.h, PO.K, PO.n_enc, PR.W, PO.tc != 0);
    if (ws_needed) { *ws_needed = L.bytes; return FP_OK; }
    if (a.grad_rows && !a.grad_ep) {
        set_error("a per_step REINFORCE rollout needs grad_ep with grad_rows");
        return FP_ERR_INVALID;
    }
    if (!a.workspace || a.workspace_bytes < L.bytes) {
        set_error("workspace too small for the per_step rollout (see fp_rollout_workspace_size)");
        return FP_ERR_INVALID;
    }
    if (!PO.params) { set_error("fp_policy_prepare must run before a per_step rollout"); return FP_ERR_INVALID; }
    uint8_t *w = (uint8_t *)a.workspace;
    PsState S;
    S.dev = (int *)(w + L.dev); S.npl = (int *)(w + L.npl); S.cand = (uint32_t *)(w + L.cand);
    S.order = (int *)(w + L.order); S.tstart = (double *)(w + L.tstart);
    S.tend = (double *)(w + L.tend); S.avail = (double *)(w + L.avail);
    S.aflops = (double *)(w + L.aflops);
    S.stat = (int *)(w + L.stat);
    DevPolicy PB = PO;  // weights + graph constants shared; activations over B*n rows
    PB.rows = n * B;
    PB.batch = B;
    PB.ps_dev = S.dev;
    for (int e = 0; e < PO.n_enc; ++e) {
        PB.H[e][0] = (double *)(w + L.H[e][0]);
        for (int k = 0; k < PO.K; ++k) {
            PB.H[e][k + 1] = (double *)(w + L.H[e][k + 1]);
            PB.Pm[e][k] = (double *)(w + L.Pm[e][k]);
            PB.Qm[e][k] = (double *)(w + L.Qm[e][k]);
            PB.AG[e][k] = (double *)(w + L.AG[e][k]);
        }
    }
    PB.Zs = (double *)(w + L.Zs); PB.A = (double *)(w + L.A); PB.G = (double *)(w + L.G);
    if (PB.tc) {  // the B x n-row X planes; columns nobody writes stay zero
        tc_set_planes(PB, w + L.X, (int64_t)n * B);
        cudaMemsetAsync(w + L.X, 0, tc_plane_bytes((int64_t)n * B, PO.K, PO.n_enc), st);
    }
    ps_init_kernel<<<(B + kPsWarps - 1) / kPsWarps, kPsWarps * 32, 0, st>>>(PR, S, B);
    const int D = PR.d, h = PO.h;
    for (int step = 0; step < n; ++step) {
        int rc = gnn_encode_rows(PB, st, false, false);
        if (rc) return rc;
        if (h <= 32) {
            if (D <= 4) ps_launch_step<4, 1>(p, pol, PB, a, S, step, st);
            else if (D <= 8) ps_launch_step<8, 1>(p, pol, PB, a, S, step, st);
            else if (D <= 16) ps_launch_step<16, 1>(p, pol, PB, a, S, step, st);
            else ps_launch_step<32, 1>(p, pol, PB, a, S, step, st);
        } else {
            if (D <= 8) ps_launch_step<8, 2>(p, pol, PB, a, S, step, st);
            else if (D <= 16) ps_launch_step<16, 2>(p, pol, PB, a, S, step, st);
            else ps_launch_step<32, 2>(p, pol, PB, a, S, step, st);
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FP_ERR_CUDA; }
    }
    const int fb = (int)std::min<int64_t>(((int64_t)B * n + 255) / 256, 4096);
    ps_finish_kernel<<<fb, 256, 0, st>>>(S, a, n, 0, 0);
    // status of episodes that finished cleanly, then the simulator's verdict
    fp_rollout_args a2 = a;
    if (a.simulate) {
        int rc = sim_launch_compact(p, a.assign, B, a.strategy, a.makespan, a.status, a.trace,
                                    a.trace_cap, a.trace_len, st);
        if (rc) return rc;
    } else {
        cudaMemsetAsync(a.status, 0, sizeof(int32_t) * B, st);
    }
    ps_finish_kernel<<<fb, 256, 0, st>>>(S, a2, n, 1, grad_ep_stride(n, PO.h, PR.d));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FP_ERR_CUDA; }
    return FP_OK;
}

}  // namespace fp

// ---------------------------------------------------------------------------
// per_step REINFORCE (reference sim_rl_stage with mp_mode="per_step":
// policy.py:353-371 + training.py:181-216, autodiff of nn.py): the log-probs
// of step t depend on that step's encodes, so the gradient backpropagates
// through one encode per step.  Per (episode, step), in order: the encoders'
// dynamic input columns are set to the placements before the step, the
// encode runs with its backward intermediates, ps_adjoint_kernel forms the
// head-table adjoints of this step's two decisions (SEL logits of the
// candidates; PLC A row, G rows via the per-device sums, M, w2, b2), folded
// with (alpha_e, beta), and the per-snapshot backward (fp_policy_backward)
// turns them into a flat gradient that is accumulated in (episode, step)
// order.  Records come from the forward per_step rollout (normalised device
// features, vertex / device, candidate bitset).  Sequential and launch-heavy
// (about 30 launches per decision): the correctness path of the per_step
// ablation, not a throughput path.
// ---------------------------------------------------------------------------
namespace fp {

// dyn columns (H0 cols 5, 6 of every encoder) = placements of steps < t
__global__ void ps_set_dyn_kernel(DevPolicy P, const double *rec, int rstride, int t, int D) {
    extern __shared__ int dv[];
    const int n = P.n;
    for (int v = threadIdx.x; v < n; v += blockDim.x) dv[v] = -1;
    __syncthreads();
    for (int s = threadIdx.x; s < t; s += blockDim.x) {
        const int2 vj = *(const int2 *)(rec + (size_t)s * rstride + 6 * D);
        dv[vj.x] = vj.y;
    }
    __syncthreads();
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
        const int d = dv[v];
        for (int e = 0; e < P.n_enc; ++e) {
            double *H0 = P.H[e][0];
            H0[(size_t)v * 7 + 5] = d < 0 ? 0.0 : 1.0;
            H0[(size_t)v * 7 + 6] = d < 0 ? 0.0 : __ddiv_rn((double)(d + 1), (double)D);
        }
    }
}

template <int MAXD, int HPL>
__global__ void __launch_bounds__(32)
ps_adjoint_kernel(DevProblem PR, DevPolicy P, const double *__restrict__ rec, int rstride, int t,
                  double al, double beta, double eps) {
    extern __shared__ int cl[];
    const int lane = lane_id();
    const int n = PR.n, D = PR.d, W = PR.W, h = P.h;
    const double ome = 1.0 - eps, slope = P.slope;
    for (int i = lane; i < n * h; i += 32) { P.dA[i] = 0.0; P.dG[i] = 0.0; }
    for (int v = lane; v < n; v += 32) P.ds[v] = 0.0;
    for (int k = lane; k < 6 * h + 1; k += 32) P.dsmall[h + k] = 0.0;
    const double *r = rec + (size_t)t * rstride;
    const int2 vj = *(const int2 *)(r + 6 * D);
    const int v = vj.x, jdx = vj.y;
    __syncwarp();
    // ---- SEL: this step's candidates, logits from this step's encode ----
    {
        const uint32_t cw = lane < W ? ((const uint32_t *)(r + 6 * D + 4))[lane] : 0u;
        const int pc = __popc(cw);
        const int incl = warp_inclusive_scan(pc);
        const int k = __shfl_sync(FP_FULL_MASK, incl, 31);
        int o = incl - pc;
        uint32_t m = cw;
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            cl[o++] = lane * 32 + b;
        }
        __syncwarp();
        double mx = -INFINITY;
        for (int i = lane; i < k; i += 32) mx = fmax(mx, P.s[cl[i]]);
        mx = warp_max(mx);
        double tot = 0.0;
        for (int i = lane; i < k; i += 32) tot += exp(P.s[cl[i]] - mx);
        tot = warp_sum(tot);
        const double ek = eps / (double)k;
        double qp = 0.0;
        for (int i = lane; i < k; i += 32) {
            const double p = exp(P.s[cl[i]] - mx) / tot;
            const double mix = __dadd_rn(__dmul_rn(p, ome), ek);
            const double lm = log(__dadd_rn(mix, 1e-30));
            qp += -ome * (lm + mix / __dadd_rn(mix, 1e-30)) * p;
        }
        qp = warp_sum(qp);
        const double pv = exp(P.s[v] - mx) / tot;
        const double mv = __dadd_rn(__dmul_rn(pv, ome), ek);
        const double c1 = ome * pv / __dadd_rn(mv, 1e-30);
        for (int i = lane; i < k; i += 32) {
            const int u = cl[i];
            const double p = exp(P.s[u] - mx) / tot;
            const double mix = __dadd_rn(__dmul_rn(p, ome), ek);
            const double lm = log(__dadd_rn(mix, 1e-30));
            const double q = -ome * (lm + mix / __dadd_rn(mix, 1e-30));
            P.ds[u] = al * (c1 * ((u == v ? 1.0 : 0.0) - p)) + beta * (p * (q - qp));
        }
    }
    // ---- PLC: pre-activations from this step's tables, lane = hidden column ----
    double Sd[MAXD][HPL], pre[MAXD][HPL];
#pragma unroll
    for (int d = 0; d < MAXD; ++d)
#pragma unroll
        for (int q = 0; q < HPL; ++q) Sd[d][q] = 0.0;
    for (int s = 0; s < t; ++s) {
        const int2 us = *(const int2 *)(rec + (size_t)s * rstride + 6 * D);
#pragma unroll
        for (int q = 0; q < HPL; ++q) {
            const int j = lane + 32 * q;
            const double g = j < h ? P.G[(size_t)us.x * h + j] : 0.0;
#pragma unroll
            for (int d = 0; d < MAXD; ++d)
                if (d == us.y) Sd[d][q] += g;
        }
    }
    const double *w2p = P.W(PR_PLC_H2_W);
    const double b2p = P.W(PR_PLC_H2_B)[0];
    double lg[MAXD];
#pragma unroll
    for (int d = 0; d < MAXD; ++d) {
        double part = 0.0;
#pragma unroll
        for (int q = 0; q < HPL; ++q) {
            const int j = lane + 32 * q;
            pre[d][q] = 0.0;
            if (j >= h || d >= D) continue;
            double a = P.A[(size_t)v * h + j] + Sd[d][q] + P.c[j];
            for (int c = 0; c < 5; ++c) a = fma(r[d * 5 + c], P.M[c * h + j], a);
            pre[d][q] = a;
            part = fma(lk(a, slope), w2p[j], part);
        }
        lg[d] = d < D ? warp_sum(part) + b2p : -INFINITY;
    }
    double mx = -INFINITY;
#pragma unroll
    for (int d = 0; d < MAXD; ++d) mx = fmax(mx, lg[d]);
    double ed[MAXD], tot = 0.0;
#pragma unroll
    for (int d = 0; d < MAXD; ++d) { ed[d] = d < D ? exp(lg[d] - mx) : 0.0; tot += ed[d]; }
    const double ekd = eps / (double)D;
    double pd[MAXD], qd[MAXD], qp = 0.0, pj = 0.0, mj = 0.0;
#pragma unroll
    for (int d = 0; d < MAXD; ++d) {
        pd[d] = qd[d] = 0.0;
        if (d >= D) continue;
        pd[d] = ed[d] / tot;
        const double mix = __dadd_rn(__dmul_rn(pd[d], ome), ekd);
        const double lm = log(__dadd_rn(mix, 1e-30));
        qd[d] = -ome * (lm + mix / __dadd_rn(mix, 1e-30));
        qp += qd[d] * pd[d];
        if (d == jdx) { pj = pd[d]; mj = mix; }
    }
    const double g0 = ome * pj / __dadd_rn(mj, 1e-30);
    double cd[MAXD], db2 = 0.0;
#pragma unroll
    for (int d = 0; d < MAXD; ++d) {
        cd[d] = d < D ? al * (g0 * ((d == jdx ? 1.0 : 0.0) - pd[d])) + beta * (pd[d] * (qd[d] - qp))
                      : 0.0;
        db2 += cd[d];
    }
#pragma unroll
    for (int q = 0; q < HPL; ++q) {
        const int j = lane + 32 * q;
        if (j >= h) continue;
        double dA = 0.0, dw = 0.0, dM[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        double dS[MAXD];
#pragma unroll
        for (int d = 0; d < MAXD; ++d) {
            dS[d] = 0.0;
            if (d >= D) continue;
            dS[d] = cd[d] * w2p[j] * lkd(pre[d][q], slope);
            dA += dS[d];
            dw = fma(cd[d], lk(pre[d][q], slope), dw);
            for (int c = 0; c < 5; ++c) dM[c] = fma(r[d * 5 + c], dS[d], dM[c]);
        }
        P.dA[(size_t)v * h + j] = dA;
        for (int c = 0; c < 5; ++c) P.dsmall[h + c * h + j] = dM[c];
        P.dsmall[6 * h + j] = dw;
        for (int s = 0; s < t; ++s) {  // G rows of the placed vertices, through S_d
            const int2 us = *(const int2 *)(rec + (size_t)s * rstride + 6 * D);
#pragma unroll
            for (int d = 0; d < MAXD; ++d)
                if (d == us.y) P.dG[(size_t)us.x * h + j] = dS[d];
        }
    }
    if (lane == 0) P.dsmall[7 * h] = db2;
}

__global__ void axpy_kernel(double *y, const double *x, int64_t count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) y[i] += x[i];
}

template <int MAXD, int HPL>
static void ps_adjoint_launch(const DevProblem &PR, const DevPolicy &P, const double *rec,
                              int rstride, int t, double al, double beta, double eps,
                              cudaStream_t st) {
    ps_adjoint_kernel<MAXD, HPL><<<1, 32, 4 * PR.n, st>>>(PR, P, rec, rstride, t, al, beta, eps);
}

}  // namespace fp

extern "C" int fp_policy_backward(fp_policy *pol, double *grad, void *stream);

#define FP_PS_CUDA(call)                                                   \
    do {                                                                   \
        cudaError_t e_ = (call);                                           \
        if (e_ != cudaSuccess) {                                           \
            fp::set_error(std::string(#call) + ": " + cudaGetErrorString(e_)); \
            return FP_ERR_CUDA;                                            \
        }                                                                  \
    } while (0)

extern "C" int fp_pg_reduce_per_step(fp_policy *pol, const double *grad_rows,
                                     const double *grad_ep, const double *alpha, double beta,
                                     int32_t B, double *grad, void *stream) {
    using namespace fp;
    if (!pol || !grad_rows || !grad_ep || !alpha || !grad || B <= 0) {
        set_error("bad pg_reduce_per_step arguments");
        return FP_ERR_INVALID;
    }
    DevPolicy &P = pol->dev;
    const DevProblem &PR = pol->problem->dev;
    if (P.forest || P.tc || pol->fused_encoder) {
        set_error("per_step REINFORCE needs the fp64 split encoder with explicit path lists");
        return FP_ERR_UNSUPPORTED;
    }
    if (!P.params) { set_error("fp_policy_prepare must run before the backward"); return FP_ERR_INVALID; }
    cudaStream_t st = (cudaStream_t)stream;
    const int n = PR.n, D = PR.d, h = P.h;
    const int rstride = grad_rec_stride(D, PR.W);
    const int64_t gstride = grad_ep_stride(n, h, D);
    std::vector<double> hdr((size_t)B * 2), al((size_t)B);
    FP_PS_CUDA(cudaMemcpy2DAsync(hdr.data(), 2 * sizeof(double), grad_ep + 2 * n,
                              gstride * sizeof(double), 2 * sizeof(double), B,
                              cudaMemcpyDeviceToHost, st));
    FP_PS_CUDA(cudaMemcpyAsync(al.data(), alpha, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
    FP_PS_CUDA(cudaStreamSynchronize(st));
    double *tmp = nullptr;
    FP_PS_CUDA(cudaMallocAsync((void **)&tmp, sizeof(double) * pol->n_params, st));
    FP_PS_CUDA(cudaMemsetAsync(grad, 0, sizeof(double) * pol->n_params, st));
    const int ab = (int)((pol->n_params + 255) / 256);
    int rc = FP_OK;
    for (int e = 0; e < B && rc == FP_OK; ++e) {
        if (hdr[2 * e] == 0.0) continue;  // failed chain: no contribution
        const double eps = hdr[2 * e + 1];
        const double *rec = grad_rows + (size_t)e * n * rstride;
        for (int t = 0; t < n && rc == FP_OK; ++t) {
            ps_set_dyn_kernel<<<1, 256, 4 * n, st>>>(P, rec, rstride, t, D);
            rc = gnn_encode_rows(P, st, true, true);
            if (rc) break;
            if (h <= 32) {
                if (D <= 4) ps_adjoint_launch<4, 1>(PR, P, rec, rstride, t, al[e], beta, eps, st);
                else if (D <= 8) ps_adjoint_launch<8, 1>(PR, P, rec, rstride, t, al[e], beta, eps, st);
                else if (D <= 16) ps_adjoint_launch<16, 1>(PR, P, rec, rstride, t, al[e], beta, eps, st);
                else ps_adjoint_launch<32, 1>(PR, P, rec, rstride, t, al[e], beta, eps, st);
            } else {
                if (D <= 8) ps_adjoint_launch<8, 2>(PR, P, rec, rstride, t, al[e], beta, eps, st);
                else if (D <= 16) ps_adjoint_launch<16, 2>(PR, P, rec, rstride, t, al[e], beta, eps, st);
                else ps_adjoint_launch<32, 2>(PR, P, rec, rstride, t, al[e], beta, eps, st);
            }
            rc = fp_policy_backward(pol, tmp, st);
            if (rc) break;
            axpy_kernel<<<ab, 256, 0, st>>>(grad, tmp, pol->n_params);
        }
    }
    // the policy's own tables back to the per-episode encode (dyn = 0)
    ps_set_dyn_kernel<<<1, 256, 4 * n, st>>>(P, grad_rows, rstride, 0, D);
    if (rc == FP_OK) rc = gnn_encode_rows(P, st, true, true);
    cudaFreeAsync(tmp, st);
    cudaError_t err = cudaGetLastError();
    if (rc == FP_OK && err != cudaSuccess) { set_error(cudaGetErrorString(err)); return FP_ERR_CUDA; }
    return rc;
}
