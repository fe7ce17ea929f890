// Stage-II REINFORCE update on the GPU (flowplace/training.py:181-216 with the
// autodiff of flowplace/nn.py:62-224, re-derived for the factorised policy).
//
//   loss = sum_e [ alpha_e * sum_t lp_e,t + beta * sum_t ent_e,t ]
//   (alpha_e = -advantage_e / B_global, beta = -w_entropy / B_global; the
//   reference's per-episode loss at B = 1; imitation: alpha = -1/B, beta = 0)
//
// 1. pg_reduce: the rollout's SEL warp wrote, per episode, the gradients of
//    sum lp and sum ent w.r.t. the SEL logits s[v]; its PLC warp recorded each
//    decision.  plc_replay_kernel (fp_rollout.cuh) replays the records with
//    the episode's (alpha_e, beta) folded in from the first step, producing
//    the PLC table gradients (A, G rows via running per-device sums; M, w2,
//    b2) and the SEL terms, reduced over the CTA's episodes in episode order;
//    pg_final_kernel sums the CTA partials in CTA order: bitwise
//    deterministic, no atomics, no per-episode rows through HBM.
// 2. head backward (SEL head + paths, PLC tables), 3. GNN backward (K rounds
//    per encoder, gather-formulated message gradients), 4. weight gradients as
//    row-contractions X^T Y over vertices (outer kernel, job list), 5. SGD.
#include <algorithm>
#include <string>
#include <vector>

#include "fp_common.cuh"
#include "fp_policy.cuh"

namespace fp {

int plc_replay(const fp_problem *p, const fp_policy *pol, const double *rec, const double *gep,
               const int32_t *assign, const double *alpha, double beta, int B, double *scratch,
               int64_t *scratch_bytes, cudaStream_t st);  // fp_rollout.cu

__device__ __forceinline__ double lkd_t(double x, double s) { return x > 0.0 ? 1.0 : s; }
__device__ __forceinline__ double lk_t(double x, double s) { return x > 0.0 ? x : s * x; }

// ---------------------------------------------------------------------------
// head backward, warp per vertex, lane = hidden column
// ---------------------------------------------------------------------------
__global__ void head_bwd_kernel(DevPolicy P) {
    griddep_launch();  // PDL chain of the backward: launch latency hidden,
    griddep_wait();    // the predecessor complete before any access
    const int lane = lane_id();
    const int v = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int n = P.n, h = P.h;
    if (v >= n) return;
    const double s = P.slope;
    // ---- SEL: s[v] = leaky(emb @ W1 + b1) @ w2 + b2 ----
    const double *w1 = P.W(PR_SEL_H1_W), *w2 = P.W(PR_SEL_H2_W);
    const double dsv = P.ds[v];
    double dh[2] = {0.0, 0.0};
    for (int t = 0; t < 2; ++t) {
        const int j = lane + 32 * t;
        if (j < h) {
            dh[t] = dsv * w2[j] * lkd_t(P.hidpre[(size_t)v * h + j], s);
            P.dhid[(size_t)v * h + j] = dh[t];
        }
    }
    // demb_i = sum_j dhid_j W1[i][j], i < 4h
    for (int i0 = 0; i0 < 4 * h; i0 += 32) {
        const int i = i0 + lane;
        double acc = 0.0;
        for (int j = 0; j < h; ++j) {
            const double dj = __shfl_sync(FP_FULL_MASK, dh[j >> 5], j & 31);
            if (i < 4 * h) acc = fma(dj, w1[(size_t)i * h + j], acc);
        }
        if (i < 4 * h) P.demb[(size_t)v * 4 * h + i] = acc;
    }
    // ---- PLC: A = H@W1a + Z@W1d, G = H@W1b ----
    const double *w1p = P.W(PR_PLC_H1_W);
    double da[2] = {0.0, 0.0}, dg[2] = {0.0, 0.0};
    for (int t = 0; t < 2; ++t) {
        const int j = lane + 32 * t;
        if (j < h) { da[t] = P.dA[(size_t)v * h + j]; dg[t] = P.dG[(size_t)v * h + j]; }
    }
    for (int t = 0; t < 2; ++t) {
        const int j = lane + 32 * t;
        double hp = 0.0, zp = 0.0;
        for (int i = 0; i < h; ++i) {
            const double ai = __shfl_sync(FP_FULL_MASK, da[i >> 5], i & 31);
            const double gi = __shfl_sync(FP_FULL_MASK, dg[i >> 5], i & 31);
            if (j < h) {
                hp = fma(ai, w1p[(size_t)j * h + i], hp);
                hp = fma(gi, w1p[(size_t)(h + j) * h + i], hp);
                zp = fma(ai, w1p[(size_t)(3 * h + j) * h + i], zp);
            }
        }
        if (j < h) {
            P.dHn[1][(size_t)v * h + j] = hp;            // dH_plc (direct)
            P.dZ[(size_t)n * h + (size_t)v * h + j] = zp;  // dZp
        }
    }
}

// dH of each encoder's output: SEL = direct + path scatters (inverse paths);
// PLC = head part; shared encoder = both.
__global__ void path_gather_kernel(DevPolicy P) {
    griddep_launch();  // PDL chain of the backward: launch latency hidden,
    griddep_wait();    // the predecessor complete before any access
    const int lane = lane_id();
    const int u = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int n = P.n, h = P.h;
    if (u >= n) return;
    for (int j = lane; j < h; j += 32) {
        double acc = P.demb[(size_t)u * 4 * h + j];
        for (int q = P.ibp_ptr[u]; q < P.ibp_ptr[u + 1]; ++q)
            acc += P.demb[(size_t)P.ibp_idx[q] * 4 * h + h + j];
        for (int q = P.itp_ptr[u]; q < P.itp_ptr[u + 1]; ++q)
            acc += P.demb[(size_t)P.itp_idx[q] * 4 * h + 2 * h + j];
        P.dZ[(size_t)u * h + j] = P.demb[(size_t)u * 4 * h + 3 * h + j];  // dZs
        const double plc = P.dHn[1][(size_t)u * h + j];
        if (P.n_enc == 1) {
            P.dH[0][(size_t)u * h + j] = acc + plc;
        } else {
            P.dH[0][(size_t)u * h + j] = acc;
            P.dH[1][(size_t)u * h + j] = plc;
        }
    }
}

// ---------------------------------------------------------------------------
// GNN backward for one (encoder, round)
// ---------------------------------------------------------------------------
// node part: dU = dH (.) leaky'(U); dH_k(direct) = dU @ phi[0:dk]^T;
// dagg = dU @ phi[dk:dk+h]^T
__global__ void gnn_bwd_node(DevPolicy P, int e, int k) {
    griddep_launch();  // PDL chain of the backward: launch latency hidden,
    griddep_wait();    // the predecessor complete before any access
    const int lane = lane_id();
    const int v = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int n = P.n, h = P.h;
    if (v >= n) return;
    const int dk = k == 0 ? 7 : h;
    const double *phw = P.W(gnn_role(e, k, 2));
    double du[2] = {0.0, 0.0};
    for (int t = 0; t < 2; ++t) {
        const int j = lane + 32 * t;
        if (j < h) {
            du[t] = P.dH[e][(size_t)v * h + j] * lkd_t(P.U[e][k][(size_t)v * h + j], P.slope);
            P.dU[(size_t)v * h + j] = du[t];
        }
    }
    for (int t = 0; t < 2; ++t) {
        const int i = lane + 32 * t;  // output row i of phi
        double hd = 0.0, ag = 0.0;
        for (int j = 0; j < h; ++j) {
            const double dj = __shfl_sync(FP_FULL_MASK, du[j >> 5], j & 31);
            if (i < dk) hd = fma(dj, phw[(size_t)i * h + j], hd);
            if (i < h) ag = fma(dj, phw[(size_t)(dk + i) * h + j], ag);
        }
        if (i < h) {
            if (k > 0) P.dHn[0][(size_t)v * h + i] = hd;  // direct part of dH_k
            P.dagg[(size_t)v * h + i] = ag;
        }
    }
}

// message part, gather-formulated over the in-message list of v (each in
// message (w->v) has a mirror (v->w) with the same edge feature):
//   Ddst[v] = sum_{w->v} dagg[v] (.) leaky'(P[w] + Q[v] + e we + b)
//   Dsrc[v] = sum_{v->w} dagg[w] (.) leaky'(P[v] + Q[w] + e we + b)
//   De[v]   = sum_{w->v} e * dagg[v] (.) leaky'(...)
// then dH_k = dH_k(direct) + Dsrc @ Ws^T + Ddst @ Wd^T   (k > 0)
__global__ void gnn_bwd_msg(DevPolicy P, int e, int k) {
    griddep_launch();  // PDL chain of the backward: launch latency hidden,
    griddep_wait();    // the predecessor complete before any access
    const int lane = lane_id();
    const int v = blockIdx.x * 4 + (threadIdx.x >> 5);
    const int n = P.n, h = P.h;
    if (v >= n) return;
    const int dk = k == 0 ? 7 : h;
    const double *Hk = P.H[e][k];
    const double *psw = P.W(gnn_role(e, k, 0)), *psb = P.W(gnn_role(e, k, 1));
    const double s = P.slope;
    auto pq = [&](int x, int j, bool dst) {  // P[x][j] (dst=false) or Q[x][j]
        if (k > 0) return dst ? P.Qm[e][k][(size_t)x * h + j] : P.Pm[e][k][(size_t)x * h + j];
        double acc = 0.0;
        const int off = dst ? dk : 0;
        for (int i = 0; i < 7; ++i) acc = fma(Hk[x * 7 + i], psw[(off + i) * h + j], acc);
        return acc;
    };
    double Dd[2] = {0, 0}, Ds[2] = {0, 0}, De[2] = {0, 0};
    for (int t = 0; t < 2; ++t) {
        const int j = lane + 32 * t;
        if (j >= h) continue;
        const double we = psw[(2 * dk) * h + j], b = psb[j];
        const double pv = pq(v, j, false), qv = pq(v, j, true);
        const double gv = P.dagg[(size_t)v * h + j];
        for (int m = P.adj_ptr[v]; m < P.adj_ptr[v + 1]; ++m) {
            const int w = P.adj_nbr[m];
            const double ev = P.adj_e[m];
            const double din = gv * lkd_t(pq(w, j, false) + qv + ev * we + b, s);
            Dd[t] += din;
            De[t] += ev * din;
            Ds[t] += P.dagg[(size_t)w * h + j] * lkd_t(pv + pq(w, j, true) + ev * we + b, s);
        }
        P.Ddst[(size_t)v * h + j] = Dd[t];
        P.Dsrc[(size_t)v * h + j] = Ds[t];
        P.De[(size_t)v * h + j] = De[t];
    }
    if (k == 0) return;
    for (int t = 0; t < 2; ++t) {
        const int i = lane + 32 * t;
        double acc = 0.0;
        for (int j = 0; j < h; ++j) {
            const double sj = __shfl_sync(FP_FULL_MASK, Ds[j >> 5], j & 31);
            const double dj = __shfl_sync(FP_FULL_MASK, Dd[j >> 5], j & 31);
            if (i < h) {
                acc = fma(sj, psw[(size_t)i * h + j], acc);
                acc = fma(dj, psw[(size_t)(h + i) * h + j], acc);
            }
        }
        if (i < h) P.dHn[0][(size_t)v * h + i] += acc;
    }
}

__global__ void copy_kernel(double *dst, const double *src, int count) {
    griddep_launch();  // PDL chain of the backward: launch latency hidden,
    griddep_wait();    // the predecessor complete before any access
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) dst[i] = src[i];
}

// ---------------------------------------------------------------------------
// weight gradients: out[i][j] = sum_r X[r][xoff + i] * Y[r][j]  (X == nullptr:
// ones -> bias), rows r < R.  Each job writes one row block of one tensor.
// ---------------------------------------------------------------------------
struct OuterJob {
    const double *X;
    const double *Y;
    double *out;
    int ldx, xoff, K, ldy, rows, h;
};

// Weight gradients as row contractions out[i][j] = sum_r X[r][xoff+i] * Y[r][j]
// (X == NULL: a bias, X = 1).  One block per output row i: the 8 warps take
// contiguous row chunks (lane = column), and the chunk partials are summed in
// warp order -- deterministic, and the rows no longer form one long
// dependent chain per output element.
constexpr int kOuterWarps = 8;

__global__ void __launch_bounds__(kOuterWarps * 32) outer_kernel(const OuterJob *jobs) {
    griddep_launch();  // PDL chain of the backward: launch latency hidden,
    griddep_wait();    // the predecessor complete before any access
    __shared__ double part[kOuterWarps][64];
    const OuterJob J = jobs[blockIdx.y];
    const int i = blockIdx.x;
    if (i >= J.K) return;  // block-uniform
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int chunk = (J.rows + kOuterWarps - 1) / kOuterWarps;
    const int r0 = warp * chunk, r1 = min(J.rows, r0 + chunk);
    double acc0 = 0.0, acc1 = 0.0;
#pragma unroll 4
    for (int r = r0; r < r1; ++r) {
        const double x = J.X ? J.X[(size_t)r * J.ldx + J.xoff + i] : 1.0;
        const double *y = J.Y + (size_t)r * J.ldy;
        if (lane < J.h) acc0 = fma(x, y[lane], acc0);
        if (lane + 32 < J.h) acc1 = fma(x, y[lane + 32], acc1);
    }
    part[warp][lane] = acc0;
    part[warp][lane + 32] = acc1;
    __syncthreads();
    if (warp == 0) {
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int w = 0; w < kOuterWarps; ++w) { a0 += part[w][lane]; a1 += part[w][lane + 32]; }
        if (lane < J.h) J.out[(size_t)i * J.h + lane] = a0;
        if (lane + 32 < J.h) J.out[(size_t)i * J.h + lane + 32] = a1;
    }
}

// PLC small terms + SEL head2 (single block): dWy = dM @ W1c^T, dby = dc @ W1c^T,
// db1 = dc, dw2/db2 from the reduction, SEL w2 / b2.
__global__ void __launch_bounds__(256) small_bwd_kernel(DevPolicy P, double *grad) {
    griddep_launch();  // PDL chain of the backward: launch latency hidden,
    griddep_wait();    // the predecessor complete before any access
    __shared__ double part[8][65];  // [warp][column | sum of ds]
    const int h = P.h, n = P.n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double *dc = P.dsmall, *dM = P.dsmall + h, *dw2 = P.dsmall + 6 * h;
    const double db2 = P.dsmall[7 * h];
    const double *w1p = P.W(PR_PLC_H1_W);
    for (int idx = threadIdx.x; idx < 6 * h; idx += blockDim.x) {
        const int r = idx / h, i = idx - r * h;  // r < 5: Wy row r; r == 5: by
        const double *src = r < 5 ? dM + r * h : dc;
        double acc = 0.0;
        for (int j = 0; j < h; ++j) acc = fma(src[j], w1p[(size_t)(2 * h + i) * h + j], acc);
        if (r < 5) grad[P.off[PR_PLC_Y_W] + r * h + i] = acc;
        else grad[P.off[PR_PLC_Y_B] + i] = acc;
    }
    for (int j = threadIdx.x; j < h; j += blockDim.x) {
        grad[P.off[PR_PLC_H1_B] + j] = dc[j];
        grad[P.off[PR_PLC_H2_W] + j] = dw2[j];
    }
    // SEL head2: dw2[j] = sum_v ds_v * leaky(hidpre[v][j]), db2 = sum_v ds_v: the
    // 8 warps take contiguous vertex chunks (lane = column), then the chunk
    // partials are summed in warp order (deterministic)
    const int chunk = (n + 7) / 8, v0 = warp * chunk, v1 = min(n, v0 + chunk);
    double a0 = 0.0, a1 = 0.0, sd = 0.0;
    for (int v = v0; v < v1; ++v) {
        const double dsv = P.ds[v];
        if (lane < h) a0 = fma(dsv, lk_t(P.hidpre[(size_t)v * h + lane], P.slope), a0);
        if (lane + 32 < h) a1 = fma(dsv, lk_t(P.hidpre[(size_t)v * h + lane + 32], P.slope), a1);
        sd += dsv;
    }
    part[warp][lane] = a0;
    part[warp][lane + 32] = a1;
    if (lane == 0) part[warp][64] = sd;
    __syncthreads();
    if (warp == 0) {
        double b0 = 0.0, b1 = 0.0, bs = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) { b0 += part[w][lane]; b1 += part[w][lane + 32]; bs += part[w][64]; }
        if (lane < h) grad[P.off[PR_SEL_H2_W] + lane] = b0;
        if (lane + 32 < h) grad[P.off[PR_SEL_H2_W] + lane + 32] = b1;
        if (lane == 0) {
            grad[P.off[PR_PLC_H2_B]] = db2;
            grad[P.off[PR_SEL_H2_B]] = bs;
        }
    }
}

__global__ void sgd_kernel(double *params, const double *grad, int64_t count, double lr,
                           const int32_t *skip) {
    griddep_wait();  // (PDL) the gradient complete
    if (skip && *skip) return;  // a failed rollout in this (or an earlier) batch: no update
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) params[i] = params[i] - lr * grad[i];
}

}  // namespace fp

using namespace fp;

struct fp_train_state {
    fp::OuterJob *jobs_dev = nullptr;
    std::vector<std::vector<fp::OuterJob>> batches;  // one launch per stage
    std::vector<int> stage_offset;
    double *bound_grad = nullptr;
    const double *bound_params = nullptr;
    void *replay = nullptr;        // fp_pg_reduce scratch: episode-row slab + CTA partials
    int64_t replay_bytes = 0;
};

void fp_train_state_free(fp_train_state *ts) {
    if (!ts) return;
    if (ts->jobs_dev) cudaFree(ts->jobs_dev);
    if (ts->replay) cudaFree(ts->replay);
    delete ts;
}

namespace fp {

static void add_job(std::vector<OuterJob> &v, const double *X, int ldx, int xoff, int K,
                    const double *Y, int ldy, int rows, int h, double *out) {
    v.push_back(OuterJob{X, Y, out, ldx, xoff, K, ldy, rows, h});
}

// Build the outer-product job lists for a given gradient buffer.
static int build_jobs(fp_policy *pol, double *grad) {
    DevPolicy &P = pol->dev;
    const int n = P.n, h = P.h;
    auto *ts = pol->train;
    ts->batches.clear();
    auto G = [&](int role) { return grad + P.off[role]; };
    if (P.off[PR_PLC_Y_W] != P.off[PR_PLC_Y_B] + h) {
        set_error("flat layout must store plc.y.b directly before plc.y.w");
        return FP_ERR_INVALID;
    }
    // stage 0: dc = sum_v dA[v] (read by the small kernel and the W1c job)
    std::vector<OuterJob> pre;
    add_job(pre, nullptr, 0, 0, 1, P.dA, h, n, h, P.dsmall);
    ts->batches.push_back(pre);
    // stage 1: heads
    std::vector<OuterJob> head;
    const double *Hsel = P.H[0][P.K], *Hplc = P.H[P.n_enc - 1][P.K];
    add_job(head, P.emb, 4 * h, 0, 4 * h, P.dhid, h, n, h, G(PR_SEL_H1_W));
    add_job(head, nullptr, 0, 0, 1, P.dhid, h, n, h, G(PR_SEL_H1_B));
    add_job(head, P.x, 5, 0, 5, P.dZ, h, n, h, G(PR_SEL_Z_W));
    add_job(head, nullptr, 0, 0, 1, P.dZ, h, n, h, G(PR_SEL_Z_B));
    add_job(head, Hplc, h, 0, h, P.dA, h, n, h, G(PR_PLC_H1_W));
    add_job(head, Hplc, h, 0, h, P.dG, h, n, h, G(PR_PLC_H1_W) + (size_t)h * h);
    // W1c rows = [by ; Wy]^T [dc ; dM]: X = rows of [by; Wy] (flat order b, w)
    add_job(head, P.params + P.off[PR_PLC_Y_B], h, 0, h, P.dsmall, h, 6, h,
            G(PR_PLC_H1_W) + (size_t)2 * h * h);
    add_job(head, P.Zp, h, 0, h, P.dA, h, n, h, G(PR_PLC_H1_W) + (size_t)3 * h * h);
    add_job(head, P.x, 5, 0, 5, P.dZ + (size_t)n * h, h, n, h, G(PR_PLC_Z_W));
    add_job(head, nullptr, 0, 0, 1, P.dZ + (size_t)n * h, h, n, h, G(PR_PLC_Z_B));
    ts->batches.push_back(head);
    // GNN stages: (e, k) in backward order
    for (int e = 0; e < P.n_enc; ++e)
        for (int k = P.K - 1; k >= 0; --k) {
            std::vector<OuterJob> js;
            const int dk = k == 0 ? 7 : h;
            add_job(js, P.H[e][k], dk, 0, dk, P.dU, h, n, h, G(gnn_role(e, k, 2)));
            add_job(js, P.AG[e][k], h, 0, h, P.dU, h, n, h, G(gnn_role(e, k, 2)) + (size_t)dk * h);
            add_job(js, nullptr, 0, 0, 1, P.dU, h, n, h, G(gnn_role(e, k, 3)));
            add_job(js, P.H[e][k], dk, 0, dk, P.Dsrc, h, n, h, G(gnn_role(e, k, 0)));
            add_job(js, P.H[e][k], dk, 0, dk, P.Ddst, h, n, h, G(gnn_role(e, k, 0)) + (size_t)dk * h);
            add_job(js, nullptr, 0, 0, 1, P.De, h, n, h, G(gnn_role(e, k, 0)) + (size_t)2 * dk * h);
            add_job(js, nullptr, 0, 0, 1, P.Ddst, h, n, h, G(gnn_role(e, k, 1)));
            ts->batches.push_back(js);
        }
    size_t total = 0;
    ts->stage_offset.clear();
    for (auto &b : ts->batches) { ts->stage_offset.push_back((int)total); total += b.size(); }
    if (ts->jobs_dev) cudaFree(ts->jobs_dev);
    if (cudaMalloc(&ts->jobs_dev, total * sizeof(OuterJob)) != cudaSuccess) {
        set_error("cudaMalloc failed for job list");
        return FP_ERR_CUDA;
    }
    std::vector<OuterJob> flat;
    for (auto &b : ts->batches) flat.insert(flat.end(), b.begin(), b.end());
    cudaMemcpy(ts->jobs_dev, flat.data(), total * sizeof(OuterJob), cudaMemcpyHostToDevice);
    ts->bound_grad = grad;
    ts->bound_params = P.params;
    return FP_OK;
}

static void launch_outer(fp_train_state *ts, int stage, cudaStream_t st) {
    const auto &b = ts->batches[stage];
    int maxk = 0;
    for (auto &j : b) maxk = std::max(maxk, j.K);
    dim3 grid(maxk, (unsigned)b.size());
    launch_pdl(outer_kernel, grid, dim3(kOuterWarps * 32), 0, st,
               (const OuterJob *)(ts->jobs_dev + ts->stage_offset[stage]));
}

}  // namespace fp

extern "C" {

int fp_pg_reduce(fp_policy *pol, const double *grad_rows, const double *grad_ep,
                 const int32_t *assign, const double *alpha, double beta, int32_t B, void *stream) {
    if (!pol || !grad_rows || !grad_ep || !assign || !alpha || B <= 0) {
        set_error("bad pg_reduce arguments");
        return FP_ERR_INVALID;
    }
    if (!pol->train) pol->train = new fp_train_state();
    auto *ts = pol->train;
    cudaStream_t st = (cudaStream_t)stream;
    int64_t need = 0;
    int rc = plc_replay(pol->problem, pol, grad_rows, grad_ep, assign, alpha, beta, B, nullptr,
                        &need, st);
    if (rc) return rc;
    if (ts->replay_bytes < need) {  // grown on demand, kept for the next updates
        if (ts->replay) { cudaStreamSynchronize(st); cudaFree(ts->replay); }
        ts->replay = nullptr;
        ts->replay_bytes = 0;
        if (cudaMalloc(&ts->replay, need) != cudaSuccess) {
            set_error("cudaMalloc failed for the REINFORCE replay scratch");
            return FP_ERR_CUDA;
        }
        ts->replay_bytes = need;
    }
    return plc_replay(pol->problem, pol, grad_rows, grad_ep, assign, alpha, beta, B,
                      (double *)ts->replay, nullptr, st);
}

int fp_policy_backward(fp_policy *pol, double *grad, void *stream) {
    if (!pol || !grad) { set_error("null argument"); return FP_ERR_INVALID; }
    DevPolicy &P = pol->dev;
    if (!P.params) { set_error("fp_policy_prepare must run before backward"); return FP_ERR_INVALID; }
    if (P.forest) { set_error("backward needs explicit SEL path lists (policy built in forest form)"); return FP_ERR_UNSUPPORTED; }
    if (P.tc) { set_error("backward needs the fp64 encoder (the bf16 tensor-core encoder is forward only)"); return FP_ERR_UNSUPPORTED; }
    if (!pol->train) pol->train = new fp_train_state();
    auto *ts = pol->train;
    if (ts->bound_grad != grad || ts->bound_params != P.params || ts->batches.empty()) {
        int rc = build_jobs(pol, grad);
        if (rc) return rc;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int n = P.n, h = P.h;
    const int g4 = (n + 3) / 4;
    cudaMemsetAsync(grad, 0, sizeof(double) * pol->n_params, st);
    launch_pdl(head_bwd_kernel, dim3(g4), dim3(128), 0, st, P);
    launch_pdl(path_gather_kernel, dim3(g4), dim3(128), 0, st, P);
    launch_outer(ts, 0, st);  // dc
    launch_pdl(small_bwd_kernel, dim3(1), dim3(256), 0, st, P, grad);
    launch_outer(ts, 1, st);  // head weight gradients
    int stage = 2;
    for (int e = 0; e < P.n_enc; ++e)
        for (int k = P.K - 1; k >= 0; --k) {
            launch_pdl(gnn_bwd_node, dim3(g4), dim3(128), 0, st, P, e, k);
            launch_pdl(gnn_bwd_msg, dim3(g4), dim3(128), 0, st, P, e, k);
            launch_outer(ts, stage++, st);
            if (k > 0)
                launch_pdl(copy_kernel, dim3((n * h + 255) / 256), dim3(256), 0, st, P.dH[e],
                           (const double *)P.dHn[0], n * h);
        }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FP_ERR_CUDA; }
    return FP_OK;
}

int fp_sgd_step_masked(double *params, const double *grad, int64_t count, double lr,
                       const int32_t *skip, void *stream) {
    if (!params || !grad || count < 0) { set_error("bad sgd arguments"); return FP_ERR_INVALID; }
    if (count == 0) return FP_OK;
    launch_pdl(sgd_kernel, dim3((unsigned)((count + 255) / 256)), dim3(256), 0, (cudaStream_t)stream,
               params, grad, count, lr, skip);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FP_ERR_CUDA; }
    return FP_OK;
}

int fp_sgd_step(double *params, const double *grad, int64_t count, double lr, void *stream) {
    return fp_sgd_step_masked(params, grad, count, lr, nullptr, stream);
}

}  // extern "C"
