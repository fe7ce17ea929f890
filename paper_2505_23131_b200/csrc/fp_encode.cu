// GNN encoder + head-table precompute (one parameter snapshot), fp64.
//
// Reference math (flowplace/policy.py:149-223), re-factored for the GPU:
//   * psi is split by input block: [H[src] | H[dst] | e] @ psi.w =
//     H[src] @ Ws + H[dst] @ Wd + e * we, so a message is
//     leaky(P[src] + Q[dst] + e*we + b) with P = H @ Ws, Q = H @ Wd computed
//     once per vertex (fused into the previous round's kernel) instead of once
//     per message; round 0 (7 input columns) recomputes P/Q on the fly.
//   * Aggregation (policy.py:166 segment_sum) is a CSR-by-destination gather,
//     one warp per destination, lane = hidden column: each message row is a
//     coalesced 256-byte load of P[src].
//   * Head tables: SEL logits s[v] for every vertex and
//     the PLC tables A = H@W1a + Z@W1d, G = H@W1b, M = Wy@W1c,
//     c = by@W1c + b1, so the rollout never re-runs a dense layer per step.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "fp_common.cuh"
#include "fp_policy.cuh"

namespace fp {

constexpr int kEncWarps = 4;

__device__ __forceinline__ double leaky(double x, double s) { return x > 0.0 ? x : s * x; }

// broadcast element i of a lane-distributed vector (HPL columns per lane)
template <int HPL>
__device__ __forceinline__ double bcast(const double (&v)[HPL], int i) {
    double r = 0.0;
#pragma unroll
    for (int q = 0; q < HPL; ++q) {
        const double t = __shfl_sync(FP_FULL_MASK, v[q], i & 31);
        if ((i >> 5) == q) r = t;
    }
    return r;
}

template <int HPL>
__global__ void __launch_bounds__(kEncWarps * 32)
encode_round_kernel(DevPolicy P, int k, int last) {
    const int lane = lane_id();
    const int gw = blockIdx.x * kEncWarps + (threadIdx.x >> 5);
    const int n = P.n, h = P.h;
    const int e = gw / max(n, 1), v = gw - e * n;
    if (e >= P.n_enc || n == 0) return;
    const int dk = k == 0 ? 7 : h;
    const double *Hk = P.H[e][k];
    const double *psw = P.W(gnn_role(e, k, 0)), *psb = P.W(gnn_role(e, k, 1));
    const double *phw = P.W(gnn_role(e, k, 2)), *phb = P.W(gnn_role(e, k, 3));
    const double s = P.slope;

    double q[HPL], we[HPL], bb[HPL], agg[HPL];
#pragma unroll
    for (int t = 0; t < HPL; ++t) {
        const int j = lane + 32 * t;
        q[t] = we[t] = bb[t] = agg[t] = 0.0;
        if (j < h) {
            if (k == 0) {
                double acc = 0.0;
                for (int i = 0; i < 7; ++i) acc = fma(Hk[v * 7 + i], psw[(dk + i) * h + j], acc);
                q[t] = acc;
            } else {
                q[t] = P.Qm[e][k][(size_t)v * h + j];
            }
            we[t] = psw[(2 * dk) * h + j];
            bb[t] = psb[j];
        }
    }
    for (int m = P.adj_ptr[v]; m < P.adj_ptr[v + 1]; ++m) {
        const int w = P.adj_nbr[m];
        const double ev = P.adj_e[m];
#pragma unroll
        for (int t = 0; t < HPL; ++t) {
            const int j = lane + 32 * t;
            if (j >= h) continue;
            double p;
            if (k == 0) {
                p = 0.0;
                for (int i = 0; i < 7; ++i) p = fma(Hk[w * 7 + i], psw[i * h + j], p);
            } else {
                p = P.Pm[e][k][(size_t)w * h + j];
            }
            agg[t] += leaky(p + q[t] + ev * we[t] + bb[t], s);
        }
    }
    // update: U = [H | agg] @ phi.w + phi.b
    double u[HPL];
#pragma unroll
    for (int t = 0; t < HPL; ++t) u[t] = 0.0;
    for (int i = 0; i < dk; ++i) {
        const double hv = Hk[(size_t)v * dk + i];
#pragma unroll
        for (int t = 0; t < HPL; ++t) {
            const int j = lane + 32 * t;
            if (j < h) u[t] = fma(hv, phw[i * h + j], u[t]);
        }
    }
    for (int i = 0; i < h; ++i) {
        const double a = bcast<HPL>(agg, i);
#pragma unroll
        for (int t = 0; t < HPL; ++t) {
            const int j = lane + 32 * t;
            if (j < h) u[t] = fma(a, phw[(dk + i) * h + j], u[t]);
        }
    }
    double hn[HPL];
#pragma unroll
    for (int t = 0; t < HPL; ++t) {
        const int j = lane + 32 * t;
        hn[t] = 0.0;
        if (j < h) {
            u[t] += phb[j];
            hn[t] = leaky(u[t], s);
            P.U[e][k][(size_t)v * h + j] = u[t];
            P.AG[e][k][(size_t)v * h + j] = agg[t];
            P.H[e][k + 1][(size_t)v * h + j] = hn[t];
        }
    }
    if (!last) {
        const double *nw = P.W(gnn_role(e, k + 1, 0));
        double pp[HPL], qq[HPL];
#pragma unroll
        for (int t = 0; t < HPL; ++t) pp[t] = qq[t] = 0.0;
        for (int i = 0; i < h; ++i) {
            const double a = bcast<HPL>(hn, i);
#pragma unroll
            for (int t = 0; t < HPL; ++t) {
                const int j = lane + 32 * t;
                if (j < h) {
                    pp[t] = fma(a, nw[i * h + j], pp[t]);
                    qq[t] = fma(a, nw[(h + i) * h + j], qq[t]);
                }
            }
        }
#pragma unroll
        for (int t = 0; t < HPL; ++t) {
            const int j = lane + 32 * t;
            if (j < h) {
                P.Pm[e][k + 1][(size_t)v * h + j] = pp[t];
                P.Qm[e][k + 1][(size_t)v * h + j] = qq[t];
            }
        }
        return;
    }
    // ---- last round: per-vertex head rows ----
    const bool feeds_sel = e == 0;
    const bool feeds_plc = P.n_enc == 1 || e == 1;
    const double *x = P.x + (size_t)v * 5;
    if (feeds_sel) {
        const double *zw = P.W(PR_SEL_Z_W), *zb = P.W(PR_SEL_Z_B);
#pragma unroll
        for (int t = 0; t < HPL; ++t) {
            const int j = lane + 32 * t;
            if (j >= h) continue;
            double z = 0.0;
            for (int i = 0; i < 5; ++i) z = fma(x[i], zw[i * h + j], z);
            P.Zs[(size_t)v * h + j] = z + zb[j];
        }
    }
    if (feeds_plc) {
        const double *zw = P.W(PR_PLC_Z_W), *zb = P.W(PR_PLC_Z_B), *w1 = P.W(PR_PLC_H1_W);
        double z[HPL], a[HPL], g[HPL];
#pragma unroll
        for (int t = 0; t < HPL; ++t) {
            const int j = lane + 32 * t;
            z[t] = a[t] = g[t] = 0.0;
            if (j >= h) continue;
            double acc = 0.0;
            for (int i = 0; i < 5; ++i) acc = fma(x[i], zw[i * h + j], acc);
            z[t] = acc + zb[j];
            P.Zp[(size_t)v * h + j] = z[t];
        }
        for (int i = 0; i < h; ++i) {
            const double hv = bcast<HPL>(hn, i), zv = bcast<HPL>(z, i);
#pragma unroll
            for (int t = 0; t < HPL; ++t) {
                const int j = lane + 32 * t;
                if (j >= h) continue;
                a[t] = fma(hv, w1[i * h + j], a[t]);
                a[t] = fma(zv, w1[(3 * h + i) * h + j], a[t]);
                g[t] = fma(hv, w1[(h + i) * h + j], g[t]);
            }
        }
#pragma unroll
        for (int t = 0; t < HPL; ++t) {
            const int j = lane + 32 * t;
            if (j < h) {
                P.A[(size_t)v * h + j] = a[t];
                P.G[(size_t)v * h + j] = g[t];
            }
        }
    }
}

// Forest-form path sums (large graphs): S(v) = sum of H over path(v), by
// pointer jumping -- after round r, S(v) covers the first 2^(r+1) vertices of
// path(v) and J(v) points 2^(r+1) vertices down it (-1 past the end).
// Round 0 reads H and the next arrays; round r >= 1 ping-pongs PS/PJ.
// Pure gather-add over n x h doubles per round (HBM / L2 bound).
__global__ void path_jump_kernel(DevPolicy P, int r) {
    const int which = blockIdx.y;  // 0 = b-paths, 1 = t-paths
    const int n = P.n, h = P.h;
    const double *Sin = r == 0 ? P.H[0][P.K] : P.PS[which][(r - 1) & 1];
    const int *Jin = r == 0 ? P.nxt[which] : P.PJ[which][(r - 1) & 1];
    double *Sout = P.PS[which][r & 1];
    int *Jout = P.PJ[which][r & 1];
    const int64_t total = (int64_t)n * h;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int v = (int)(i / h), j = (int)(i - (int64_t)v * h);
        const int w = Jin[v];
        Sout[i] = w >= 0 ? Sin[i] + Sin[(size_t)w * h + j] : Sin[i];
        if (j == 0) Jout[v] = w >= 0 ? Jin[w] : -1;
    }
}

// SEL head over every vertex: s[v] = head(H[v] | sum_bpath H | sum_tpath H | Z[v]).
template <int HPL>
__global__ void __launch_bounds__(kEncWarps * 32) encode_sel_kernel(DevPolicy P) {
    const int lane = lane_id();
    const int v = blockIdx.x * kEncWarps + (threadIdx.x >> 5);
    const int n = P.n, h = P.h;
    const double s = P.slope;
    const double *Hs = P.H[0][P.K];
    if (blockIdx.x == 0 && (threadIdx.x >> 5) == 0) {
        // M = Wy @ W1c (5 x h), c = by @ W1c + b1  (PLC, policy.py:218-222)
        const double *yw = P.W(PR_PLC_Y_W), *yb = P.W(PR_PLC_Y_B), *w1 = P.W(PR_PLC_H1_W),
                     *b1 = P.W(PR_PLC_H1_B);
        for (int j = lane; j < h; j += 32) {
            for (int r = 0; r < 5; ++r) {
                double acc = 0.0;
                for (int i = 0; i < h; ++i) acc = fma(yw[r * h + i], w1[(2 * h + i) * h + j], acc);
                P.M[r * h + j] = acc;
            }
            double acc = 0.0;
            for (int i = 0; i < h; ++i) acc = fma(yb[i], w1[(2 * h + i) * h + j], acc);
            P.c[j] = acc + b1[j];
        }
    }
    if (v >= n) return;
    double em[4][HPL];
#pragma unroll
    for (int t = 0; t < HPL; ++t) {
        const int j = lane + 32 * t;
        em[0][t] = em[1][t] = em[2][t] = em[3][t] = 0.0;
        if (j >= h) continue;
        em[0][t] = Hs[(size_t)v * h + j];
        double hb = 0.0, ht = 0.0;
        if (P.forest) {
            const int rr = P.jump_rounds;
            hb = rr == 0 ? em[0][t] : P.PS[0][(rr - 1) & 1][(size_t)v * h + j];
            ht = rr == 0 ? em[0][t] : P.PS[1][(rr - 1) & 1][(size_t)v * h + j];
        } else {
            for (int p = P.bp_ptr[v]; p < P.bp_ptr[v + 1]; ++p)
                hb += Hs[(size_t)P.bp_idx[p] * h + j];
            for (int p = P.tp_ptr[v]; p < P.tp_ptr[v + 1]; ++p)
                ht += Hs[(size_t)P.tp_idx[p] * h + j];
        }
        em[1][t] = hb;
        em[2][t] = ht;
        em[3][t] = P.Zs[(size_t)v * h + j];
        for (int b = 0; b < 4; ++b) P.emb[(size_t)v * 4 * h + b * h + j] = em[b][t];
    }
    const double *w1 = P.W(PR_SEL_H1_W), *b1 = P.W(PR_SEL_H1_B), *w2 = P.W(PR_SEL_H2_W),
                 *b2 = P.W(PR_SEL_H2_B);
    double acc[HPL];
#pragma unroll
    for (int t = 0; t < HPL; ++t) acc[t] = 0.0;
    for (int b = 0; b < 4; ++b)
        for (int i = 0; i < h; ++i) {
            const double ev = bcast<HPL>(em[b], i);
#pragma unroll
            for (int t = 0; t < HPL; ++t) {
                const int j = lane + 32 * t;
                if (j < h) acc[t] = fma(ev, w1[(b * h + i) * h + j], acc[t]);
            }
        }
    double part = 0.0;
#pragma unroll
    for (int t = 0; t < HPL; ++t) {
        const int j = lane + 32 * t;
        if (j < h) {
            const double pre = acc[t] + b1[j];
            P.hidpre[(size_t)v * h + j] = pre;
            part = fma(leaky(pre, s), w2[j], part);
        }
    }
    part = warp_sum(part);
    if (lane == 0) P.s[v] = part + b2[0];
}

#define FP_CUDA_RET(call)                                                             \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess) {                                                      \
            set_error(std::string(#call) + ": " + cudaGetErrorString(e_));            \
            return FP_ERR_CUDA;                                                       \
        }                                                                             \
    } while (0)

int policy_prepare(fp_policy *pol, const double *params, cudaStream_t st) {
    DevPolicy &P = pol->dev;
    P.params = params;
    if (P.n == 0) return FP_OK;
    const int rows = P.n_enc * P.n;
    const int grid = (rows + kEncWarps - 1) / kEncWarps;
    for (int k = 0; k < P.K; ++k) {
        if (P.h <= 32)
            encode_round_kernel<1><<<grid, kEncWarps * 32, 0, st>>>(P, k, k == P.K - 1);
        else
            encode_round_kernel<2><<<grid, kEncWarps * 32, 0, st>>>(P, k, k == P.K - 1);
        FP_CUDA_RET(cudaGetLastError());
    }
    if (P.forest)
        for (int r = 0; r < P.jump_rounds; ++r) {
            const int64_t total = (int64_t)P.n * P.h;
            const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
            path_jump_kernel<<<dim3(blocks, 2), 256, 0, st>>>(P, r);
            FP_CUDA_RET(cudaGetLastError());
        }
    const int g2 = (P.n + kEncWarps - 1) / kEncWarps;
    if (P.h <= 32)
        encode_sel_kernel<1><<<g2, kEncWarps * 32, 0, st>>>(P);
    else
        encode_sel_kernel<2><<<g2, kEncWarps * 32, 0, st>>>(P);
    FP_CUDA_RET(cudaGetLastError());
    return FP_OK;
}

}  // namespace fp

using namespace fp;

extern "C" {

int fp_policy_create(const fp_problem *p, const fp_policy_desc *desc, fp_policy **out) {
    if (!p || !desc || !out) { set_error("null argument"); return FP_ERR_INVALID; }
    const int n = p->dev.n, h = desc->hidden, K = desc->k_rounds;
    if (h < 1 || h > kMaxHidden || K < 1 || K > kMaxRounds) {
        set_error("hidden must be in [1, 64] and k_rounds in [1, 8]");
        return FP_ERR_UNSUPPORTED;
    }
    const int n_enc = desc->shared_encoder ? 1 : 2;
    for (int r = 0; r < PR_COUNT; ++r) {
        int64_t o = desc->param_offsets[r];
        bool needed = r >= PR_SEL_Z_W;
        if (r < PR_SEL_Z_W) {
            const int e = r / (kMaxRounds * 4), k = (r / 4) % kMaxRounds;
            needed = e < n_enc && k < K;
        }
        if (needed && (o < 0 || o >= desc->n_params)) {
            set_error("missing parameter offset for role " + std::to_string(r));
            return FP_ERR_INVALID;
        }
    }
    const int M = desc->adj_ptr[n];
    const bool forest = desc->bpath_ptr == nullptr;
    if (forest && (!desc->bnext || !desc->tnext)) {
        set_error("need either path lists or next arrays");
        return FP_ERR_INVALID;
    }
    const int Lb = forest ? 0 : desc->bpath_ptr[n], Lt = forest ? 0 : desc->tpath_ptr[n];
    int jump_rounds = 0;
    if (forest) {
        // longest path (vertices) over both forests -> ceil(log2) jumping rounds
        int64_t longest = 1;
        for (const int32_t *nx : {desc->bnext, desc->tnext}) {
            std::vector<int> len(n, 0), stack;
            for (int v = 0; v < n; ++v) {
                int u = v;
                while (u >= 0 && len[u] == 0) {
                    stack.push_back(u);
                    u = nx[u];
                    if ((int)stack.size() > n) { set_error("next arrays contain a cycle"); return FP_ERR_INVALID; }
                }
                int base = u >= 0 ? len[u] : 0;
                while (!stack.empty()) { len[stack.back()] = ++base; stack.pop_back(); }
                longest = std::max<int64_t>(longest, len[v]);
            }
        }
        while ((int64_t(1) << jump_rounds) < longest) ++jump_rounds;
    }
    // inverse path lists: for u, the vertices v whose path contains u
    auto invert = [&](const int32_t *ptr, const int32_t *idx, std::vector<int> &iptr,
                      std::vector<int> &iidx) {
        iptr.assign(n + 1, 0);
        for (int i = 0; i < ptr[n]; ++i) iptr[idx[i] + 1]++;
        for (int u = 0; u < n; ++u) iptr[u + 1] += iptr[u];
        iidx.resize(ptr[n]);
        std::vector<int> fill(iptr.begin(), iptr.end() - 1);
        for (int v = 0; v < n; ++v)
            for (int i = ptr[v]; i < ptr[v + 1]; ++i) iidx[fill[idx[i]]++] = v;
    };
    std::vector<int> ibp(n + 1, 0), ibi, itp(n + 1, 0), iti;
    if (!forest) {
        invert(desc->bpath_ptr, desc->bpath_idx, ibp, ibi);
        invert(desc->tpath_ptr, desc->tpath_idx, itp, iti);
    }

    // arena layout
    std::vector<std::pair<size_t, size_t>> parts;  // (offset, bytes)
    size_t size = 0;
    auto take = [&](size_t bytes) {
        size = (size + 255) / 256 * 256;
        size_t o = size;
        size += std::max<size_t>(bytes, 8);
        return o;
    };
    const size_t nh = (size_t)std::max(n, 1) * h * 8;
    size_t o_x = take((size_t)n * 5 * 8), o_ap = take((size_t)(n + 1) * 4),
           o_an = take((size_t)M * 4), o_ae = take((size_t)M * 8),
           o_bp = take((size_t)(n + 1) * 4), o_bi = take((size_t)Lb * 4),
           o_tp = take((size_t)(n + 1) * 4), o_ti = take((size_t)Lt * 4),
           o_ibp = take((size_t)(n + 1) * 4), o_ibi = take((size_t)Lb * 4),
           o_itp = take((size_t)(n + 1) * 4), o_iti = take((size_t)Lt * 4);
    size_t o_nx[2] = {0, 0}, o_PS[2][2] = {{0, 0}, {0, 0}}, o_PJ[2][2] = {{0, 0}, {0, 0}};
    if (forest)
        for (int w = 0; w < 2; ++w) {
            o_nx[w] = take((size_t)n * 4);
            for (int q = 0; q < 2; ++q) { o_PS[w][q] = take(nh); o_PJ[w][q] = take((size_t)n * 4); }
        }
    size_t o_H[2][kMaxRounds + 1], o_P[2][kMaxRounds], o_Q[2][kMaxRounds], o_U[2][kMaxRounds],
        o_AG[2][kMaxRounds];
    for (int e = 0; e < n_enc; ++e) {
        o_H[e][0] = take((size_t)std::max(n, 1) * 7 * 8);
        for (int k = 0; k < K; ++k) {
            o_H[e][k + 1] = take(nh);
            o_P[e][k] = take(nh);
            o_Q[e][k] = take(nh);
            o_U[e][k] = take(nh);
            o_AG[e][k] = take(nh);
        }
    }
    size_t o_Zs = take(nh), o_emb = take(nh * 4), o_hp = take(nh), o_s = take((size_t)n * 8),
           o_Zp = take(nh), o_A = take(nh), o_G = take(nh), o_M = take((size_t)5 * h * 8),
           o_c = take((size_t)h * 8);
    size_t o_dH[2], o_dHn[2];
    for (int e = 0; e < 2; ++e) { o_dH[e] = take(nh); o_dHn[e] = take(nh); }
    size_t o_dU = take(nh), o_Ds = take(nh), o_Dd = take(nh), o_dagg = take(nh),
           o_De = take(nh), o_dhid = take(nh), o_demb = take(nh * 4), o_dZ = take(nh * 2),
           o_ds = take((size_t)n * 8), o_dA = take(nh), o_dG = take(nh),
           o_dsm = take((size_t)(16 * h + 64) * 8);
    const int prow = 16;  // episode chunks of the deterministic reduction
    size_t o_part = take((size_t)prow * ((size_t)std::max(n, 1) * (2 * h + 1) + 16 * h + 64) * 8);

    fp_policy *pol = new fp_policy();
    pol->problem = p;
    pol->n_params = desc->n_params;
    if (cudaMalloc(&pol->arena, size) != cudaSuccess) {
        delete pol;
        set_error("cudaMalloc failed for policy arena");
        return FP_ERR_CUDA;
    }
    uint8_t *b = (uint8_t *)pol->arena;
    cudaMemset(b, 0, size);
    auto up = [&](size_t o, const void *src, size_t bytes) {
        if (bytes) cudaMemcpy(b + o, src, bytes, cudaMemcpyHostToDevice);
    };
    up(o_x, desc->x_static, (size_t)n * 5 * 8);
    up(o_ap, desc->adj_ptr, (size_t)(n + 1) * 4);
    up(o_an, desc->adj_src, (size_t)M * 4);
    up(o_ae, desc->adj_edge, (size_t)M * 8);
    if (!forest) {
        up(o_bp, desc->bpath_ptr, (size_t)(n + 1) * 4);
        up(o_bi, desc->bpath_idx, (size_t)Lb * 4);
        up(o_tp, desc->tpath_ptr, (size_t)(n + 1) * 4);
        up(o_ti, desc->tpath_idx, (size_t)Lt * 4);
    } else {
        up(o_nx[0], desc->bnext, (size_t)n * 4);
        up(o_nx[1], desc->tnext, (size_t)n * 4);
    }
    up(o_ibp, ibp.data(), (size_t)(n + 1) * 4);
    up(o_ibi, ibi.data(), (size_t)Lb * 4);
    up(o_itp, itp.data(), (size_t)(n + 1) * 4);
    up(o_iti, iti.data(), (size_t)Lt * 4);
    // H0 = [x_static | dyn = 0] (per_episode mode, policy.py:343-350)
    std::vector<double> h0((size_t)n * 7, 0.0);
    for (int v = 0; v < n; ++v)
        for (int i = 0; i < 5; ++i) h0[(size_t)v * 7 + i] = desc->x_static[(size_t)v * 5 + i];
    for (int e = 0; e < n_enc; ++e) up(o_H[e][0], h0.data(), h0.size() * 8);
    FP_CUDA_RET(cudaGetLastError());

    DevPolicy &P = pol->dev;
    std::memset(&P, 0, sizeof(P));
    P.n = n; P.h = h; P.K = K; P.n_enc = n_enc; P.slope = desc->leaky_slope;
    for (int r = 0; r < PR_COUNT; ++r) P.off[r] = desc->param_offsets[r];
    P.x = (const double *)(b + o_x);
    P.adj_ptr = (const int *)(b + o_ap); P.adj_nbr = (const int *)(b + o_an);
    P.adj_e = (const double *)(b + o_ae);
    P.bp_ptr = (const int *)(b + o_bp); P.bp_idx = (const int *)(b + o_bi);
    P.tp_ptr = (const int *)(b + o_tp); P.tp_idx = (const int *)(b + o_ti);
    P.ibp_ptr = (const int *)(b + o_ibp); P.ibp_idx = (const int *)(b + o_ibi);
    P.itp_ptr = (const int *)(b + o_itp); P.itp_idx = (const int *)(b + o_iti);
    P.forest = forest ? 1 : 0;
    P.jump_rounds = jump_rounds;
    if (forest)
        for (int w = 0; w < 2; ++w) {
            P.nxt[w] = (const int *)(b + o_nx[w]);
            for (int q = 0; q < 2; ++q) {
                P.PS[w][q] = (double *)(b + o_PS[w][q]);
                P.PJ[w][q] = (int *)(b + o_PJ[w][q]);
            }
        }
    for (int e = 0; e < n_enc; ++e) {
        P.H[e][0] = (double *)(b + o_H[e][0]);
        for (int k = 0; k < K; ++k) {
            P.H[e][k + 1] = (double *)(b + o_H[e][k + 1]);
            P.Pm[e][k] = (double *)(b + o_P[e][k]);
            P.Qm[e][k] = (double *)(b + o_Q[e][k]);
            P.U[e][k] = (double *)(b + o_U[e][k]);
            P.AG[e][k] = (double *)(b + o_AG[e][k]);
        }
    }
    P.Zs = (double *)(b + o_Zs); P.emb = (double *)(b + o_emb); P.hidpre = (double *)(b + o_hp);
    P.s = (double *)(b + o_s); P.Zp = (double *)(b + o_Zp); P.A = (double *)(b + o_A);
    P.G = (double *)(b + o_G); P.M = (double *)(b + o_M); P.c = (double *)(b + o_c);
    for (int e = 0; e < 2; ++e) { P.dH[e] = (double *)(b + o_dH[e]); P.dHn[e] = (double *)(b + o_dHn[e]); }
    P.dU = (double *)(b + o_dU); P.Dsrc = (double *)(b + o_Ds); P.Ddst = (double *)(b + o_Dd);
    P.dagg = (double *)(b + o_dagg); P.De = (double *)(b + o_De);
    P.dhid = (double *)(b + o_dhid); P.demb = (double *)(b + o_demb); P.dZ = (double *)(b + o_dZ);
    P.ds = (double *)(b + o_ds); P.dA = (double *)(b + o_dA);
    P.dG = (double *)(b + o_dG); P.dsmall = (double *)(b + o_dsm);
    P.partial = (double *)(b + o_part); P.partial_rows = prow;
    *out = pol;
    return FP_OK;
}

int fp_policy_destroy(fp_policy *pol) {
    if (!pol) return FP_OK;
    if (pol->train) fp_train_state_free(pol->train);
    if (pol->arena) cudaFree(pol->arena);
    delete pol;
    return FP_OK;
}

int fp_policy_prepare(fp_policy *pol, const double *params, void *stream) {
    if (!pol || !params) { set_error("null argument"); return FP_ERR_INVALID; }
    return policy_prepare(pol, params, (cudaStream_t)stream);
}

int fp_policy_table(const fp_policy *pol, int32_t which, const double **ptr, int64_t *count) {
    if (!pol || !ptr || !count) { set_error("null argument"); return FP_ERR_INVALID; }
    const DevPolicy &P = pol->dev;
    const int64_t nh = (int64_t)P.n * P.h;
    switch (which) {
        case FP_TABLE_H_SEL: *ptr = P.H[0][P.K]; *count = nh; break;
        case FP_TABLE_H_PLC: *ptr = P.H[P.n_enc - 1][P.K]; *count = nh; break;
        case FP_TABLE_SEL_LOGIT: *ptr = P.s; *count = P.n; break;
        case FP_TABLE_PLC_A: *ptr = P.A; *count = nh; break;
        case FP_TABLE_PLC_G: *ptr = P.G; *count = nh; break;
        case FP_TABLE_PLC_M: *ptr = P.M; *count = 5 * P.h; break;
        case FP_TABLE_PLC_C: *ptr = P.c; *count = P.h; break;
        default: set_error("unknown table"); return FP_ERR_INVALID;
    }
    return FP_OK;
}

}  // extern "C"
