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
#include <type_traits>
#include <vector>

#include "fp_common.cuh"
#include "fp_policy.cuh"
#include "fp_gnn.cuh"

namespace fp {

constexpr int kEncWarps = 8;

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

// Weight staging: every block of an encoder reads the same small matrices,
// so they are copied to shared memory once per block (h <= 32) and the
// per-vertex MLPs read them with conflict-free LDS (lane = column).
struct RoundW {
    const double *psw, *psb, *phw, *phb, *nw;  // psi (k==0: 15 rows; else the edge row only)
    const double *szw, *szb, *pzw, *pzb, *w1a, *w1b, *w1d;  // last-round head weights
};

__device__ __forceinline__ void stage(double *dst, const double *src, int count) {
    for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = src[i];
}

// doubles of shared memory the staged weights of round k need
__host__ __device__ inline int round_smem_doubles(int h, int k, bool last, bool sel, bool plc) {
    const int dk = k == 0 ? 7 : h;
    int c = (k == 0 ? (2 * dk + 1) * h : h) + h + (dk + h) * h + h;
    if (!last) c += 2 * h * h;
    else {
        if (sel) c += 6 * h;
        if (plc) c += 6 * h + 3 * h * h;
    }
    return c;
}

// One GNN round for every vertex of one encoder (blockIdx.y): gather +
// segment-reduce of the messages into v (CSR by destination, message order
// kept), the phi update, and either the next round's P/Q projections or the
// last round's head rows.  Warps stride over destinations; a warp loads up
// to 32 message (source, edge) pairs with one coalesced access, then gathers
// the P[src] rows four at a time (independent 256-byte loads in flight) and
// accumulates them in message order (bit-identical to the sequential sum).
// BWD: also store U / AG / Zp for the REINFORCE backward (compact graphs).
// HC: hidden width as a compile-time constant (0 = runtime P.h) so the
// per-vertex MLP loops fully unroll -- the loads and shuffles of later
// columns then overlap the dependent fp64 FMA chain.
template <int HPL, int HC, bool STAGE, bool BWD>
__global__ void __launch_bounds__(kEncWarps * 32, 3)
encode_round_kernel(DevPolicy P, int k, int last) {
    extern __shared__ __align__(16) double wsm[];
    const int lane = lane_id();
    const int warp = threadIdx.x >> 5;
    const int e = blockIdx.y;
    const int n = P.n, h = HC ? HC : P.h;
    const int dk = k == 0 ? 7 : h;
    const double *Hk = P.H[e][k];
    const double s = P.slope;
    const bool feeds_sel = e == 0;
    const bool feeds_plc = P.n_enc == 1 || e == 1;

    RoundW W;
    {
        const double *psw = P.W(gnn_role(e, k, 0)), *psb = P.W(gnn_role(e, k, 1));
        const double *phw = P.W(gnn_role(e, k, 2)), *phb = P.W(gnn_role(e, k, 3));
        const double *nw = last ? nullptr : P.W(gnn_role(e, k + 1, 0));
        if constexpr (STAGE) {
            double *o = wsm;
            auto put = [&](const double *src, int count) {
                stage(o, src, count);
                const double *at = o;
                o += count;
                return at;
            };
            W.psw = k == 0 ? put(psw, (2 * dk + 1) * h) : put(psw + (size_t)2 * dk * h, h) - (size_t)2 * dk * h;
            W.psb = put(psb, h);
            W.phw = put(phw, (dk + h) * h);
            W.phb = put(phb, h);
            W.nw = last ? nullptr : put(nw, 2 * h * h);
            W.szw = W.szb = W.pzw = W.pzb = W.w1a = W.w1b = W.w1d = nullptr;
            if (last && feeds_sel) { W.szw = put(P.W(PR_SEL_Z_W), 5 * h); W.szb = put(P.W(PR_SEL_Z_B), h); }
            if (last && feeds_plc) {
                const double *w1 = P.W(PR_PLC_H1_W);
                W.pzw = put(P.W(PR_PLC_Z_W), 5 * h);
                W.pzb = put(P.W(PR_PLC_Z_B), h);
                W.w1a = put(w1, h * h);
                W.w1b = put(w1 + (size_t)h * h, h * h);
                W.w1d = put(w1 + (size_t)3 * h * h, h * h);
            }
            __syncthreads();
        } else {
            W.psw = psw; W.psb = psb; W.phw = phw; W.phb = phb; W.nw = nw;
            W.szw = P.W(PR_SEL_Z_W); W.szb = P.W(PR_SEL_Z_B);
            W.pzw = P.W(PR_PLC_Z_W); W.pzb = P.W(PR_PLC_Z_B);
            const double *w1 = P.W(PR_PLC_H1_W);
            W.w1a = w1; W.w1b = w1 + (size_t)h * h; W.w1d = w1 + (size_t)3 * h * h;
        }
    }

    for (int v = blockIdx.x * kEncWarps + warp; v < n; v += gridDim.x * kEncWarps) {
        double q[HPL], we[HPL], bb[HPL], agg[HPL];
        // this vertex's own input row, one element per lane (broadcast by shfl)
        const double hrow0 = lane < dk ? Hk[(size_t)v * dk + lane] : 0.0;
        const double hrow1 = (HPL > 1 && lane + 32 < dk) ? Hk[(size_t)v * dk + lane + 32] : 0.0;
#pragma unroll
        for (int t = 0; t < HPL; ++t) {
            const int j = lane + 32 * t;
            q[t] = we[t] = bb[t] = agg[t] = 0.0;
            if (j < h) {
                if (k == 0) {
                    double acc = 0.0;
                    for (int i = 0; i < 7; ++i)
                        acc = fma(__shfl_sync(FP_FULL_MASK, hrow0, i), W.psw[(dk + i) * h + j], acc);
                    q[t] = acc;
                } else {
                    q[t] = P.Qm[e][k][(size_t)v * h + j];
                }
                we[t] = W.psw[(2 * dk) * h + j];
                bb[t] = W.psb[j];
            }
        }
        const int m0 = P.adj_ptr[v], m1 = P.adj_ptr[v + 1];
        for (int c0 = m0; c0 < m1; c0 += 32) {
            const int cnt = min(32, m1 - c0);
            const int my_w = lane < cnt ? P.adj_nbr[c0 + lane] : 0;
            const double my_e = lane < cnt ? P.adj_e[c0 + lane] : 0.0;
            for (int i0 = 0; i0 < cnt; i0 += 4) {
                int wv[4];
                double ev[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    wv[u] = __shfl_sync(FP_FULL_MASK, my_w, (i0 + u) & 31);
                    ev[u] = __shfl_sync(FP_FULL_MASK, my_e, (i0 + u) & 31);
                }
#pragma unroll
                for (int t = 0; t < HPL; ++t) {
                    const int j = lane + 32 * t;
                    if (j >= h) continue;
                    double pv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        pv[u] = 0.0;
                        if (i0 + u < cnt) {
                            if (k == 0) {
                                const double *hw = Hk + (size_t)wv[u] * 7;
                                double p = 0.0;
                                for (int i = 0; i < 7; ++i) p = fma(hw[i], W.psw[i * h + j], p);
                                pv[u] = p;
                            } else {
                                pv[u] = P.Pm[e][k][(size_t)wv[u] * h + j];
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (i0 + u < cnt) agg[t] += leaky(pv[u] + q[t] + ev[u] * we[t] + bb[t], s);
                }
            }
        }
        // update: U = [H | agg] @ phi.w + phi.b
        double u[HPL];
#pragma unroll
        for (int t = 0; t < HPL; ++t) u[t] = 0.0;
        auto self_term = [&](auto DK) {
            constexpr int dkc = decltype(DK)::value;
            const int dkr = dkc ? dkc : dk;
#pragma unroll 8
            for (int i = 0; i < dkr; ++i) {
                const double hv = __shfl_sync(FP_FULL_MASK, i < 32 ? hrow0 : hrow1, i & 31);
#pragma unroll
                for (int t = 0; t < HPL; ++t) {
                    const int j = lane + 32 * t;
                    if (j < h) u[t] = fma(hv, W.phw[i * h + j], u[t]);
                }
            }
        };
        if (k == 0) self_term(std::integral_constant<int, 7>{});
        else self_term(std::integral_constant<int, HC>{});
#pragma unroll 8
        for (int i = 0; i < h; ++i) {
            const double a = bcast<HPL>(agg, i);
#pragma unroll
            for (int t = 0; t < HPL; ++t) {
                const int j = lane + 32 * t;
                if (j < h) u[t] = fma(a, W.phw[(dk + i) * h + j], u[t]);
            }
        }
        double hn[HPL];
#pragma unroll
        for (int t = 0; t < HPL; ++t) {
            const int j = lane + 32 * t;
            hn[t] = 0.0;
            if (j < h) {
                u[t] += W.phb[j];
                hn[t] = leaky(u[t], s);
                if constexpr (BWD) {
                    P.U[e][k][(size_t)v * h + j] = u[t];
                    P.AG[e][k][(size_t)v * h + j] = agg[t];
                }
                P.H[e][k + 1][(size_t)v * h + j] = hn[t];
            }
        }
        if (!last) {
            double pp[HPL], qq[HPL];
#pragma unroll
            for (int t = 0; t < HPL; ++t) pp[t] = qq[t] = 0.0;
#pragma unroll 8
            for (int i = 0; i < h; ++i) {
                const double a = bcast<HPL>(hn, i);
#pragma unroll
                for (int t = 0; t < HPL; ++t) {
                    const int j = lane + 32 * t;
                    if (j < h) {
                        pp[t] = fma(a, W.nw[i * h + j], pp[t]);
                        qq[t] = fma(a, W.nw[(h + i) * h + j], qq[t]);
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
            continue;
        }
        // ---- last round: per-vertex head rows ----
        const double xr = lane < 5 ? P.x[(size_t)v * 5 + lane] : 0.0;
        if (feeds_sel) {
#pragma unroll
            for (int t = 0; t < HPL; ++t) {
                const int j = lane + 32 * t;
                double z = 0.0;
                for (int i = 0; i < 5; ++i)
                    z = fma(__shfl_sync(FP_FULL_MASK, xr, i), W.szw[i * h + j < 5 * h ? i * h + j : 0], z);
                if (j < h) P.Zs[(size_t)v * h + j] = z + W.szb[j];
            }
        }
        if (feeds_plc) {
            double z[HPL], a[HPL], g[HPL];
#pragma unroll
            for (int t = 0; t < HPL; ++t) {
                const int j = lane + 32 * t;
                z[t] = a[t] = g[t] = 0.0;
                double acc = 0.0;
                for (int i = 0; i < 5; ++i)
                    acc = fma(__shfl_sync(FP_FULL_MASK, xr, i), W.pzw[i * h + j < 5 * h ? i * h + j : 0], acc);
                if (j >= h) continue;
                z[t] = acc + W.pzb[j];
                if constexpr (BWD) P.Zp[(size_t)v * h + j] = z[t];
            }
#pragma unroll 8
            for (int i = 0; i < h; ++i) {
                const double hv = bcast<HPL>(hn, i), zv = bcast<HPL>(z, i);
#pragma unroll
                for (int t = 0; t < HPL; ++t) {
                    const int j = lane + 32 * t;
                    if (j >= h) continue;
                    a[t] = fma(hv, W.w1a[i * h + j], a[t]);
                    a[t] = fma(zv, W.w1d[i * h + j], a[t]);
                    g[t] = fma(hv, W.w1b[i * h + j], g[t]);
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
}

// Forest-form path sums (large graphs): S(v) = sum of H over path(v), by
// pointer jumping -- after round r, S(v) covers the first 2^(r+1) vertices of
// path(v) and J(v) points 2^(r+1) vertices down it (-1 past the end).
// Round 0 reads H and the next arrays; round r >= 1 ping-pongs PS/PJ.
// Pure gather-add over n x h doubles per round (HBM / L2 bound).
template <bool VEC2>
__global__ void path_jump_kernel(DevPolicy P, int r) {
    const int which = blockIdx.y;  // 0 = b-paths, 1 = t-paths
    const int n = P.n, h = P.h;
    const double *Sin = r == 0 ? P.H[0][P.K] : P.PS[which][(r - 1) & 1];
    const int *Jin = r == 0 ? P.nxt[which] : P.PJ[which][(r - 1) & 1];
    double *Sout = P.PS[which][r & 1];
    int *Jout = P.PJ[which][r & 1];
    if constexpr (VEC2) {  // h even: 16-byte accesses, two columns per thread
        const int h2 = h >> 1;
        const int64_t total = (int64_t)n * h2;
        const double2 *S2 = (const double2 *)Sin;
        double2 *O2 = (double2 *)Sout;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
             i += (int64_t)gridDim.x * blockDim.x) {
            const int v = (int)(i / h2), j = (int)(i - (int64_t)v * h2);
            const int w = Jin[v];
            double2 a = S2[i];
            if (w >= 0) {
                const double2 b = S2[(size_t)w * h2 + j];
                a.x += b.x;
                a.y += b.y;
            }
            O2[i] = a;
            if (j == 0) Jout[v] = w >= 0 ? Jin[w] : -1;
        }
    } else {
        const int64_t total = (int64_t)n * h;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
             i += (int64_t)gridDim.x * blockDim.x) {
            const int v = (int)(i / h), j = (int)(i - (int64_t)v * h);
            const int w = Jin[v];
            Sout[i] = w >= 0 ? Sin[i] + Sin[(size_t)w * h + j] : Sin[i];
            if (j == 0) Jout[v] = w >= 0 ? Jin[w] : -1;
        }
    }
}

// SEL head over every vertex: s[v] = head(H[v] | sum_bpath H | sum_tpath H | Z[v]).
// head1.w (4h x h) staged in shared memory; BWD also stores the embedding and
// pre-activation rows the backward reads.
template <int HPL, int HC, bool STAGE, bool BWD>
__global__ void __launch_bounds__(kEncWarps * 32, 3) encode_sel_kernel(DevPolicy P) {
    extern __shared__ __align__(16) double wsm[];
    const int lane = lane_id();
    const int n = P.n, h = HC ? HC : P.h;
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
    const double *w1 = P.W(PR_SEL_H1_W), *b1 = P.W(PR_SEL_H1_B), *w2 = P.W(PR_SEL_H2_W),
                 *b2 = P.W(PR_SEL_H2_B);
    if constexpr (STAGE) {
        stage(wsm, w1, 4 * h * h);
        __syncthreads();
        w1 = wsm;
    }
    for (int v = blockIdx.x * kEncWarps + (threadIdx.x >> 5); v < n;
         v += gridDim.x * kEncWarps) {
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
            if constexpr (BWD)
                for (int b = 0; b < 4; ++b) P.emb[(size_t)v * 4 * h + b * h + j] = em[b][t];
        }
        double acc[HPL];
#pragma unroll
        for (int t = 0; t < HPL; ++t) acc[t] = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll 8
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
                if constexpr (BWD) P.hidpre[(size_t)v * h + j] = pre;
                part = fma(leaky(pre, s), w2[j], part);
            }
        }
        part = warp_sum(part);
        if (lane == 0) P.s[v] = part + b2[0];
    }
}

#define FP_CUDA_RET(call)                                                             \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess) {                                                      \
            set_error(std::string(#call) + ": " + cudaGetErrorString(e_));            \
            return FP_ERR_CUDA;                                                       \
        }                                                                             \
    } while (0)

// ---------------------------------------------------------------------------
// Aggregation-kernel timer (measurement only, fp_agg_timer_*): when enabled,
// an event pair is recorded on the launching stream around every aggregation
// launch, so bench.py can report the kernel's own average duration over its
// timed region.  Host-side bookkeeping, one encoder thread at a time.
// ---------------------------------------------------------------------------
namespace {
struct AggTimer {
    bool on = false;
    std::vector<cudaEvent_t> ev;  // pairs
    size_t used = 0;
};
AggTimer &agg_timer() {
    static AggTimer t;
    return t;
}
}  // namespace

// FP_AGG_STAGED=0 turns the staged batched aggregation off (A/B runs only)
bool agg_staged_enabled() {
    static const bool on = !(getenv("FP_AGG_STAGED") && atoi(getenv("FP_AGG_STAGED")) == 0);
    return on;
}

void agg_timer_begin(cudaStream_t st) {
    AggTimer &t = agg_timer();
    if (!t.on) return;
    if (t.used + 2 > t.ev.size()) {
        for (int i = 0; i < 2; ++i) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            t.ev.push_back(e);
        }
    }
    cudaEventRecord(t.ev[t.used], st);
}

void agg_timer_end(cudaStream_t st) {
    AggTimer &t = agg_timer();
    if (!t.on) return;
    cudaEventRecord(t.ev[t.used + 1], st);
    t.used += 2;
}

int agg_timer_enable(int on) {
    AggTimer &t = agg_timer();
    t.on = on != 0;
    t.used = 0;
    return FP_OK;
}

int agg_timer_read(double *total_ms, int64_t *launches) {
    AggTimer &t = agg_timer();
    double tot = 0.0;
    for (size_t i = 0; i < t.used; i += 2) {
        FP_CUDA_RET(cudaEventSynchronize(t.ev[i + 1]));
        float ms = 0.f;
        FP_CUDA_RET(cudaEventElapsedTime(&ms, t.ev[i], t.ev[i + 1]));
        tot += ms;
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = (int64_t)(t.used / 2);
    t.used = 0;
    return FP_OK;
}


template <int HPL, int HC, bool STAGE, bool BWD>
static int launch_encode(DevPolicy &P, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int vblocks = (P.n + kEncWarps - 1) / kEncWarps;
    for (int k = 0; k < P.K; ++k) {
        const bool last = k == P.K - 1;
        const int64_t smem = STAGE ? 8LL * round_smem_doubles(P.h, k, last, true, true) : 0;
        auto kern = encode_round_kernel<HPL, HC, STAGE, BWD>;
        if (smem > 48 * 1024)
            FP_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem));
        // staged weights amortise over many vertices per block: one resident wave
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kEncWarps * 32, (size_t)smem);
        const int bx = STAGE ? std::min(vblocks, std::max(1, sms * std::max(occ, 1) / P.n_enc))
                             : vblocks;
        kern<<<dim3(std::max(bx, 1), P.n_enc), kEncWarps * 32, smem, st>>>(P, k, last);
        FP_CUDA_RET(cudaGetLastError());
    }
    if (P.forest)
        for (int r = 0; r < P.jump_rounds; ++r) {
            const int64_t total = (int64_t)P.n * P.h;
            const int blocks = (int)std::min<int64_t>((total / 2 + 255) / 256, (int64_t)sms * 16);
            if (P.h % 2 == 0)
                path_jump_kernel<true><<<dim3(blocks, 2), 256, 0, st>>>(P, r);
            else
                path_jump_kernel<false><<<dim3(blocks, 2), 256, 0, st>>>(P, r);
            FP_CUDA_RET(cudaGetLastError());
        }
    const int64_t smem2 = STAGE ? 8LL * 4 * P.h * P.h : 0;
    auto kern2 = encode_sel_kernel<HPL, HC, STAGE, BWD>;
    if (smem2 > 48 * 1024)
        FP_CUDA_RET(cudaFuncSetAttribute(kern2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem2));
    int occ2 = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, kern2, kEncWarps * 32, (size_t)smem2);
    const int bx2 = STAGE ? std::min(vblocks, sms * std::max(occ2, 1)) : vblocks;
    kern2<<<std::max(bx2, 1), kEncWarps * 32, smem2, st>>>(P);
    FP_CUDA_RET(cudaGetLastError());
    return FP_OK;
}

// Split encoder: aggregation kernels (HBM) + DMMA node-MLP kernels, for
// hidden widths that tile by 8 (every PolicyConfig the reference ships).
template <int H, bool BWD>
static int launch_gnn_tc(DevPolicy &P, cudaStream_t st, bool sel_head = true) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int warps = 8, threads = warps * 32;
    const int tiles = (P.rows + 7) / 8;
    const int tile_blocks = (tiles + warps - 1) / warps;
    auto grid_for = [&](const void *kern, int64_t smem, int want) {
        int occ = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, (size_t)smem) !=
                cudaSuccess || occ < 1)
            occ = 1;
        return std::max(1, std::min(want, std::max(1, sms * occ / P.n_enc)));
    };
    auto set_smem = [&](const void *kern, int64_t smem) {
        if (smem > 48 * 1024)
            return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        return cudaSuccess;
    };
    if (P.tc && (BWD || (H != 16 && H != 32))) {
        set_error("the bf16 tensor-core encoder is forward-only, hidden 16 or 32");
        return FP_ERR_UNSUPPORTED;
    }
    if (sel_head && !P.forest && P.rows <= kSmallEncodeRows && !P.tc) {
        // + shared-memory H_sel copy, path sums and SEL path lists (block 0)
        int64_t smem = 8LL * (sel_smem_doubles(H) + 3LL * P.n * H) +
                       4LL * (2 * (P.n + 1) + P.n_bpath + P.n_tpath);
        for (int k = 0; k < P.K; ++k)
            smem = std::max<int64_t>(smem, 8LL * node_smem_doubles(H, k, k == P.K - 1));
        // 512 threads for h <= 32: the aggregation / path-sum / weight-staging
        // phases spread over 16 warps (FFNN 44.6 -> 38.4 us, 128 registers, no
        // spills; h = 64 would spill at 128 and keeps 256).  FP_SMALL_THREADS=256
        // for A/B runs.
        static const bool env256 = getenv("FP_SMALL_THREADS") && atoi(getenv("FP_SMALL_THREADS")) == 256;
        if (H <= 32 && !env256) {
            const void *kern = (const void *)gnn_small_kernel<H, BWD, 512>;
            FP_CUDA_RET(set_smem(kern, smem));
            gnn_small_kernel<H, BWD, 512><<<P.n_enc, 512, smem, st>>>(P);
        } else {
            const void *kern = (const void *)gnn_small_kernel<H, BWD>;
            FP_CUDA_RET(set_smem(kern, smem));
            gnn_small_kernel<H, BWD><<<P.n_enc, threads, smem, st>>>(P);
        }
        FP_CUDA_RET(cudaGetLastError());
        return FP_OK;
    }
    {
        const int64_t smem = 8LL * (2 * (2 * H / 8) * 32);
        const void *kern = (const void *)gnn_proj0_kernel<H>;
        FP_CUDA_RET(set_smem(kern, smem));
        gnn_proj0_kernel<H><<<dim3(grid_for(kern, smem, tile_blocks), P.n_enc), threads, smem, st>>>(P);
        FP_CUDA_RET(cudaGetLastError());
    }
    constexpr int VPW = H / 2 >= 32 ? 1 : 32 / (H / 2);
    const int agg_blocks = (P.rows + 8 * VPW - 1) / (8 * VPW);
    for (int k = 0; k < P.K; ++k) {
        const bool last = k == P.K - 1;
        int agg_S = 0;  // staged batched path: stages that fit one block per SM
        if (P.rows >= 2 * P.n && P.rows % P.n == 0 && agg_staged_enabled()) {
            int optin = 0;
            cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            for (int S = 4; S >= 2 && !agg_S; --S)
                if (agg_staged_smem(P.n, P.n_msgs, H, P.tc, S) <= optin &&
                    (S == 2 || 2LL * P.n * H * (P.tc ? 4 : 8) * S <= 160 * 1024))
                    agg_S = S;
        }
        if (agg_S) {
            const int64_t smem = agg_staged_smem(P.n, P.n_msgs, H, P.tc, agg_S);
            const void *kern = P.tc ? (const void *)gnn_agg_staged_kernel<H, true>
                                    : (const void *)gnn_agg_staged_kernel<H, false>;
            FP_CUDA_RET(set_smem(kern, smem));
            const int B = P.rows / P.n;
            const dim3 grid(std::max(1, std::min(B, sms / P.n_enc)), P.n_enc);
            agg_timer_begin(st);
            if (P.tc) FP_CUDA_RET(launch_pdl(gnn_agg_staged_kernel<H, true>, grid, dim3(1024), (size_t)smem, st, P, k, agg_S));
            else FP_CUDA_RET(launch_pdl(gnn_agg_staged_kernel<H, false>, grid, dim3(1024), (size_t)smem, st, P, k, agg_S));
            FP_CUDA_RET(cudaGetLastError());
            agg_timer_end(st);
        } else {
            agg_timer_begin(st);
            if (P.tc) {
                const void *kern = (const void *)gnn_agg_kernel<H, true>;
                gnn_agg_kernel<H, true><<<dim3(grid_for(kern, 0, agg_blocks), P.n_enc), 256, 0, st>>>(P, k);
            } else {
                const void *kern = (const void *)gnn_agg_kernel<H>;
                FP_CUDA_RET(launch_pdl(gnn_agg_kernel<H>, dim3(grid_for(kern, 0, agg_blocks), P.n_enc),
                                       dim3(256), 0, st, P, k));
            }
            FP_CUDA_RET(cudaGetLastError());
            agg_timer_end(st);
        }
        if (P.tc) {  // bf16 node MLPs on tcgen05, operands by TMA
            const int rc = tc_node_launch(P, k, last, st);
            if (rc) return rc;
            continue;
        }
        const int64_t smem = 8LL * node_smem_doubles(H, k, last);
        const void *kern = k == 0 ? (const void *)gnn_node_kernel<H, true, BWD>
                                  : (const void *)gnn_node_kernel<H, false, BWD>;
        FP_CUDA_RET(set_smem(kern, smem));
        const dim3 grid(grid_for(kern, smem, tile_blocks), P.n_enc);
        if (k == 0)
            FP_CUDA_RET(launch_pdl(gnn_node_kernel<H, true, BWD>, grid, dim3(threads), (size_t)smem, st, P, k, (int)last));
        else
            FP_CUDA_RET(launch_pdl(gnn_node_kernel<H, false, BWD>, grid, dim3(threads), (size_t)smem, st, P, k, (int)last));
        FP_CUDA_RET(cudaGetLastError());
    }
    if (!sel_head) return FP_OK;
    if (!P.forest) {
        FP_CUDA_RET(launch_pdl(gnn_pathsum_kernel<H>, dim3(std::max(1, std::min((P.n + 7) / 8, sms * 8))),
                               dim3(256), 0, st, P));
        FP_CUDA_RET(cudaGetLastError());
    }
    if (P.forest)
        for (int r = 0; r < P.jump_rounds; ++r) {
            const int64_t total = (int64_t)P.n * H;
            const int blocks = (int)std::min<int64_t>((total / 2 + 255) / 256, (int64_t)sms * 16);
            path_jump_kernel<true><<<dim3(blocks, 2), 256, 0, st>>>(P, r);
            FP_CUDA_RET(cudaGetLastError());
        }
    {
        const int64_t smem = 8LL * sel_smem_doubles(H);
        const void *kern = (const void *)gnn_sel_kernel<H, BWD>;
        FP_CUDA_RET(set_smem(kern, smem));
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, (size_t)smem);
        const int gx = std::max(1, std::min(tile_blocks, sms * std::max(occ, 1)));
        FP_CUDA_RET(launch_pdl(gnn_sel_kernel<H, BWD>, dim3(gx), dim3(threads), (size_t)smem, st, P));
        FP_CUDA_RET(cudaGetLastError());
    }
    return FP_OK;
}

template <int H>
static int launch_gnn_tc_any(DevPolicy &P, cudaStream_t st) {
    return (P.forest || P.tc) ? launch_gnn_tc<H, false>(P, st) : launch_gnn_tc<H, true>(P, st);
}

int gnn_encode_rows(DevPolicy &P, cudaStream_t st, bool bwd, bool sel_head) {
    switch (P.h) {
#define FP_CASE(HH) \
        case HH: return bwd ? launch_gnn_tc<HH, true>(P, st, sel_head) : launch_gnn_tc<HH, false>(P, st, sel_head);
        FP_CASE(8) FP_CASE(16) FP_CASE(32) FP_CASE(64)
#undef FP_CASE
        default:
            set_error("the batched encoder needs hidden in {8, 16, 32, 64}");
            return FP_ERR_UNSUPPORTED;
    }
}

int policy_prepare(fp_policy *pol, const double *params, cudaStream_t st) {
    {
        DevPolicy &P = pol->dev;
        P.params = params;
        if (P.n == 0) return FP_OK;
        if (!pol->fused_encoder) switch (P.h) {
            case 8: return launch_gnn_tc_any<8>(P, st);
            case 16: return launch_gnn_tc_any<16>(P, st);
            case 32: return launch_gnn_tc_any<32>(P, st);
            case 64: return launch_gnn_tc_any<64>(P, st);
            default: break;
        }
    }
    DevPolicy &P = pol->dev;
    P.params = params;
    if (P.n == 0) return FP_OK;
    // forest-form policies (large graphs) are forward-only: no backward rows
    const bool bwd = !P.forest;
    if (P.h == 32)
        return bwd ? launch_encode<1, 32, true, true>(P, st) : launch_encode<1, 32, true, false>(P, st);
    if (P.h < 32)
        return bwd ? launch_encode<1, 0, true, true>(P, st) : launch_encode<1, 0, true, false>(P, st);
    return bwd ? launch_encode<2, 0, false, true>(P, st) : launch_encode<2, 0, false, false>(P, st);
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
    else
        for (int w = 0; w < 2; ++w) o_PS[w][0] = take(nh);  // explicit-list path sums
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
    P.rows = n; P.batch = 1; P.D = p->dev.d; P.ps_dev = nullptr;
    for (int r = 0; r < PR_COUNT; ++r) P.off[r] = desc->param_offsets[r];
    P.x = (const double *)(b + o_x);
    P.adj_ptr = (const int *)(b + o_ap); P.adj_nbr = (const int *)(b + o_an);
    P.adj_e = (const double *)(b + o_ae);
    P.n_msgs = (int)M;
    P.n_params = desc->n_params;
    P.bp_ptr = (const int *)(b + o_bp); P.bp_idx = (const int *)(b + o_bi);
    P.tp_ptr = (const int *)(b + o_tp); P.tp_idx = (const int *)(b + o_ti);
    P.n_bpath = forest ? 0 : (int)Lb;
    P.n_tpath = forest ? 0 : (int)Lt;
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
    else
        for (int w = 0; w < 2; ++w) P.PS[w][0] = (double *)(b + o_PS[w][0]);
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

    *out = pol;
    return FP_OK;
}

int fp_policy_destroy(fp_policy *pol) {
    if (!pol) return FP_OK;
    if (pol->train) fp_train_state_free(pol->train);
    if (pol->arena) cudaFree(pol->arena);
    if (pol->tc_planes) cudaFree(pol->tc_planes);
    delete pol;
    return FP_OK;
}

int fp_agg_timer_enable(int32_t on) { return fp::agg_timer_enable(on); }

int fp_agg_timer_read(double *total_ms, int64_t *launches) {
    return fp::agg_timer_read(total_ms, launches);
}

int fp_policy_set_encoder(fp_policy *pol, int32_t mode) {
    if (!pol) { set_error("null argument"); return FP_ERR_INVALID; }
    DevPolicy &P = pol->dev;
    if (mode == FP_ENCODER_TC) {
        if (P.h != 16 && P.h != 32) {
            set_error("the bf16 tensor-core encoder needs hidden 16 or 32");
            return FP_ERR_UNSUPPORTED;
        }
        if (!pol->tc_planes && P.n > 0) {
            const int64_t bytes = tc_plane_bytes(P.n, P.K, P.n_enc);
            if (cudaMalloc(&pol->tc_planes, bytes) != cudaSuccess) {
                set_error("cudaMalloc failed for the bf16 encoder planes");
                return FP_ERR_CUDA;
            }
            cudaMemset(pol->tc_planes, 0, bytes);
        }
        if (pol->tc_planes) tc_set_planes(P, pol->tc_planes, P.n);
        P.tc = 1;
        pol->fused_encoder = 0;
        return FP_OK;
    }
    if (mode != FP_ENCODER_DMMA && mode != FP_ENCODER_FUSED) {
        set_error("unknown encoder mode");
        return FP_ERR_INVALID;
    }
    P.tc = 0;
    pol->fused_encoder = mode == FP_ENCODER_FUSED;
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
