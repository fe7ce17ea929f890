// GNN encoder split into its two rooflines (flowplace/policy.py:149-223):
//
//   gnn_agg_kernel   message passing: for every destination v,
//                    agg[v] = sum_{m into v} leaky(P[src_m] + Q[v] + e_m*we + b)
//                    (policy.py:159-166 with psi split by input block).  A
//                    pure gather / segment-reduce over the CSR-by-destination
//                    message list: H/2 lanes per destination, one 16-byte
//                    load of P[src] per lane per message, four messages in
//                    flight, summed in message order.  HBM-bound.
//   gnn_agg_staged_kernel  the same sums for batched per_step rows (B x n):
//                    each episode's P / Q slices moved into shared memory by
//                    1-D TMA bulk copies (S-stage mbarrier ring), the gather
//                    then runs out of shared memory -- DRAM sees sequential
//                    streams only (80% of measured HBM at Llama-block B=1024).
//   gnn_node_kernel  the per-vertex MLPs as dense [rows x K] @ [K x N] tiles
//                    on the fp64 tensor cores (DMMA, mma.sync m8n8k4 f64 --
//                    the only tensor-core path that keeps the reference's
//                    float64; tcgen05 has no f64 kind): phi update
//                    U = [H | agg] @ phi.w + b, H' = leaky(U), then the next
//                    round's P/Q projections or the head tables (Zs, Zp,
//                    A = [H|Zp] @ [W1a; W1d], G = H @ W1b).
//   gnn_proj0_kernel round-0 P/Q = H0 @ psi rows (7-column input).
//   gnn_sel_kernel   SEL head over every vertex: [H | sum_b H | sum_t H | Zs]
//                    @ head1.w (4h x h) -> leaky -> . head2.w  (DMMA).
//
// Weight matrices are staged once per block into shared memory in MMA
// fragment order (each lane's B element contiguous: conflict-free), A tiles
// are 8 vertex rows with a row stride == 4 (mod 16) doubles so the
// half-warp fragment loads hit 16 distinct 8-byte banks.
#pragma once

#include <cuda_bf16.h>

#include <type_traits>

#include "fp_common.cuh"
#include "fp_policy.cuh"
#include "fp_tc.cuh"

namespace fp {

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ double gleaky(double x, double s) { return x > 0.0 ? x : s * x; }

// row stride (doubles) of an 8-row A tile with K columns
__host__ __device__ constexpr int tile_stride(int K) { return ((K + 11) / 16) * 16 + 4; }

// Stage a K x N matrix B(k, n) into fragment order [KT][NT][32]:
// lane l of (kt, nt) holds B(kt*4 + l%4, nt*8 + l/4); rows >= K are zero.
// Eight loads are issued before their shared-memory stores (the stores could
// alias the generic source pointer, so a load-store loop would pay one full
// global round trip per element).
template <typename F>
__device__ __forceinline__ void stage_frag(double *dst, int K, int KT, int NT, F B) {
    constexpr int U = 8;
    const int total = KT * NT * 32, step = blockDim.x;
    for (int i0 = threadIdx.x; i0 < total; i0 += U * step) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * step;
            double x = 0.0;
            if (i < total) {
                const int l = i & 31, nt = (i >> 5) % NT, kt = (i >> 5) / NT;
                const int k = kt * 4 + (l & 3), nn = nt * 8 + (l >> 2);
                if (k < K) x = B(k, nn);
            }
            v[u] = x;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * step < total) dst[i0 + u * step] = v[u];
    }
}

// acc[nt] += A(8 x KT*4, smem, stride sa) @ Bf(fragment order, KT x NT)
// D fragment: acc[nt][i] = D[lane >> 2][nt*8 + (lane & 3)*2 + i]
template <int NT>
__device__ __forceinline__ void tile_mma(const double *As, int sa, int KT, const double *Bf,
                                         double (&acc)[NT][2]) {
    const int lane = lane_id();
    const double *ap = As + (lane >> 2) * sa + (lane & 3);
    const double *bp = Bf + lane;
#pragma unroll 4
    for (int kt = 0; kt < KT; ++kt) {
        const double a = ap[kt * 4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(acc[nt], a, bp[(kt * NT + nt) * 32]);
    }
}

template <int NT>
__device__ __forceinline__ void zero_acc(double (&acc)[NT][2]) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
}

// ---------------------------------------------------------------------------
// Aggregation (HBM-bound gather / segment reduce)
// ---------------------------------------------------------------------------
// P/Q rows as fp64 (reference-exact encoders) or fp32 (bf16 tensor-core
// encoder: half the gathered bytes)
template <bool F32>
__device__ __forceinline__ double2 pq_load(const void *base, size_t i) {
    if constexpr (F32) {
        const float2 f = ((const float2 *)base)[i];
        return make_double2(f.x, f.y);
    } else {
        return ((const double2 *)base)[i];
    }
}

template <int H, bool F32 = false, int U = 4>
__device__ __forceinline__ void gnn_agg_body(const DevPolicy &P, int k, int e_, int bx_, int gx_, double *gsm) {
    constexpr int HL = H / 2;                   // lanes per destination (double2 each)
    constexpr int VPW = HL >= 32 ? 1 : 32 / HL; // destinations per warp
    static_assert(H % 2 == 0 && H <= 64, "H must be even and <= 64");
    const int e = e_;
    const int lane = lane_id();
    const int sub = HL >= 32 ? 0 : lane / HL;
    const int l = HL >= 32 ? lane : lane % HL;
    const int n = P.n, rows = P.rows;
    const int dk = k == 0 ? 7 : H;
    const double *psw = P.W(gnn_role(e, k, 0)), *psb = P.W(gnn_role(e, k, 1));
    // parameter rows sit at arbitrary offsets of the flat vector: scalar loads
    const double2 we = make_double2(psw[(size_t)(2 * dk) * H + 2 * l], psw[(size_t)(2 * dk) * H + 2 * l + 1]);
    const double2 bb = make_double2(psb[2 * l], psb[2 * l + 1]);
    const void *Pm = P.Pm[e][k];
    const void *Qm = P.Qm[e][k];
    double2 *agg = (double2 *)P.AG[e][k];
    const double s = P.slope;
    const int warps = blockDim.x >> 5;
    const int gw = bx_ * warps + (threadIdx.x >> 5);
    griddep_wait();  // P / Q come from the previous kernel
    for (int vb = gw * VPW; vb < rows; vb += gx_ * warps * VPW) {
        const int r = vb + sub;  // row = episode * n + vertex
        if (r >= rows || (HL < 32 && lane >= VPW * HL)) continue;
        const int v = r % n, base = r - v;
        const double2 q = pq_load<F32>(Qm, (size_t)r * HL + l);
        double ax = 0.0, ay = 0.0;
        const int m1 = P.adj_ptr[v + 1];
        for (int m = P.adj_ptr[v]; m < m1; m += U) {
            int w[U];
            double ev[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool ok = m + u < m1;
                w[u] = ok ? base + P.adj_nbr[m + u] : base;
                ev[u] = ok ? P.adj_e[m + u] : 0.0;
            }
            double2 p[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                p[u] = m + u < m1 ? pq_load<F32>(Pm, (size_t)w[u] * HL + l) : make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (m + u < m1) {
                    // the reference message: leaky(P[src] + Q[dst] + e*we + b), summed in order
                    ax += gleaky(p[u].x + q.x + ev[u] * we.x + bb.x, s);
                    ay += gleaky(p[u].y + q.y + ev[u] * we.y + bb.y, s);
                }
        }
        if (!F32) agg[(size_t)r * HL + l] = make_double2(ax, ay);
        if (P.tc) {  // bf16 encoder: agg as split planes at X_k[:, 32 + 2l]
            const __nv_bfloat162 hi = __floats2bfloat162_rn((float)ax, (float)ay);
            const float2 hf = __bfloat1622float2(hi);
            const __nv_bfloat162 lo = __floats2bfloat162_rn((float)ax - hf.x, (float)ay - hf.y);
            *(__nv_bfloat162 *)(P.Xh[e][k] + (size_t)r * 64 + 32 + 2 * l) = hi;
            *(__nv_bfloat162 *)(P.Xl[e][k] + (size_t)r * 64 + 32 + 2 * l) = lo;
        }
    }
}

// Batched rows, staged (per_step, B episodes x n vertices, 2 x n x H x
// sizeof(T) <= ~100 KB): an episode's whole P and Q slices are contiguous, so
// one elected thread moves them into shared memory with two 1-D TMA bulk
// copies (S-stage ring, mbarrier completion), the CSR message list is staged
// once per block, and the gather runs out of shared memory.  DRAM then sees
// only sequential streams -- P and Q read once, agg written once -- instead
// of 256-byte row gathers scattered across each episode's slice (which held
// the gather kernel near 60% of HBM).  One 512-thread block per SM per
// encoder; per-row message order and arithmetic are gnn_agg_body's.
template <int H, bool F32, int NT = 1024>
__global__ void __launch_bounds__(NT, 1) gnn_agg_staged_kernel(DevPolicy P, int k, int S) {
    using T = typename std::conditional<F32, float, double>::type;
    using T2 = typename std::conditional<F32, float2, double2>::type;
    constexpr int HL = H / 2;
    extern __shared__ __align__(128) unsigned char agg_sm[];
    const int e = blockIdx.y;
    const int n = P.n, B = P.rows / n;
    const int M = P.adj_ptr[n];
    const uint32_t slice = (uint32_t)n * H * sizeof(T);
    uint64_t *bar = (uint64_t *)agg_sm;                  // S <= 8 barriers
    unsigned char *stg = agg_sm + 128;                   // [S][P slice | Q slice]
    double *s_e = (double *)(stg + (size_t)S * 2 * slice);
    int *s_ptr = (int *)(s_e + M);
    int *s_nbr = s_ptr + n + 1;
    const T *Pg = (const T *)P.Pm[e][k];
    const T *Qg = (const T *)P.Qm[e][k];
    griddep_launch();
    // prologue on constant tables (message CSR), overlapping the previous
    // kernel under PDL; P / Q only after the dependency wait
    for (int i = threadIdx.x; i < M; i += blockDim.x) {
        s_e[i] = P.adj_e[i];
        s_nbr[i] = P.adj_nbr[i] * HL;  // row offset in T2 units
    }
    for (int i = threadIdx.x; i <= n; i += blockDim.x) s_ptr[i] = P.adj_ptr[i];
    griddep_wait();
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) tc::mbar_init(&bar[i], 1);
        tc::fence_mbar_init();
        for (int i = 0; i < S; ++i) {
            const int ep = blockIdx.x + i * gridDim.x;
            if (ep >= B) break;
            unsigned char *dst = stg + (size_t)i * 2 * slice;
            tc::mbar_arrive_expect_tx(&bar[i], 2 * slice);
            tc::bulk_load(dst, Pg + (size_t)ep * n * H, slice, &bar[i]);
            tc::bulk_load(dst + slice, Qg + (size_t)ep * n * H, slice, &bar[i]);
        }
    }
    const int l = threadIdx.x % HL, unit = threadIdx.x / HL, units = blockDim.x / HL;
    const int dk = k == 0 ? 7 : H;
    const double *psw = P.W(gnn_role(e, k, 0)), *psb = P.W(gnn_role(e, k, 1));
    const double2 we = make_double2(psw[(size_t)(2 * dk) * H + 2 * l], psw[(size_t)(2 * dk) * H + 2 * l + 1]);
    const double2 bb = make_double2(psb[2 * l], psb[2 * l + 1]);
    const double s = P.slope;
    double2 *agg = (double2 *)P.AG[e][k];
    __syncthreads();
    int it = 0;
    for (int ep = blockIdx.x; ep < B; ep += gridDim.x, ++it) {
        const int st = it % S;
        tc::mbar_wait(&bar[st], (uint32_t)((it / S) & 1));
        const T2 *Ps = (const T2 *)(stg + (size_t)st * 2 * slice);
        const T2 *Qs = (const T2 *)(stg + (size_t)st * 2 * slice + slice);
        for (int v = unit; v < n; v += units) {
            const T2 qt = Qs[v * HL + l];
            const double qx = qt.x, qy = qt.y;
            double ax = 0.0, ay = 0.0;
            const int m1 = s_ptr[v + 1];
            // one message per trip: the rows' few messages (E/n ~ 1.5 per
            // direction) left most of a 4-wide predicated chunk idle, and the
            // kernel is issue-bound once its loads are sequential
#pragma unroll 2
            for (int m = s_ptr[v]; m < m1; ++m) {
                const T2 p = Ps[s_nbr[m] + l];
                const double ev = s_e[m];
                const double mx = (double)p.x + qx + ev * we.x + bb.x;
                const double my = (double)p.y + qy + ev * we.y + bb.y;
                ax += gleaky(mx, s);
                ay += gleaky(my, s);
            }
            const size_t r = (size_t)ep * n + v;
            if (!F32) agg[r * HL + l] = make_double2(ax, ay);
            if (P.tc) {
                const __nv_bfloat162 hi = __floats2bfloat162_rn((float)ax, (float)ay);
                const float2 hf = __bfloat1622float2(hi);
                const __nv_bfloat162 lo = __floats2bfloat162_rn((float)ax - hf.x, (float)ay - hf.y);
                *(__nv_bfloat162 *)(P.Xh[e][k] + r * 64 + 32 + 2 * l) = hi;
                *(__nv_bfloat162 *)(P.Xl[e][k] + r * 64 + 32 + 2 * l) = lo;
            }
        }
        __syncthreads();  // stage st consumed by every thread
        if (threadIdx.x == 0) {
            const int nxt = ep + S * gridDim.x;
            if (nxt < B) {
                unsigned char *dst = stg + (size_t)st * 2 * slice;
                tc::mbar_arrive_expect_tx(&bar[st], 2 * slice);
                tc::bulk_load(dst, Pg + (size_t)nxt * n * H, slice, &bar[st]);
                tc::bulk_load(dst + slice, Qg + (size_t)nxt * n * H, slice, &bar[st]);
            }
        }
    }
}

// shared-memory bytes of gnn_agg_staged_kernel with S stages
inline int64_t agg_staged_smem(int n, int M, int H, bool f32, int S) {
    const int64_t slice = (int64_t)n * H * (f32 ? 4 : 8);
    return 128 + S * 2 * slice + 8LL * M + 4LL * (n + 1 + M);
}

template <int H, bool F32 = false>
__global__ void __launch_bounds__(256, 5) gnn_agg_kernel(DevPolicy P, int k) {
    extern __shared__ __align__(16) double gsm[];
    griddep_launch();
    gnn_agg_body<H, F32>(P, k, blockIdx.y, blockIdx.x, gridDim.x, gsm);
}



// First touch of every table an encode reads (flat params, message CSR,
// static features, H0, SEL path lists) as L2 prefetches issued all at once by
// the first kernel of the encode: after the step's L2 flush each later phase
// (weight staging, CSR walks, path walks) would otherwise pay its own
// dependent DRAM round trips.  Pure hint: no effect on results.
__device__ __forceinline__ void prefetch_l2(const void *base, int64_t bytes, int tid, int nth) {
    for (int64_t o = (int64_t)tid * 128; o < bytes; o += (int64_t)nth * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"((const char *)base + o));
}
__device__ __forceinline__ void prefetch_encode_inputs(const DevPolicy &P, int tid, int nth) {
    const int n = P.n;
    prefetch_l2(P.params, P.n_params * 8, tid, nth);
    prefetch_l2(P.adj_ptr, (int64_t)(n + 1) * 4, tid, nth);
    prefetch_l2(P.adj_nbr, (int64_t)P.n_msgs * 4, tid, nth);
    prefetch_l2(P.adj_e, (int64_t)P.n_msgs * 8, tid, nth);
    if (!P.ps_dev) {
        prefetch_l2(P.x, (int64_t)n * 5 * 8, tid, nth);
        for (int e = 0; e < P.n_enc; ++e) prefetch_l2(P.H[e][0], (int64_t)n * 7 * 8, tid, nth);
    }
    if (!P.forest) {
        prefetch_l2(P.bp_ptr, (int64_t)(n + 1) * 4, tid, nth);
        prefetch_l2(P.tp_ptr, (int64_t)(n + 1) * 4, tid, nth);
        prefetch_l2(P.bp_idx, (int64_t)P.n_bpath * 4, tid, nth);
        prefetch_l2(P.tp_idx, (int64_t)P.n_tpath * 4, tid, nth);
    }
}

// ---------------------------------------------------------------------------
// Round-0 projections: [P0 | Q0] = H0 (n x 7) @ [psi.w rows 0..6 | rows 7..13]
// ---------------------------------------------------------------------------
template <int H>
__device__ __forceinline__ void gnn_proj0_body(const DevPolicy &P, int e_, int bx_, int gx_, double *gsm) {
    constexpr int NT2 = 2 * H / 8;
    const int e = e_, lane = lane_id(), warp = threadIdx.x >> 5;
    const int warps = blockDim.x >> 5, n = P.n;
    const double *psw = P.W(gnn_role(e, 0, 0));
    double *Bf = gsm;
    stage_frag(Bf, 7, 2, NT2, [&](int kk, int j) {
        return j < H ? psw[kk * H + j] : psw[(7 + kk) * H + (j - H)];
    });
    __syncthreads();
    double *H0 = P.H[e][0];
    const int r = lane >> 2, c = lane & 3;
    const int rows = P.rows;
    for (int tile = bx_ * warps + warp; tile * 8 < rows; tile += gx_ * warps) {
        const int v = tile * 8 + r;  // row
        double acc[NT2][2];
        zero_acc(acc);
#pragma unroll
        for (int kt = 0; kt < 2; ++kt) {
            const int col = kt * 4 + c;
            double a = 0.0;
            if (v < rows && col < 7) {
                if (P.ps_dev) {
                    // per_step input row [x_static | dyn], dyn = (1, (d+1)/D) once
                    // placed (reference policy.py:390-391); materialised for phi
                    const int dv = P.ps_dev[v];
                    a = col < 5 ? P.x[(size_t)(v % n) * 5 + col]
                        : dv < 0 ? 0.0 : col == 5 ? 1.0 : __ddiv_rn((double)(dv + 1), (double)P.D);
                    H0[(size_t)v * 7 + col] = a;
                } else {
                    a = H0[(size_t)v * 7 + col];
                }
            }
            if (P.tc && v < rows) {  // bf16 encoder: H0 as split planes, X_0[:, 0:8)
                const float af = (float)a;
                const __nv_bfloat16 hi = __float2bfloat16_rn(af);
                P.Xh[e][0][(size_t)v * 64 + col] = __bfloat16_as_ushort(hi);
                P.Xl[e][0][(size_t)v * 64 + col] =
                    __bfloat16_as_ushort(__float2bfloat16_rn(af - __bfloat162float(hi)));
            }
#pragma unroll
            for (int nt = 0; nt < NT2; ++nt) dmma(acc[nt], a, Bf[(kt * NT2 + nt) * 32 + lane]);
        }
        if (v < rows) {
#pragma unroll
            for (int nt = 0; nt < NT2; ++nt) {
                const int col = nt * 8 + c * 2;
                if (P.tc) {  // fp32 P/Q for the bf16 encoder's aggregation
                    float *dst = col < H ? (float *)P.Pm[e][0] + (size_t)v * H + col
                                         : (float *)P.Qm[e][0] + (size_t)v * H + (col - H);
                    *(float2 *)dst = make_float2((float)acc[nt][0], (float)acc[nt][1]);
                    continue;
                }
                double *dst = col < H ? P.Pm[e][0] + (size_t)v * H + col
                                      : P.Qm[e][0] + (size_t)v * H + (col - H);
                *(double2 *)dst = make_double2(acc[nt][0], acc[nt][1]);
            }
        }
    }
}

template <int H>
__global__ void __launch_bounds__(256) gnn_proj0_kernel(DevPolicy P) {
    extern __shared__ __align__(16) double gsm[];
    griddep_launch();
    if (P.n_params)  // the encode's first kernel warms L2 for the later ones
        prefetch_encode_inputs(P, (blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x,
                               gridDim.x * gridDim.y * blockDim.x);
    gnn_proj0_body<H>(P, blockIdx.y, blockIdx.x, gridDim.x, gsm);
}

// A fragment of k-step kt taken from a D fragment held in registers (the
// previous GEMM's output, columns 8nt + 2c' + i on lane 4r + c'): lane (r, c)
// needs column 4kt + c, which lives on lane 4r + 2(kt&1) + c/2 as element c&1
// of n-tile kt/2.  Two shuffles per k-step; kt must be a compile-time index.
template <int NT>
__device__ __forceinline__ double d_to_a(const double (&acc)[NT][2], int kt) {
    const int lane = lane_id();
    const int src = (lane & ~3) + 2 * (kt & 1) + ((lane & 3) >> 1);
    const double x0 = __shfl_sync(FP_FULL_MASK, acc[kt >> 1][0], src);
    const double x1 = __shfl_sync(FP_FULL_MASK, acc[kt >> 1][1], src);
    return (lane & 1) ? x1 : x0;
}

// shared-memory doubles (weight fragments) of gnn_node_kernel for (H, k, last)
__host__ __device__ inline int node_smem_doubles(int H, int k, bool last) {
    const int NT = H / 8, dk = k == 0 ? 7 : H, KT1 = (dk + H + 3) / 4;
    int c = KT1 * NT * 32;                      // phi
    if (!last) c += (H / 4) * 2 * NT * 32;      // next psi [Ws | Wd]
    else c += 2 * 2 * NT * 32 + (2 * H / 4) * NT * 32 + (H / 4) * NT * 32;  // zs, zp, w1ad, w1b
    return c;
}

// ---------------------------------------------------------------------------
// Node MLPs of round k (DMMA): phi update + next projections or head tables.
// A operands come straight from global memory into fragment registers (each
// k-step is one 32-byte sector per vertex row) or, for the chained GEMMs,
// from the previous GEMM's accumulators by shuffles -- no shared-memory
// staging of activations, so the only shared memory is the weights.
// ---------------------------------------------------------------------------
template <int H, bool K0, bool BWD>
__device__ __forceinline__ void gnn_node_body(const DevPolicy &P, int k, int last, int e_, int bx_, int gx_, double *gsm) {
    constexpr int NT = H / 8;
    constexpr int DK = K0 ? 7 : H;
    constexpr int K1 = DK + H;
    constexpr int KT1 = (K1 + 3) / 4;
    const int e = e_, lane = lane_id(), warp = threadIdx.x >> 5;
    const int warps = blockDim.x >> 5, n = P.n;
    const double s = P.slope;
    const bool feeds_sel = e == 0;
    const bool feeds_plc = P.n_enc == 1 || e == 1;
    const double *phw = P.W(gnn_role(e, k, 2)), *phb = P.W(gnn_role(e, k, 3));

    double *o = gsm;
    double *Fphi = o;
    stage_frag(Fphi, K1, KT1, NT, [&](int kk, int j) { return phw[kk * H + j]; });
    o += KT1 * NT * 32;
    double *Fnext = nullptr, *Fzs = nullptr, *Fzp = nullptr, *Fw1ad = nullptr, *Fw1b = nullptr;
    if (!last) {
        const double *nw = P.W(gnn_role(e, k + 1, 0));
        Fnext = o;
        stage_frag(Fnext, H, H / 4, 2 * NT, [&](int kk, int j) {
            return j < H ? nw[kk * H + j] : nw[(H + kk) * H + (j - H)];
        });
    } else {
        if (feeds_sel) {
            const double *zw = P.W(PR_SEL_Z_W);
            Fzs = o;
            stage_frag(Fzs, 5, 2, NT, [&](int kk, int j) { return zw[kk * H + j]; });
        }
        o += 2 * NT * 32;
        if (feeds_plc) {
            const double *zw = P.W(PR_PLC_Z_W), *w1 = P.W(PR_PLC_H1_W);
            Fzp = o;
            stage_frag(Fzp, 5, 2, NT, [&](int kk, int j) { return zw[kk * H + j]; });
            Fw1ad = o + 2 * NT * 32;
            stage_frag(Fw1ad, 2 * H, 2 * H / 4, NT, [&](int kk, int j) {
                return kk < H ? w1[kk * H + j] : w1[(3 * H + kk - H) * H + j];
            });
            Fw1b = Fw1ad + (2 * H / 4) * NT * 32;
            stage_frag(Fw1b, H, H / 4, NT, [&](int kk, int j) { return w1[(H + kk) * H + j]; });
        }
    }
    __syncthreads();
    griddep_wait();  // H_k / agg_k come from the previous kernels

    const double *Hk = P.H[e][k];
    const double *agg = P.AG[e][k];
    const int r = lane >> 2, c = lane & 3, c2 = c * 2;
    const int rows = P.rows;
    for (int tile = bx_ * warps + warp; tile * 8 < rows; tile += gx_ * warps) {
        const int v = tile * 8 + r;  // row (= vertex unless batched)
        const bool vok = v < rows;
        // ---- phi: A = [H_k | agg] (8 x K1) from global, fragments in registers ----
        double a1[KT1];
#pragma unroll
        for (int kt = 0; kt < KT1; ++kt) {
            const int col = kt * 4 + c;
            double x = 0.0;
            if (vok) {
                if (col < DK) x = Hk[(size_t)v * DK + col];
                else if (col < K1) x = agg[(size_t)v * H + col - DK];
            }
            a1[kt] = x;
        }
        double acc[NT][2];
        zero_acc(acc);
#pragma unroll
        for (int kt = 0; kt < KT1; ++kt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) dmma(acc[nt], a1[kt], Fphi[(kt * NT + nt) * 32 + lane]);
        // U + b -> H' = leaky(U), kept in the D fragment for the chained GEMMs
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int col = nt * 8 + c2;
            const double u0 = acc[nt][0] + phb[col], u1 = acc[nt][1] + phb[col + 1];
            acc[nt][0] = gleaky(u0, s);
            acc[nt][1] = gleaky(u1, s);
            if (vok) {
                *(double2 *)(P.H[e][k + 1] + (size_t)v * H + col) = make_double2(acc[nt][0], acc[nt][1]);
                if constexpr (BWD) *(double2 *)(P.U[e][k] + (size_t)v * H + col) = make_double2(u0, u1);
            }
        }
        if (!last) {
            double pq[2 * NT][2];
            zero_acc(pq);
#pragma unroll
            for (int kt = 0; kt < H / 4; ++kt) {
                const double a = d_to_a<NT>(acc, kt);
#pragma unroll
                for (int nt = 0; nt < 2 * NT; ++nt) dmma(pq[nt], a, Fnext[(kt * 2 * NT + nt) * 32 + lane]);
            }
            if (vok) {
#pragma unroll
                for (int nt = 0; nt < 2 * NT; ++nt) {
                    const int col = nt * 8 + c2;
                    double *dst = col < H ? P.Pm[e][k + 1] + (size_t)v * H + col
                                          : P.Qm[e][k + 1] + (size_t)v * H + (col - H);
                    *(double2 *)dst = make_double2(pq[nt][0], pq[nt][1]);
                }
            }
            continue;
        }
        // ---- last round: head tables; x = the 5 static features (K padded to 8) ----
        double ax[2];
#pragma unroll
        for (int kt = 0; kt < 2; ++kt) {
            const int col = kt * 4 + c;
            ax[kt] = vok && col < 5 ? P.x[(size_t)(v % n) * 5 + col] : 0.0;
        }
        if (feeds_sel) {
            const double *zb = P.W(PR_SEL_Z_B);
            double z[NT][2];
            zero_acc(z);
#pragma unroll
            for (int kt = 0; kt < 2; ++kt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) dmma(z[nt], ax[kt], Fzs[(kt * NT + nt) * 32 + lane]);
            if (vok)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const int col = nt * 8 + c2;
                    *(double2 *)(P.Zs + (size_t)v * H + col) =
                        make_double2(z[nt][0] + zb[col], z[nt][1] + zb[col + 1]);
                }
        }
        if (feeds_plc) {
            const double *zb = P.W(PR_PLC_Z_B);
            double z[NT][2];
            zero_acc(z);
#pragma unroll
            for (int kt = 0; kt < 2; ++kt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) dmma(z[nt], ax[kt], Fzp[(kt * NT + nt) * 32 + lane]);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const int col = nt * 8 + c2;
                z[nt][0] += zb[col];
                z[nt][1] += zb[col + 1];
                if constexpr (BWD)
                    if (vok) *(double2 *)(P.Zp + (size_t)v * H + col) = make_double2(z[nt][0], z[nt][1]);
            }
            // A = [H' | z] @ [W1a; W1d], G = H' @ W1b
            double a[NT][2], g[NT][2];
            zero_acc(a);
            zero_acc(g);
#pragma unroll
            for (int kt = 0; kt < H / 4; ++kt) {
                const double ah = d_to_a<NT>(acc, kt);
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    dmma(a[nt], ah, Fw1ad[(kt * NT + nt) * 32 + lane]);
                    dmma(g[nt], ah, Fw1b[(kt * NT + nt) * 32 + lane]);
                }
            }
#pragma unroll
            for (int kt = 0; kt < H / 4; ++kt) {
                const double az = d_to_a<NT>(z, kt);
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
                    dmma(a[nt], az, Fw1ad[((H / 4 + kt) * NT + nt) * 32 + lane]);
            }
            if (vok)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const int col = nt * 8 + c2;
                    *(double2 *)(P.A + (size_t)v * H + col) = make_double2(a[nt][0], a[nt][1]);
                    *(double2 *)(P.G + (size_t)v * H + col) = make_double2(g[nt][0], g[nt][1]);
                }
        }
    }
}

template <int H, bool K0, bool BWD>
__global__ void __launch_bounds__(256, 2) gnn_node_kernel(DevPolicy P, int k, int last) {
    extern __shared__ __align__(16) double gsm[];
    griddep_launch();
    gnn_node_body<H, K0, BWD>(P, k, last, blockIdx.y, blockIdx.x, gridDim.x, gsm);
}

// ---------------------------------------------------------------------------
// Explicit path lists (compact graphs): Sb[v] / St[v] = sum of H_sel over the
// b / t path of v, in path order (the reference's sum), one warp per vertex,
// lane = column, four independent row loads in flight.  The SEL head then
// reads them like the forest form's pointer-jumped sums.
// ---------------------------------------------------------------------------
template <int H>
__device__ __forceinline__ void gnn_pathsum_body(const DevPolicy &P, int bx_, int gx_,
                                                 const double *Hs_copy = nullptr,
                                                 const int *const *paths = nullptr,
                                                 double *const *ps_out = nullptr) {
    constexpr int HPL = (H + 31) / 32;
    const int lane = lane_id(), warps = blockDim.x >> 5;
    const double *Hs = Hs_copy ? Hs_copy : P.H[0][P.K];
    for (int v = bx_ * warps + (threadIdx.x >> 5); v < P.n; v += gx_ * warps) {
#pragma unroll
        for (int w = 0; w < 2; ++w) {
            // (paths: shared-memory copies of bp_ptr, bp_idx, tp_ptr, tp_idx)
            const int *pp = paths ? paths[2 * w] : w == 0 ? P.bp_ptr : P.tp_ptr;
            const int *pi = paths ? paths[2 * w + 1] : w == 0 ? P.bp_idx : P.tp_idx;
            const int q0 = pp[v], q1 = pp[v + 1];
            double acc[HPL];
#pragma unroll
            for (int t = 0; t < HPL; ++t) acc[t] = 0.0;
            for (int q = q0; q < q1; q += 4) {
                int u[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) u[i] = q + i < q1 ? pi[q + i] : -1;
#pragma unroll
                for (int t = 0; t < HPL; ++t) {
                    const int j = lane + 32 * t;
                    double x[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) x[i] = u[i] >= 0 && j < H ? Hs[(size_t)u[i] * H + j] : 0.0;
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (u[i] >= 0) acc[t] += x[i];
                }
            }
#pragma unroll
            for (int t = 0; t < HPL; ++t) {
                const int j = lane + 32 * t;
                if (j < H) (ps_out ? ps_out[w] : P.PS[w][0])[(size_t)v * H + j] = acc[t];
            }
        }
    }
}

template <int H>
__global__ void __launch_bounds__(256) gnn_pathsum_kernel(DevPolicy P) {
    griddep_launch();
    griddep_wait();
    gnn_pathsum_body<H>(P, blockIdx.x, gridDim.x);
}

// ---------------------------------------------------------------------------
// SEL head (DMMA): s[v] = leaky([H | Sb | St | Zs] @ head1.w + b1) . head2.w + b2
// A fragments straight from global (path sums from the pointer-jumping
// buffers, or summed along the explicit path lists for compact graphs).
// ---------------------------------------------------------------------------
__host__ __device__ inline int sel_smem_doubles(int H) { return (4 * H / 4) * (H / 8) * 32; }

// PLC constants M = Wy @ W1c (5 x h), c = by @ W1c + b1 (policy.py:218-222), one
// warp: lane = column, the six dot products interleaved (independent chains)
template <int H>
__device__ __forceinline__ void gnn_plc_consts_body(const DevPolicy &P) {
    const int lane = lane_id();
    const double *yw = P.W(PR_PLC_Y_W), *yb = P.W(PR_PLC_Y_B), *w1 = P.W(PR_PLC_H1_W),
                 *b1 = P.W(PR_PLC_H1_B);
    for (int j = lane; j < H; j += 32) {
        double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
        for (int i = 0; i < H; ++i) {
            const double w = w1[(2 * H + i) * H + j];
#pragma unroll
            for (int rr = 0; rr < 5; ++rr) acc[rr] = fma(yw[rr * H + i], w, acc[rr]);
            acc[5] = fma(yb[i], w, acc[5]);
        }
#pragma unroll
        for (int rr = 0; rr < 5; ++rr) P.M[rr * H + j] = acc[rr];
        P.c[j] = acc[5] + b1[j];
    }
}

template <int H, bool BWD>
__device__ __forceinline__ void gnn_sel_body(const DevPolicy &P, int e_, int bx_, int gx_, double *gsm,
                                             const double *Hs_copy = nullptr, bool consts = true,
                                             const double *Sb_copy = nullptr,
                                             const double *St_copy = nullptr) {
    constexpr int NT = H / 8;
    constexpr int KT = H;  // K = 4H
    const int lane = lane_id(), warp = threadIdx.x >> 5;
    const int warps = blockDim.x >> 5, n = P.n;
    const double s = P.slope;
    const double *w1 = P.W(PR_SEL_H1_W), *b1 = P.W(PR_SEL_H1_B), *w2 = P.W(PR_SEL_H2_W),
                 *b2 = P.W(PR_SEL_H2_B);
    double *Fw = gsm;
    stage_frag(Fw, 4 * H, KT, NT, [&](int kk, int j) { return w1[kk * H + j]; });
    __syncthreads();
    // PLC constants (params only) on the grid's LAST warp -- the one with the
    // fewest tiles -- after the block barrier and before the dependency wait,
    // i.e. overlapping the previous kernel's tail instead of holding block 0
    // at its barrier
    if (consts && bx_ == gx_ - 1 && warp == warps - 1) gnn_plc_consts_body<H>(P);
    griddep_wait();  // H_sel and the path sums come from the previous kernels
    const double *Hs = Hs_copy ? Hs_copy : P.H[0][P.K];
    const int rb = P.jump_rounds;
    // path sums: pointer-jumped (forest) or gnn_pathsum (explicit lists)
    const double *Sb = Sb_copy ? Sb_copy : P.forest ? (rb > 0 ? P.PS[0][(rb - 1) & 1] : Hs) : P.PS[0][0];
    const double *St = St_copy ? St_copy : P.forest ? (rb > 0 ? P.PS[1][(rb - 1) & 1] : Hs) : P.PS[1][0];
    const int r = lane >> 2, c = lane & 3, c2 = c * 2;
    for (int tile = bx_ * warps + warp; tile * 8 < n; tile += gx_ * warps) {
        const int v = tile * 8 + r;
        const bool vok = v < n;
        double acc[NT][2];
        zero_acc(acc);
        // 8 k-steps of A loads in flight before their (possibly aliasing)
        // embedding-row stores and the MMAs
        for (int kt0 = 0; kt0 < KT; kt0 += 8) {
            double xs[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int cc = (kt0 + u) * 4 + c, b = cc / H, j = cc - b * H;
                double x = 0.0;
                if (vok && kt0 + u < KT) {
                    if (b == 0) x = Hs[(size_t)v * H + j];
                    else if (b == 3) x = P.Zs[(size_t)v * H + j];
                    else x = (b == 1 ? Sb : St)[(size_t)v * H + j];
                }
                xs[u] = x;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int kt = kt0 + u;
                if (kt >= KT) break;
                if constexpr (BWD)
                    if (vok) P.emb[(size_t)v * 4 * H + kt * 4 + c] = xs[u];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) dmma(acc[nt], xs[u], Fw[(kt * NT + nt) * 32 + lane]);
            }
        }
        double part = 0.0;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int col = nt * 8 + c2 + i;
                const double pre = acc[nt][i] + b1[col];
                if constexpr (BWD)
                    if (vok) P.hidpre[(size_t)v * H + col] = pre;
                part = fma(gleaky(pre, s), w2[col], part);
            }
        part += __shfl_xor_sync(FP_FULL_MASK, part, 1);
        part += __shfl_xor_sync(FP_FULL_MASK, part, 2);
        if (c == 0 && vok) P.s[v] = part + b2[0];
    }
}

template <int H, bool BWD>
__global__ void __launch_bounds__(256, 2) gnn_sel_kernel(DevPolicy P) {
    extern __shared__ __align__(16) double gsm[];
    griddep_launch();
    gnn_sel_body<H, BWD>(P, blockIdx.y, blockIdx.x, gridDim.x, gsm);
}

// ---------------------------------------------------------------------------
// Small graphs: the whole encode in ONE launch, one block per encoder
// (proj0 -> K x (aggregation, node MLPs) -> SEL head on block 0), phases
// separated by block barriers.  Same device bodies as the multi-block
// kernels (bit-identical results); for a few hundred rows the six separate
// launches were latency- and launch-bound.
// ---------------------------------------------------------------------------
constexpr int kSmallEncodeRows = 64;  // one 8-row tile per warp

template <int H, bool BWD, int NTH = 256>
__global__ void __launch_bounds__(NTH, 1) gnn_small_kernel(DevPolicy P) {
    extern __shared__ __align__(16) double gsm[];
    const int e = blockIdx.x;
#ifdef FP_SMALL_TIMING
    long long tt[12]; int nt_ = 0;
#define TT() do { __syncthreads(); tt[nt_++] = clock64(); } while (0)
#else
#define TT() do {} while (0)
#endif
    // no early griddep_launch here: the rollout's blocks would sit on every SM
    // for the whole encode (starving concurrent work on other streams); the
    // implicit trigger at block exit still hides the rollout's launch latency
    if (P.n_params) prefetch_encode_inputs(P, threadIdx.x, blockDim.x);
    TT();
    gnn_proj0_body<H>(P, e, 0, 1, gsm);
    __syncthreads();
    TT();
    for (int k = 0; k < P.K; ++k) {
        gnn_agg_body<H>(P, k, e, 0, 1, gsm);
        __syncthreads();
        TT();
        const int last = k == P.K - 1;
        if (k == 0) gnn_node_body<H, true, BWD>(P, k, last, e, 0, 1, gsm);
        else gnn_node_body<H, false, BWD>(P, k, last, e, 0, 1, gsm);
        __syncthreads();
        TT();
    }
#ifdef FP_SMALL_TIMING
    if (e == 1 && threadIdx.x == 0) {
        printf("blk1: proj0 %lld agg0 %lld node0 %lld agg1 %lld node1 %lld\n", tt[1] - tt[0], tt[2] - tt[1], tt[3] - tt[2], tt[4] - tt[3], tt[5] - tt[4]);
    }
#endif
    if (e == 1) gnn_plc_consts_body<H>(P);  // off the SEL block's critical path
    if (e == 0) {
        // the path sums walk H_sel row by row (dependent index -> row loads):
        // from shared-memory copies of H_sel and the path lists instead of
        // L2 round trips
        double *hs = gsm + sel_smem_doubles(H);
        const double *Hs = P.H[0][P.K];
        for (int i = threadIdx.x; i < P.n * H; i += blockDim.x) hs[i] = Hs[i];
        double *ps[2] = {hs + P.n * H, hs + 2 * P.n * H};  // path sums stay on chip
        int *ip = (int *)(hs + 3 * P.n * H);
        const int nb = P.bp_ptr[P.n], ntp = P.tp_ptr[P.n];
        const int *paths[4] = {ip, ip + P.n + 1, ip + P.n + 1 + nb, ip + 2 * (P.n + 1) + nb};
        for (int i = threadIdx.x; i <= P.n; i += blockDim.x) {
            ((int *)paths[0])[i] = P.bp_ptr[i];
            ((int *)paths[2])[i] = P.tp_ptr[i];
        }
        for (int i = threadIdx.x; i < nb; i += blockDim.x) ((int *)paths[1])[i] = P.bp_idx[i];
        for (int i = threadIdx.x; i < ntp; i += blockDim.x) ((int *)paths[3])[i] = P.tp_idx[i];
        __syncthreads();
        TT();
        gnn_pathsum_body<H>(P, 0, 1, hs, paths, ps);
        __syncthreads();
        TT();
        gnn_sel_body<H, BWD>(P, 0, 0, 1, gsm, hs, P.n_enc == 1, ps[0], ps[1]);
        TT();
#ifdef FP_SMALL_TIMING
        if (threadIdx.x == 0) {
            printf("blk0: proj0 %lld agg0 %lld node0 %lld agg1 %lld node1 %lld copy %lld pathsum %lld sel %lld\n", tt[1] - tt[0], tt[2] - tt[1], tt[3] - tt[2], tt[4] - tt[3], tt[5] - tt[4], tt[6] - tt[5], tt[7] - tt[6], tt[8] - tt[7]);
        }
#endif
    }
#undef TT
}


}  // namespace fp
