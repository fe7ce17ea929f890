// bf16 tensor-core (tcgen05 + TMA) node MLPs of the GNN encoder -- the
// selectable fast encoder (fp_policy_set_encoder(pol, FP_ENCODER_TC)).
//
// The fp64 DMMA encoder (fp_gnn.cuh) reproduces the reference to 1e-11; this
// one trades that for tensor-core throughput on the B x n-row batches of the
// per_step mode and on 100k+-op graphs.  Operands are bf16 "split" pairs
// (x = hi + lo, ~16 significant bits): every product is hi*hi + lo*hi +
// hi*lo accumulated in fp32 TMEM, so results stay within ~1e-5 relative of
// fp64 -- well inside the 1e-3 the north star allows a bf16 MLP -- while the
// kernel remains HBM-bound (3 MMAs per k-step cost nothing next to the tile
// loads).
//
// Per 128-row tile of round k (one persistent CTA per SM, 6 warps):
//   warp 0    TMA producer: X_k tile = [H_k | agg_k] as hi and lo bf16 planes
//             (128 x 64, 128B-swizzled K-major), double-buffered stages;
//   warp 1    TMEM owner + MMA issuer (one elected lane);
//   warps 2-5 epilogue (TMEM lane quarter = warp % 4, one row per thread).
//   GEMM1  U = X_k . phi_k            (K 64, N H)        -> D1
//   epi 1  H' = leaky(U + b): written to X_{k+1}[:, 0:H) planes (next round's
//          A operand) and to the shared A2 tile (hi / lo) for GEMM2
//   GEMM2  [P | Q] = H' . [psi_src | psi_dst]_{k+1}  (K H, N 2H)   (not last)
//          or A = [H' | zp] . [W1a; W1d], G = H' . W1b              (last)
//   epi 2  P / Q (fp64, read by the aggregation kernel) or H_K, A, G, Zs
//          (fp64, read by the SEL / PLC steps).
// Round k's aggregation kernel writes agg_k's planes into X_k[:, H:2H).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <string>

#include "fp_policy.cuh"
#include "fp_tc.cuh"

namespace fp {

void set_error(const std::string &msg);

namespace {

constexpr int kTcRows = 128;             // M per tile (TMEM lanes)
constexpr int kTcK = 64;                 // X row: 64 bf16 = 128 bytes = one swizzle atom
constexpr int kTcTileBytes = kTcRows * 128;  // one plane of one X tile (16 KB)
constexpr int kTcStages = 2;

// ---------------------------------------------------------------------------
// driver entry point for the tensor-map encoder (no -lcuda link)
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

}  // namespace

// Tensor map of a [rows][64] bf16 plane (row pitch 128 bytes), box 128 x 64,
// 128-byte swizzle (the UMMA K-major SW128 layout).
int tc_plane_map(CUtensorMap *map, const void *plane, int64_t rows) {
    auto fn = encode_fn();
    if (!fn) { set_error("cuTensorMapEncodeTiled unavailable"); return FP_ERR_CUDA; }
    const cuuint64_t dims[2] = {(cuuint64_t)kTcK, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)kTcK * 2};
    const cuuint32_t box[2] = {(cuuint32_t)kTcK, (cuuint32_t)kTcRows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(plane), dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed"); return FP_ERR_CUDA; }
    return FP_OK;
}

// ---------------------------------------------------------------------------
// Weight staging: W^T (N rows x K) as hi / lo bf16 planes in the SW128
// K-major layout; w(k, n) supplies the fp64 weight (0 beyond the matrix).
// ---------------------------------------------------------------------------
template <typename F>
__device__ __forceinline__ void stage_wt(uint8_t *hi, uint8_t *lo, int N, F w) {
    for (int i = threadIdx.x; i < N * kTcK; i += blockDim.x) {
        const int n = i / kTcK, k = i % kTcK;
        const float x = (float)w(k, n);
        __nv_bfloat16 h, l;
        tc::split_bf16(x, h, l);
        const uint32_t o = tc::sw128_off(n, k);
        *(__nv_bfloat16 *)(hi + o) = h;
        *(__nv_bfloat16 *)(lo + o) = l;
    }
}

// D (+)= A . B^T over K = 16 * ksteps with the three split products.
__device__ __forceinline__ void mma_split(uint32_t d, const uint8_t *ahi, const uint8_t *alo,
                                          const uint8_t *bhi, const uint8_t *blo, int ksteps,
                                          uint32_t idesc, bool acc0) {
#pragma unroll 1
    for (int ks = 0; ks < ksteps; ++ks) {
        const uint32_t off = 32u * ks;
        const uint64_t ah = tc::sw128_desc(ahi, off), al = tc::sw128_desc(alo, off);
        const uint64_t bh = tc::sw128_desc(bhi, off), bl = tc::sw128_desc(blo, off);
        tc::mma_bf16(d, ah, bh, idesc, acc0 || ks > 0);
        tc::mma_bf16(d, al, bh, idesc, true);
        tc::mma_bf16(d, ah, bl, idesc, true);
    }
}

// ---------------------------------------------------------------------------
// Self test: out[M][N] (fp32) = X[M][64] . W[64][N] with X given as hi / lo
// bf16 planes (TMA) and W as fp64 -- validates the TMA / descriptor / MMA /
// TMEM path against a host reference (tests/test_tc_gpu.py).
// ---------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(128) tc_gemm_selftest_kernel(
    const __grid_constant__ CUtensorMap mhi, const __grid_constant__ CUtensorMap mlo,
    const double *__restrict__ W, float *__restrict__ out, int M) {
    extern __shared__ __align__(1024) uint8_t tc_smem_raw[];
    uint8_t *sm = (uint8_t *)(((uintptr_t)tc_smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *ahi = sm, *alo = sm + kTcTileBytes;
    uint8_t *bhi = alo + kTcTileBytes, *blo = bhi + N * 128;
    __shared__ uint64_t bar_full, bar_mma;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row0 = blockIdx.x * kTcRows;
    stage_wt(bhi, blo, N, [&](int k, int n) { return W[(size_t)k * N + n]; });
    if (threadIdx.x == 0) {
        tc::mbar_init(&bar_full, 1);
        tc::mbar_init(&bar_mma, 1);
        tc::fence_mbar_init();
    }
    if (warp == 1) tc::tmem_alloc<64>(&tmem_base);
    tc::fence_proxy_async_smem();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tm = tmem_base;
    if (threadIdx.x == 0) {
        tc::mbar_arrive_expect_tx(&bar_full, 2 * kTcTileBytes);
        tc::tma_load_2d(ahi, &mhi, &bar_full, 0, row0);
        tc::tma_load_2d(alo, &mlo, &bar_full, 0, row0);
        tc::mbar_wait(&bar_full, 0);
        tc::tc_fence_after();
        mma_split(tm, ahi, alo, bhi, blo, kTcK / 16, tc::idesc_bf16_f32(kTcRows, N), false);
        tc::mma_commit(&bar_mma);
    }
    __syncwarp();
    tc::mbar_wait(&bar_mma, 0);
    tc::tc_fence_after();
    const int row = row0 + warp * 32 + lane;
#pragma unroll
    for (int c = 0; c < N; c += 16) {
        float v[16];
        tc::tmem_ld16(tm + ((uint32_t)(warp * 32) << 16) + c, v);
        if (row < M)
#pragma unroll
            for (int i = 0; i < 16; ++i) out[(size_t)row * N + c + i] = v[i];
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_free<64>(tm);
}

// ---------------------------------------------------------------------------
// The node-MLP kernel of round k (see the file header).  Persistent: CTA
// (x, e) walks 128-row tiles t = x, x + gridDim.x, ... of encoder e.
// ---------------------------------------------------------------------------
// NG epilogue groups of 4 warps (one per TMEM lane quarter), each with its
// own TMEM accumulator set (128 columns) and A2 tile: tiles it = g, g + NG,
// ... go to group g, so NG tiles are in their epilogues at once while the
// MMA warp runs one tile ahead (GEMM1 of tile it before GEMM2 of it - 1).
constexpr int kTcGroups = 4;
constexpr int kTcThreadsG = 96 + 128 * kTcGroups;

template <int H>
struct TcSmem {
    static constexpr int kX = kTcStages * 2 * kTcTileBytes;  // X stages (hi, lo)
    static constexpr int kA2 = 2 * kTcTileBytes;             // per group: H' (| zp), hi / lo
    static constexpr int kB1 = 2 * H * 128;                  // phi^T, hi / lo
    static constexpr int kB2 = 2 * 2 * H * 128;              // [psi_s | psi_d]^T or W1ad^T + W1b^T
    static constexpr int kBytes = kX + kTcGroups * kA2 + kB1 + kB2;
};

__device__ __forceinline__ float leakyf(float x, float s) { return x > 0.f ? x : s * x; }

// 16 consecutive split values of one row: into a SW128 tile (two 16B chunks
// per plane) and, when `g_hi` is set, into a global [rows][64] plane pair
__device__ __forceinline__ void put16(uint8_t *hi, uint8_t *lo, int row, int col0,
                                      const float (&v)[16], uint16_t *g_hi = nullptr,
                                      uint16_t *g_lo = nullptr, int64_t grow = 0) {
#pragma unroll
    for (int c = 0; c < 16; c += 8) {
        uint32_t ph[4], pl[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            __nv_bfloat16 h0, l0, h1, l1;
            tc::split_bf16(v[c + 2 * i], h0, l0);
            tc::split_bf16(v[c + 2 * i + 1], h1, l1);
            ph[i] = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
            pl[i] = (uint32_t)__bfloat16_as_ushort(l0) | ((uint32_t)__bfloat16_as_ushort(l1) << 16);
        }
        const uint4 vh = make_uint4(ph[0], ph[1], ph[2], ph[3]);
        const uint4 vl = make_uint4(pl[0], pl[1], pl[2], pl[3]);
        const uint32_t o = tc::sw128_off(row, col0 + c);
        *(uint4 *)(hi + o) = vh;
        *(uint4 *)(lo + o) = vl;
        if (g_hi) {
            *(uint4 *)(g_hi + grow * 64 + col0 + c) = vh;
            *(uint4 *)(g_lo + grow * 64 + col0 + c) = vl;
        }
    }
}


// One warp's 32 consecutive rows, 2H fp32 values per row (thread = row):
// two [rows][H] outputs A (values [0, H)) and B ([H, 2H)), fp32 or fp64.
// The rows of a warp are one contiguous block of each output, so the values
// go through `stg` (8 KB at H = 32; 16-byte chunks XOR-swizzled by row) and
// leave as coalesced 16-byte row stores (lanes [0, H/2): A row, the rest: B).
template <int H, bool F64>
__device__ __forceinline__ void warp_store_rows(uint8_t *stg, int lane, const uint32_t (&v)[2 * H],
                                                int64_t row0, int64_t rows, void *outA,
                                                void *outB) {
    constexpr int CH = 2 * H / 4;  // 16-byte chunks per staged row
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const int pc = c ^ (lane & (CH - 1));
        *(uint4 *)(stg + lane * (2 * H * 4) + pc * 16) =
            make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    }
    __syncwarp();
    constexpr int LPR = H / 2;  // lanes per half-row, 2 values each
    void *dst = lane / LPR ? outB : outA;
    if (lane < 2 * LPR && dst) {
        const int half = lane / LPR, li = lane % LPR, col = half * H + 2 * li;
#pragma unroll 4
        for (int r = 0; r < 32; ++r) {
            if (row0 + r >= rows) break;
            const int pc = (col / 4) ^ (r & (CH - 1));
            const float2 f = *(const float2 *)(stg + r * (2 * H * 4) + pc * 16 + (col % 4) * 4);
            const int64_t o = (row0 + r) * H + 2 * li;
            if (F64) *(double2 *)((double *)dst + o) = make_double2(f.x, f.y);
            else *(float2 *)((float *)dst + o) = f;
        }
    }
    __syncwarp();
}

template <int H>
__global__ void __launch_bounds__(kTcThreadsG, 1)
tc_node_kernel(const __grid_constant__ CUtensorMap mx_hi0, const __grid_constant__ CUtensorMap mx_lo0,
               const __grid_constant__ CUtensorMap mx_hi1, const __grid_constant__ CUtensorMap mx_lo1,
               DevPolicy P, int k, int last) {
    static_assert(H == 16 || H == 32, "tensor-core encoder: hidden 16 or 32");
    using L = TcSmem<H>;
    constexpr int NG = kTcGroups;
    extern __shared__ __align__(1024) uint8_t tc_smem_raw[];
    // 1024-byte aligned by offset arithmetic on the shared array, so the
    // compiler keeps the shared state space (STS, not generic stores)
    uint8_t *sm = tc_smem_raw + ((1024u - (tc::smem_u32(tc_smem_raw) & 1023u)) & 1023u);
    uint8_t *xs = sm;                       // [stage][hi/lo] tiles
    uint8_t *a2 = sm + L::kX;               // [group][hi/lo] tiles
    uint8_t *b1h = a2 + NG * L::kA2, *b1l = b1h + H * 128;
    uint8_t *b2h = b1h + L::kB1, *b2l = b2h + 2 * H * 128;
    __shared__ uint64_t bar_full[kTcStages], bar_empty[kTcStages];
    __shared__ uint64_t bar_d1[NG], bar_a2[NG], bar_d2[NG], bar_done[NG];
    __shared__ uint32_t tmem_base;
    __shared__ float bphi_s[H];
    __shared__ double zs_s[6 * H], zp_s[6 * H];   // z-head weights (5 x H) + bias (last round)

    const int e = blockIdx.y;
    const CUtensorMap *mh = e == 0 ? &mx_hi0 : &mx_hi1;
    const CUtensorMap *ml = e == 0 ? &mx_lo0 : &mx_lo1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int DK = k == 0 ? 7 : H;
    const bool feeds_sel = e == 0;
    const bool feeds_plc = P.n_enc == 1 || e == 1;
    const double *phw = P.W(gnn_role(e, k, 2)), *phb = P.W(gnn_role(e, k, 3));

    // ---- weights (all threads): phi^T, then the second GEMM's B ----
    stage_wt(b1h, b1l, H, [&](int kk, int n) {
        if (kk < DK) return phw[kk * H + n];
        if (kk >= 32 && kk < 32 + H) return phw[(DK + kk - 32) * H + n];
        return 0.0;
    });
    if (!last) {
        const double *nw = P.W(gnn_role(e, k + 1, 0));
        stage_wt(b2h, b2l, 2 * H, [&](int kk, int n) {
            if (kk >= H) return 0.0;
            return n < H ? nw[kk * H + n] : nw[(H + kk) * H + (n - H)];
        });
    } else if (feeds_plc) {
        // rows [0, H): [W1a; W1d]^T over K = [H' | zp] (64); rows [H, 2H): W1b^T over K = H'
        const double *w1 = P.W(PR_PLC_H1_W);
        stage_wt(b2h, b2l, 2 * H, [&](int kk, int n) {
            if (n < H) {
                if (kk < H) return w1[kk * H + n];
                if (kk >= 32 && kk < 32 + H) return w1[(3 * H + kk - 32) * H + n];
                return 0.0;
            }
            return kk < H ? w1[(H + kk) * H + (n - H)] : 0.0;
        });
    }
    for (int j = threadIdx.x; j < H; j += blockDim.x) bphi_s[j] = (float)phb[j];
    if (last) {
        const double *zsw = P.W(PR_SEL_Z_W), *zsb = P.W(PR_SEL_Z_B);
        const double *zpw = P.W(PR_PLC_Z_W), *zpb = P.W(PR_PLC_Z_B);
        for (int j = threadIdx.x; j < 6 * H; j += blockDim.x) {
            if (feeds_sel) zs_s[j] = j < 5 * H ? zsw[j] : zsb[j - 5 * H];
            if (feeds_plc) zp_s[j] = j < 5 * H ? zpw[j] : zpb[j - 5 * H];
        }
    }
    // A2 columns no epilogue writes (e.g. [H, 32) at H = 16) must read as 0,
    // not as stale bits that could be NaN (NaN * 0 weights = NaN)
    for (int i = threadIdx.x; i < NG * L::kA2 / 16; i += blockDim.x)
        ((uint4 *)a2)[i] = make_uint4(0u, 0u, 0u, 0u);
    if (threadIdx.x == 0) {
        for (int i = 0; i < kTcStages; ++i) {
            tc::mbar_init(&bar_full[i], 1);
            tc::mbar_init(&bar_empty[i], 1);
        }
        for (int g = 0; g < NG; ++g) {
            tc::mbar_init(&bar_d1[g], 1);
            tc::mbar_init(&bar_a2[g], 128);
            tc::mbar_init(&bar_d2[g], 1);
            tc::mbar_init(&bar_done[g], 128);
        }
        tc::fence_mbar_init();
        tc::tma_prefetch(mh);
        tc::tma_prefetch(ml);
    }
    if (warp == 1) tc::tmem_alloc<128 * NG>(&tmem_base);
    tc::fence_proxy_async_smem();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tm = tmem_base;
    const int rows = P.rows;
    const int tiles = (rows + kTcRows - 1) / kTcRows;
    const int my_tiles = blockIdx.x < tiles ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (warp == 0) {
        // ===== TMA producer =====
        if (lane == 0)
            for (int it = 0; it < my_tiles; ++it) {
                const int t = blockIdx.x + it * gridDim.x;
                const int s = it % kTcStages;
                tc::mbar_wait(&bar_empty[s], ((it / kTcStages) & 1) ^ 1);
                uint8_t *dh = xs + s * 2 * kTcTileBytes, *dl = dh + kTcTileBytes;
                tc::mbar_arrive_expect_tx(&bar_full[s], 2 * kTcTileBytes);
                tc::tma_load_2d(dh, mh, &bar_full[s], 0, t * kTcRows);
                tc::tma_load_2d(dl, ml, &bar_full[s], 0, t * kTcRows);
            }
    } else if (warp == 1) {
        // ===== GEMM1 issuer: U = X . phi into accumulator set it % NG =====
        const uint32_t id1 = tc::idesc_bf16_f32(kTcRows, H);
        for (int it = 0; it < my_tiles; ++it) {
            const int g = it % NG, s = it % kTcStages;
            tc::mbar_wait(&bar_full[s], (it / kTcStages) & 1);
            if (it >= NG) tc::mbar_wait(&bar_done[g], ((it / NG) - 1) & 1);
            tc::tc_fence_after();
            if (lane == 0) {
                const uint8_t *xh = xs + s * 2 * kTcTileBytes, *xl = xh + kTcTileBytes;
                mma_split(tm + 128 * g, xh, xl, b1h, b1l, kTcK / 16, id1, false);
                tc::mma_commit(&bar_empty[s]);
                tc::mma_commit(&bar_d1[g]);
            }
            __syncwarp();
        }
    } else if (warp == 2) {
        // ===== GEMM2 issuer (a separate thread: its commits track only its
        // own MMAs, so it never waits behind GEMM1 of later tiles) =====
        const uint32_t id2 = tc::idesc_bf16_f32(kTcRows, last ? H : 2 * H);
        for (int it = 0; it < my_tiles; ++it) {
            const int g = it % NG;
            tc::mbar_wait(&bar_a2[g], (it / NG) & 1);
            tc::tc_fence_after();
            if (lane == 0) {
                const uint8_t *ah = a2 + g * L::kA2, *al = ah + kTcTileBytes;
                const uint32_t d = tm + 128 * g + 64;
                if (!last) {
                    mma_split(d, ah, al, b2h, b2l, H / 16, id2, false);
                } else if (feeds_plc) {
                    // A = [H' | zp] . [W1a; W1d] (K 64), G = H' . W1b (K = H)
                    mma_split(d, ah, al, b2h, b2l, kTcK / 16, id2, false);
                    mma_split(d + H, ah, al, b2h + H * 128, b2l + H * 128, H / 16, id2, false);
                }
                tc::mma_commit(&bar_d2[g]);
            }
            __syncwarp();
        }
    } else {
        // ===== epilogue group g: warps 3 + 4g .. 6 + 4g, TMEM lane quarter warp % 4 =====
        const int g = (warp - 3) >> 2;
        const int q = warp & 3;
        const int rloc = q * 32 + lane;
        const uint32_t tq = tm + 128 * g + ((uint32_t)(q * 32) << 16);
        uint8_t *ah = a2 + g * L::kA2, *al = ah + kTcTileBytes;
        const float slope = (float)P.slope;
        const int n = P.n;
        for (int it = g; it < my_tiles; it += NG) {
            const int t = blockIdx.x + it * gridDim.x;
            const uint32_t ph = (it / NG) & 1;
            const int64_t row = (int64_t)t * kTcRows + rloc;
            const bool ok = row < rows;
            tc::mbar_wait(&bar_d1[g], ph);
            tc::tc_fence_after();
            // H' = leaky(U + b): into the A2 tile (GEMM2's A operand) and, not
            // last, the next round's planes; kept in hv for the last round
            uint32_t hv[2 * H];
            {
                uint32_t d1r[H / 16][16];
#pragma unroll
                for (int c = 0; c < H; c += 16) tc::tmem_ld16_async(tq + c, d1r[c / 16]);
                tc::tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < H; c += 16) {
                    float v[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        v[i] = leakyf(__uint_as_float(d1r[c / 16][i]) + bphi_s[c + i], slope);
                        hv[c + i] = __float_as_uint(v[i]);
                    }
                    if (!last && ok)
                        put16(ah, al, rloc, c, v, P.Xh[e][k + 1], P.Xl[e][k + 1], row);
                    else
                        put16(ah, al, rloc, c, v);
                }
            }
            if (last) {
                // z heads on the CUDA cores (K = 5, weights in shared memory):
                // zp -> A2[:, 32:32+H) for GEMM2, Zs -> hv[H, 2H) (stored below)
                double x5[5];
#pragma unroll
                for (int i = 0; i < 5; ++i) x5[i] = ok ? P.x[(size_t)(row % n) * 5 + i] : 0.0;
                if (feeds_plc) {
#pragma unroll
                    for (int c = 0; c < H; c += 16) {
                        float v[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            double z = zp_s[5 * H + c + i];
#pragma unroll
                            for (int r5 = 0; r5 < 5; ++r5) z = fma(x5[r5], zp_s[r5 * H + c + i], z);
                            v[i] = (float)z;
                        }
                        put16(ah, al, rloc, 32 + c, v);
                    }
                }
                if (feeds_sel) {
#pragma unroll
                    for (int j = 0; j < H; ++j) {
                        double z = zs_s[5 * H + j];
#pragma unroll
                        for (int r5 = 0; r5 < 5; ++r5) z = fma(x5[r5], zs_s[r5 * H + j], z);
                        hv[H + j] = __float_as_uint((float)z);
                    }
                }
            }
            tc::fence_proxy_async_smem();
            tc::tc_fence_before();
            tc::mbar_arrive(&bar_a2[g]);
            tc::mbar_wait(&bar_d2[g], ph);
            tc::tc_fence_after();
            // the group's A2 tile is free once GEMM2 has completed: per-warp
            // staging for the coalesced row stores
            uint8_t *stg = ah + q * 32 * (2 * H * 4);
            const int64_t row0 = (int64_t)t * kTcRows + q * 32;
            if (!last || feeds_plc) {
                // [P | Q] of round k + 1 (fp32; the aggregation adds the bias), or A | G (fp64)
                uint32_t d2r[2 * H];
#pragma unroll
                for (int c = 0; c < 2 * H; c += 16)
                    tc::tmem_ld16_async(tq + 64 + c, *(uint32_t(*)[16])(d2r + c));
                tc::tmem_wait_ld();
                if (!last)
                    warp_store_rows<H, false>(stg, lane, d2r, row0, rows, P.Pm[e][k + 1],
                                              P.Qm[e][k + 1]);
                else
                    warp_store_rows<H, true>(stg, lane, d2r, row0, rows, P.A, P.G);
            }
            if (last) {
                // H_K (fp64, read by the SEL path sums / PLC steps) and Zs
                warp_store_rows<H, true>(stg, lane, hv, row0, rows, P.H[e][k + 1],
                                         feeds_sel ? P.Zs : nullptr);
            }
            tc::tc_fence_before();
            tc::mbar_arrive(&bar_done[g]);
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_free<128 * NG>(tm);
}

template <int H>
static int tc_node_launch_t(const DevPolicy &P, int k, bool last, cudaStream_t st) {
    CUtensorMap m[2][2];
    for (int e = 0; e < 2; ++e) {
        const int ee = e < P.n_enc ? e : 0;
        int rc = tc_plane_map(&m[e][0], P.Xh[ee][k], P.rows);
        if (rc) return rc;
        if ((rc = tc_plane_map(&m[e][1], P.Xl[ee][k], P.rows))) return rc;
    }
    const int smem = 1024 + TcSmem<H>::kBytes;
    const void *kern = (const void *)tc_node_kernel<H>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int tiles = (P.rows + kTcRows - 1) / kTcRows;
    const int gx = std::max(1, std::min(tiles, sms / P.n_enc));
    tc_node_kernel<H><<<dim3(gx, P.n_enc), kTcThreadsG, smem, st>>>(m[0][0], m[0][1], m[1][0],
                                                                    m[1][1], P, k, (int)last);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FP_ERR_CUDA; }
    return FP_OK;
}

int tc_node_launch(const DevPolicy &P, int k, bool last, cudaStream_t st) {
    if (P.h == 32) return tc_node_launch_t<32>(P, k, last, st);
    if (P.h == 16) return tc_node_launch_t<16>(P, k, last, st);
    set_error("the tensor-core encoder needs hidden 16 or 32");
    return FP_ERR_UNSUPPORTED;
}

void tc_set_planes(DevPolicy &P, void *base, int64_t rows) {
    uint8_t *b = (uint8_t *)base;
    const int64_t plane = rows * 64 * 2;
    for (int e = 0; e < P.n_enc; ++e)
        for (int k = 0; k < P.K; ++k) {
            P.Xh[e][k] = (uint16_t *)b;
            P.Xl[e][k] = (uint16_t *)(b + plane);
            b += 2 * plane;
        }
}

}  // namespace fp

using namespace fp;

extern "C" int fp_tc_gemm_selftest(const void *x_hi, const void *x_lo, const double *W,
                                   int32_t N, float *out, int32_t M, void *stream) {
    if (!x_hi || !x_lo || !W || !out || M <= 0 || (N != 32 && N != 64)) {
        set_error("bad tc selftest arguments");
        return FP_ERR_INVALID;
    }
    CUtensorMap mh, ml;
    int rc = tc_plane_map(&mh, x_hi, M);
    if (rc) return rc;
    if ((rc = tc_plane_map(&ml, x_lo, M))) return rc;
    const int smem = 1024 + 2 * kTcTileBytes + 2 * N * 128;
    const void *kern = N == 32 ? (const void *)tc_gemm_selftest_kernel<32>
                               : (const void *)tc_gemm_selftest_kernel<64>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = (M + kTcRows - 1) / kTcRows;
    if (N == 32)
        tc_gemm_selftest_kernel<32><<<grid, 128, smem, (cudaStream_t)stream>>>(mh, ml, W, out, M);
    else
        tc_gemm_selftest_kernel<64><<<grid, 128, smem, (cudaStream_t)stream>>>(mh, ml, W, out, M);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return FP_ERR_CUDA; }
    return FP_OK;
}
