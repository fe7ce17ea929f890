// Shared device helpers for the flowplace B200 kernels (sm_100a).
#pragma once

#include <cstdlib>

#include <cstdint>
#include <cuda_runtime.h>

#define FP_FULL_MASK 0xffffffffu

// Phase profiling (profiling build only: -DFP_PHASE_PROFILE).  Accumulates
// clock64 deltas per phase into g_phase_cycles[phase] (one atomic per warp
// per phase per step, lane 0) -- never compiled into the product library.
#ifdef FP_PHASE_PROFILE
static __device__ unsigned long long g_phase_cycles[64];
static __device__ unsigned long long g_phase_count[64];
// per-warp register accumulators (constant phase ids), flushed once per warp
#define FP_PHASE_DECL unsigned long long fp_acc_[32] = {0}; unsigned fp_cnt_[32] = {0}
#define FP_PHASE_BEGIN(var) long long var = clock64()
#define FP_PHASE_END(var, id)                                     \
    do {                                                          \
        long long now_ = clock64();                               \
        fp_acc_[(id) & 31] += (unsigned long long)(now_ - var);   \
        fp_cnt_[(id) & 31] += 1;                                  \
        var = now_;                                               \
    } while (0)
#define FP_PHASE_FLUSH(base)                                                    \
    do {                                                                        \
        if ((threadIdx.x & 31) == 0)                                            \
            for (int i_ = 0; i_ < 32; ++i_)                                     \
                if (fp_cnt_[i_]) {                                              \
                    atomicAdd(&g_phase_cycles[(base) + i_], fp_acc_[i_]);        \
                    atomicAdd(&g_phase_count[(base) + i_], (unsigned long long)fp_cnt_[i_]); \
                }                                                               \
    } while (0)
// milestone of an episode (slots 40..47): cycles since the block started
#define FP_MARK(id, t0)                                                        \
    do {                                                                       \
        if ((threadIdx.x & 31) == 0) {                                         \
            atomicAdd(&g_phase_cycles[id], (unsigned long long)(clock64() - (t0))); \
            atomicAdd(&g_phase_count[id], 1ull);                               \
        }                                                                      \
    } while (0)
#define FP_T0_DECL(var) const long long var = clock64()
#else
#define FP_PHASE_DECL
#define FP_PHASE_BEGIN(var)
#define FP_PHASE_END(var, id)
#define FP_PHASE_FLUSH(base)
#define FP_MARK(id, t0)
#define FP_T0_DECL(var)
#endif

namespace fp {

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Programmatic dependent launch (PDL): a kernel launched with
// programmatic stream serialization may start while its predecessor drains;
// griddep_wait() blocks until the predecessor grid has completed and its
// writes are visible (a no-op for an ordinary launch), griddep_launch() lets
// the successor start its prologue.  Every PDL-launched kernel calls
// griddep_wait() before touching its predecessors' outputs (and so keeps the
// completion order transitive).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

#ifndef __CUDACC_RTC__
// host: launch `kern` with programmatic stream serialization (FP_PDL=0: off)
inline bool pdl_enabled() {
    static const bool on = !(getenv("FP_PDL") && atoi(getenv("FP_PDL")) == 0);
    return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
    if (!pdl_enabled()) {
        kern<<<grid, block, smem, st>>>(args...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}
#endif

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FP_FULL_MASK, v, o);
    return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FP_FULL_MASK, v, o));
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FP_FULL_MASK, v, o));
    return v;
}

// CPython >= 3.12 builtin sum() over floats (bltinmodule.c): Neumaier
// compensation, the compensation added once at the end when nonzero and
// finite.  The reference sums predecessor FLOPs with sum()
// (flowplace/policy.py:243), so the device feature needs the same rounding.
struct NeuSum {
    double s = 0.0, c = 0.0;
    __device__ __forceinline__ void add(double x) {
        const double t = __dadd_rn(s, x);
        c = __dadd_rn(c, fabs(s) >= fabs(x) ? __dadd_rn(__dsub_rn(s, t), x)
                                            : __dadd_rn(__dsub_rn(x, t), s));
        s = t;
    }
    __device__ __forceinline__ double value() const {
        return (c != 0.0 && isfinite(c)) ? __dadd_rn(s, c) : s;
    }
};

// Order-preserving map double -> uint64 (total order for non-NaN values).
__device__ __forceinline__ uint64_t f64_key(double x) {
    const uint64_t b = (uint64_t)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double f64_unkey(uint64_t k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k));
}

// Exact fp64 min / max across the warp with two integer REDUX steps
// (hi word, then lo word among lanes holding the extreme hi word).
__device__ __forceinline__ double warp_min_redux(double x) {
    const uint64_t k = f64_key(x);
    const unsigned hi = __reduce_min_sync(FP_FULL_MASK, (unsigned)(k >> 32));
    const unsigned lo = __reduce_min_sync(FP_FULL_MASK, (unsigned)(k >> 32) == hi ? (unsigned)k
                                                                               : 0xffffffffu);
    return f64_unkey(((uint64_t)hi << 32) | lo);
}
__device__ __forceinline__ double warp_max_redux(double x) {
    const uint64_t k = f64_key(x);
    const unsigned hi = __reduce_max_sync(FP_FULL_MASK, (unsigned)(k >> 32));
    const unsigned lo = __reduce_max_sync(FP_FULL_MASK, (unsigned)(k >> 32) == hi ? (unsigned)k : 0u);
    return f64_unkey(((uint64_t)hi << 32) | lo);
}

// Inclusive prefix sum over the first 2^LOG lanes (lane order).
template <int LOG, typename T>
__device__ __forceinline__ T warp_scan_pow2(T v) {
    const int l = lane_id();
#pragma unroll
    for (int i = 0; i < LOG; ++i) {
        const int o = 1 << i;
        T u = __shfl_up_sync(FP_FULL_MASK, v, o);
        if ((l & ((1 << LOG) - 1)) >= o) v += u;
    }
    return v;
}

// Inclusive prefix sum across the warp (lane order).
template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
    const int l = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(FP_FULL_MASK, v, o);
        if (l >= o) v += u;
    }
    return v;
}

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11).  Counter = (episode, step, head, 0),
// key = (seed lo, seed hi).  Known-answer vectors checked in the tests.
// ---------------------------------------------------------------------------
struct U4 { uint32_t x, y, z, w; };

__host__ __device__ __forceinline__ void mulhilo32(uint32_t a, uint32_t b, uint32_t& hi,
                                                   uint32_t& lo) {
    uint64_t p = (uint64_t)a * (uint64_t)b;
    hi = (uint32_t)(p >> 32);
    lo = (uint32_t)p;
}

__host__ __device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo32(0xD2511F53u, c.x, hi0, lo0);
        mulhilo32(0xCD9E8D57u, c.z, hi1, lo1);
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    }
    return c;
}

// Two uniforms in [0, 1) with 53 random bits each.
__host__ __device__ __forceinline__ void uniform2(U4 r, double& u1, double& u2) {
    const double s = 1.0 / 9007199254740992.0;  // 2^-53
    u1 = (double)((((uint64_t)r.y << 32) | r.x) >> 11) * s;
    u2 = (double)((((uint64_t)r.w << 32) | r.z) >> 11) * s;
}

// Per-step Philox draws, 32 steps at a time: lane j computes the draw of
// step (32*floor(step/32) + j) once, the step reads it with two shuffles --
// keeps the 10-round Philox off every step's dependent chain.  Call once per
// step from all 32 lanes (warp-uniform).
__device__ __forceinline__ void step_draw(int step, uint32_t ctr_ep, uint32_t head, uint32_t k0,
                                          uint32_t k1, double &c1, double &c2, double &u1,
                                          double &u2) {
    if ((step & 31) == 0)
        uniform2(philox4x32_10(U4{ctr_ep, (uint32_t)(step + (threadIdx.x & 31)), head, 0u}, k0, k1),
                 c1, c2);
    u1 = __shfl_sync(FP_FULL_MASK, c1, step & 31);
    u2 = __shfl_sync(FP_FULL_MASK, c2, step & 31);
}

}  // namespace fp
