// Dependent-chain latencies on this GPU, in cycles per loop trip (about 19 of
// which are the loop itself): DFMA, DADD, FFMA, SHFL (32-bit and a double),
// LDS, exp / log / sqrt_rn / rcp / div_rn / rsqrt (fp64), fmax, REDUX.  One warp,
// clock64 around 256-long chains.  Measured on B200.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/lat tools/micro/lat.cu
#include <cstdio>
#include <cuda_runtime.h>
#define N 256
__global__ void k(double *out, long long *cyc, double x0, float f0) {
    double x = x0 + threadIdx.x * 1e-9; float f = f0 + threadIdx.x;
    int i0 = threadIdx.x;
    __shared__ double sm[64];
    sm[threadIdx.x] = x; sm[threadIdx.x + 32] = x;
    __syncwarp();
    long long t0, t1;
#define TIME(id, body) t0 = clock64(); _Pragma("unroll 1") for (int r = 0; r < N; ++r) { body; } t1 = clock64(); if (threadIdx.x == 0) cyc[id] = t1 - t0;
    TIME(0, x = fma(x, 1.0000001, 1e-7));
    TIME(1, x = x + 1e-7);
    TIME(2, f = fmaf(f, 1.0000001f, 1e-7f));
    TIME(3, i0 = __shfl_sync(0xffffffffu, i0, (threadIdx.x + 1) & 31));
    TIME(4, x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31));
    TIME(5, x = sm[(__double_as_longlong(x) & 1) + threadIdx.x]);
    TIME(6, x = exp(x) * 1e-3);
    TIME(7, x = log(x + 2.0));
    TIME(8, x = __dsqrt_rn(x + 1.0));
    TIME(9, x = 1.0 / (x + 1.0));
    TIME(10, x = __ddiv_rn(x, 1.0000001));
    TIME(11, x = fmax(x, 1e-3) );
    TIME(12, {long long b = __double_as_longlong(x); x = __longlong_as_double(b ^ 1);} x = x + 0.0);
    TIME(13, { unsigned v = __reduce_max_sync(0xffffffffu, (unsigned)i0); i0 = v + 1; });
    TIME(14, loop_empty:;);
    TIME(15, x = rsqrt(x + 1.0));
    out[threadIdx.x] = x + f + i0;
}
int main() {
    double *o; long long *c; cudaMalloc(&o, 256); cudaMalloc(&c, 16 * 8);
    k<<<1, 32>>>(o, c, 1.0, 1.0f); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, 1.0, 1.0f); cudaDeviceSynchronize();
    long long h[16]; cudaMemcpy(h, c, 16 * 8, cudaMemcpyDeviceToHost);
    const char *nm[] = {"dfma", "dadd", "ffma", "shfl32", "shfl_f64", "lds_f64", "exp_f64", "log_f64",
                        "sqrt_rn_f64", "rcp_f64", "div_rn_f64", "fmax_f64", "xor+dadd", "redux_max", "loop",
                        "rsqrt_f64"};
    for (int i = 0; i < 16; ++i) printf("%-12s %6.1f cyc/iter\n", nm[i], (double)h[i] / N);
    return 0;
}
