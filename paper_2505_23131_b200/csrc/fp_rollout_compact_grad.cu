#define FP_GRAD true
// Explicit instantiations of the compact (shared-memory) REINFORCE rollout
// kernels and the Stage-II replay of their decision records.
#include "fp_rollout.cuh"

namespace fp {
#define FP_INST(MAXD, HPL)                                                                  \
    template int launch_rollout<MAXD, HPL, FP_GRAD>(const fp_problem *, const fp_policy *,  \
                                                    const fp_rollout_args &, cudaStream_t); \
    template int launch_plc_replay<MAXD, HPL>(                                              \
        const fp_problem *, const fp_policy *, const double *, const double *,              \
        const int32_t *, const double *, double, int, double *, int64_t *, cudaStream_t);
FP_INST(4, 1) FP_INST(8, 1) FP_INST(16, 1) FP_INST(32, 1) FP_INST(8, 2) FP_INST(16, 2) FP_INST(32, 2)
}  // namespace fp

using namespace fp;
extern "C" {
#ifdef FP_PHASE_PROFILE
int fp_phase_read_grad(unsigned long long *cycles, unsigned long long *counts, int reset) {
    cudaMemcpyFromSymbol(cycles, g_phase_cycles, sizeof(unsigned long long) * 64);
    cudaMemcpyFromSymbol(counts, g_phase_count, sizeof(unsigned long long) * 64);
    if (reset) {
        unsigned long long z[64] = {0};
        cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
        cudaMemcpyToSymbol(g_phase_count, z, sizeof(z));
    }
    return FP_OK;
}
#endif
}
