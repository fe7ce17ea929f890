// Explicit instantiations of the wide (HBM-resident) rollout kernels.
#include "fp_rollout.cuh"

namespace fp {
#define FP_INST(MAXD, HPL)                                                                  \
    template int launch_rollout_wide<MAXD, HPL>(const fp_problem *, const fp_policy *,      \
                                                const fp_rollout_args &, int64_t *, cudaStream_t);
FP_INST(4, 1) FP_INST(8, 1) FP_INST(16, 1) FP_INST(32, 1) FP_INST(8, 2) FP_INST(16, 2) FP_INST(32, 2)
}  // namespace fp
