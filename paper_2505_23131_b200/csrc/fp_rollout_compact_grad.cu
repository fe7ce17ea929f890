#define FP_GRAD true
// Explicit instantiations of the compact (shared-memory) rollout kernels.
#include "fp_rollout.cuh"

namespace fp {
#define FP_INST(MAXD, HPL)                                                                  \
    template int launch_rollout<MAXD, HPL, FP_GRAD>(const fp_problem *, const fp_policy *,  \
                                                    const fp_rollout_args &, cudaStream_t);
FP_INST(4, 1) FP_INST(8, 1) FP_INST(16, 1) FP_INST(32, 1) FP_INST(8, 2) FP_INST(16, 2) FP_INST(32, 2)
}  // namespace fp
