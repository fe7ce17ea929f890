// Rollout dispatch + C ABI.  The kernels and their launch templates live in
// fp_rollout.cuh; the template instantiations are spread over
// fp_rollout_compact.cu (REINFORCE rows off / on) and fp_rollout_wide.cu so
// nvcc compiles them in parallel.
#include "fp_rollout.cuh"

namespace fp {

#define FP_ROLLOUT_CONFIGS(X) X(4, 1) X(8, 1) X(16, 1) X(32, 1) X(8, 2) X(16, 2) X(32, 2)
#define FP_DECL(MAXD, HPL)                                                                       \
    extern template int launch_rollout<MAXD, HPL, false>(const fp_problem *, const fp_policy *,  \
                                                         const fp_rollout_args &, cudaStream_t); \
    extern template int launch_rollout<MAXD, HPL, true>(const fp_problem *, const fp_policy *,   \
                                                        const fp_rollout_args &, cudaStream_t);  \
    extern template int launch_rollout_wide<MAXD, HPL>(const fp_problem *, const fp_policy *,    \
                                                       const fp_rollout_args &, int64_t *,       \
                                                       cudaStream_t);                            \
    extern template int launch_plc_replay<MAXD, HPL>(                                            \
        const fp_problem *, const fp_policy *, const double *, const double *, const int32_t *, \
        const double *, double, int, double *, int64_t *, cudaStream_t);
FP_ROLLOUT_CONFIGS(FP_DECL)
#undef FP_DECL

static bool rollout_compact_fits(const fp_problem *p, const fp_policy *pol, bool grad) {
    const DevProblem &PR = p->dev;
    (void)pol; (void)grad;  // REINFORCE records live in the workspace, not shared memory
    const EpLayout L = make_layout(PR.n, PR.W, PR.R, PR.SM, true, 0);
    // the compact SEL chain keeps the candidate bitset in one word per lane
    return PR.n <= 1024 && fp_align(8 * PR.n, 16) + (int64_t)L.bytes <= 227 * 1024;
}

// Compact kernel while it keeps the register-bound 8 episodes per SM resident
// (episode slice <= ~27 KB of shared memory, n up to ~350 at d = 8); past
// that the wide kernel's 8 resident episodes with L2-resident state win
// (measured: n = 500 compact 9.2 ms vs wide 6.3 ms per 1024 episodes).  The
// REINFORCE rows exist only on the compact path, so grad keeps it while it fits.
static bool rollout_use_compact(const fp_problem *p, const fp_policy *pol, bool grad) {
    if (!rollout_compact_fits(p, pol, grad)) return false;
    if (grad) return true;
    const DevProblem &PR = p->dev;
    const EpLayout L = make_layout(PR.n, PR.W, PR.R, PR.SM, true, 0);
    const int64_t smem = fp_align(8 * PR.n, 16) + (int64_t)L.bytes;
    return (228 * 1024) / (smem + 1024) >= 8;
}

template <int MAXD, int HPL>
static int dispatch_grad(const fp_problem *p, const fp_policy *pol, const fp_rollout_args &a,
                         int64_t *ws_needed, cudaStream_t st) {
    const bool grad = a.grad_rows != nullptr;
    const bool wide = (a.flags & FP_FLAG_WIDE) || !rollout_use_compact(p, pol, grad);
    if (wide) {
        if (grad) {
            set_error("REINFORCE rows need the compact (shared-memory) rollout: graph too large");
            return FP_ERR_UNSUPPORTED;
        }
        return launch_rollout_wide<MAXD, HPL>(p, pol, a, ws_needed, st);
    }
    if (ws_needed) {
        *ws_needed = 0;  // REINFORCE records live in grad_rows
        return FP_OK;
    }
    return grad ? launch_rollout<MAXD, HPL, true>(p, pol, a, st)
                : launch_rollout<MAXD, HPL, false>(p, pol, a, st);
}

// Stage-II replay of the PLC decision records + deterministic episode
// reduction (fp_pg_reduce); scratch_bytes != NULL: size query only.
int plc_replay(const fp_problem *p, const fp_policy *pol, const double *rec, const double *gep,
               const int32_t *assign, const double *alpha, double beta, int B, double *scratch,
               int64_t *scratch_bytes, cudaStream_t st) {
    const int D = p->dev.d, h = pol->dev.h;
#define FP_RP(MD, HP) \
    return launch_plc_replay<MD, HP>(p, pol, rec, gep, assign, alpha, beta, B, scratch, scratch_bytes, st)
    if (h <= 32) {
        if (D <= 4) FP_RP(4, 1);
        if (D <= 8) FP_RP(8, 1);
        if (D <= 16) FP_RP(16, 1);
        FP_RP(32, 1);
    }
    if (D <= 8) FP_RP(8, 2);
    if (D <= 16) FP_RP(16, 2);
    FP_RP(32, 2);
#undef FP_RP
}

int per_step_rollout(const fp_problem *p, const fp_policy *pol, const fp_rollout_args &a,
                     int64_t *ws_needed, cudaStream_t st);  // fp_per_step.cu

static int dispatch(const fp_problem *p, const fp_policy *pol, const fp_rollout_args &a,
                    int64_t *ws_needed, cudaStream_t st) {
    if (a.flags & FP_FLAG_PER_STEP) return per_step_rollout(p, pol, a, ws_needed, st);
    const int D = p->dev.d, h = pol->dev.h;
    if (h <= 32) {
        if (D <= 4) return dispatch_grad<4, 1>(p, pol, a, ws_needed, st);
        if (D <= 8) return dispatch_grad<8, 1>(p, pol, a, ws_needed, st);
        if (D <= 16) return dispatch_grad<16, 1>(p, pol, a, ws_needed, st);
        return dispatch_grad<32, 1>(p, pol, a, ws_needed, st);
    }
    if (D <= 8) return dispatch_grad<8, 2>(p, pol, a, ws_needed, st);
    if (D <= 16) return dispatch_grad<16, 2>(p, pol, a, ws_needed, st);
    return dispatch_grad<32, 2>(p, pol, a, ws_needed, st);
}

}  // namespace fp

using namespace fp;

extern "C" {



int fp_grad_ep_stride(const fp_policy *pol, int32_t d, int64_t *stride) {
    if (!pol || !stride) { set_error("null argument"); return FP_ERR_INVALID; }
    *stride = grad_ep_stride(pol->dev.n, pol->dev.h, d);
    return FP_OK;
}

int fp_grad_rec_stride(const fp_policy *pol, int32_t d, int64_t *stride) {
    if (!pol || !stride) { set_error("null argument"); return FP_ERR_INVALID; }
    *stride = grad_rec_stride(d, (pol->dev.n + 31) / 32);
    return FP_OK;
}

int fp_rollout_workspace_size(const fp_problem *p, const fp_policy *pol, int32_t B,
                              int32_t flags, int32_t grad, int64_t *bytes) {
    if (!p || !pol || !bytes) { set_error("null argument"); return FP_ERR_INVALID; }
    *bytes = 0;
    if (B <= 0) return FP_OK;
    fp_rollout_args a{};
    a.B = B;
    a.flags = flags;
    a.grad_rows = grad ? (double *)1 : nullptr;  // only tested for non-null
    return dispatch(p, pol, a, bytes, 0);
}

int fp_rollout_batch(const fp_problem *p, const fp_policy *pol, const fp_rollout_args *args,
                     void *stream) {
    if (!p || !pol || !args || !args->assign || !args->status) {
        set_error("null argument");
        return FP_ERR_INVALID;
    }
    const fp_rollout_args &a = *args;
    if (a.B <= 0) return FP_OK;
    if (a.mode == FP_MODE_FORCED && !a.forced) { set_error("FORCED mode needs actions"); return FP_ERR_INVALID; }
    if (a.mode < 0 || a.mode > 3) { set_error("unknown mode"); return FP_ERR_INVALID; }
    if (a.grad_rows && !a.grad_ep) { set_error("grad_rows needs grad_ep"); return FP_ERR_INVALID; }
    if (a.simulate && !a.makespan) { set_error("simulate needs makespan"); return FP_ERR_INVALID; }
    return dispatch(p, pol, a, nullptr, (cudaStream_t)stream);
}

}  // extern "C"
