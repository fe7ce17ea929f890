/*
 * flowplace_b200 — C ABI of the B200-native DOPPLER rollout hot path.
 *
 * Plain C types only (pointers + sizes); device pointers are raw CUDA
 * allocations owned by the caller (torch tensors in the Python host), the
 * stream argument is a cudaStream_t passed as void*.  Every entry point
 * returns an FP_* status; fp_last_error() gives the message.  No call
 * allocates device memory except *_create (one-time, per graph / policy)
 * and the host-array drop-in fp_run_packed.
 *
 * Reference interfaces replaced (paths relative to the reference pkg/src):
 *   fp_run_packed      <- flowplace/_simcore.pyx:39-45   run_packed(...)  (Python->Cython FFI)
 *   fp_problem_create  <- flowplace/simulate.py:194-237 _pack(...)       (packed once per graph)
 *   fp_sim_batch       <- flowplace/simulate.py:251-266 exec_time(...)   (batched over assignments)
 *   fp_policy_*        <- flowplace/policy.py:149-402   gnn_encode / sel_forward / plc_forward /
 *                                                        PolicyContext.rollout
 *   fp_pg_*            <- flowplace/training.py:181-216 _rl_stage update (+ nn.py:184-277)
 */
#ifndef FLOWPLACE_B200_H
#define FLOWPLACE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* call status */
#define FP_OK 0
#define FP_ERR_INVALID 1
#define FP_ERR_CUDA 2
#define FP_ERR_UNSUPPORTED 3
#define FP_ERR_DEADLOCK 4
#define FP_ERR_OVERFLOW 5

/* simulator strategies (flowplace/simulate.py:37-38) */
#define FP_STRATEGY_FIFO 0
#define FP_STRATEGY_DEPTH_FIRST 1
#define FP_STRATEGY_BREADTH_FIRST 2

/* launch flags (fp_sim_batch flags, fp_rollout_args.flags) */
#define FP_FLAG_WIDE 1  /* force the HBM-resident (wide) episode path even when the
                           compact shared-memory path would fit (tests / benchmarks) */
#define FP_FLAG_PER_STEP 4   /* mp_mode = "per_step" (policy.py:353-371): re-encode both
                                GNNs with the placement columns before every decision
                                (B x n-row batched encode per step; forward only) */
#define FP_FLAG_TIE_RANDOM 2 /* FP_MODE_TEACHER: break equal-t-level selection ties
                                uniformly at random (Philox), as critical_path_assign's
                                trials do (heuristics.py:76-83, 114-117) */

/* per-episode status codes written by batched kernels */
#define FP_EP_OK 0
#define FP_EP_DEADLOCK 1        /* makespan slot holds the deadlock time   */
#define FP_EP_TRACE_OVERFLOW 2  /* trace_cap too small; makespan still valid */
#define FP_EP_BAD_ACTION 3      /* forced action outside candidates / devices */

/* One schedule event, the reference's (tkind, v, a, b, time, etype) record
 * (flowplace/_simpy.py:7-9): kind 0 exec (a = device, b = -1), 1 transfer
 * (a = src, b = dst); etype 0 beg, 1 end.  16 bytes. */
typedef struct fp_event {
    double time;
    int32_t v;
    int8_t kind;
    int8_t etype;
    int8_t a;
    int8_t b;
} fp_event;

/* The packed problem of flowplace/simulate.py:194-237, host pointers. */
typedef struct fp_graph_desc {
    int32_t n, d;
    const int32_t *pred_indptr, *pred_indices; /* [n+1], [E] sorted preds */
    const int32_t *succ_indptr, *succ_indices; /* [n+1], [E] sorted succs */
    const uint8_t *is_entry;                   /* [n] */
    const double *flops, *obytes;              /* [n] */
    const double *rates, *bw;                  /* [d], [d*d] */
    const int32_t *eslots, *tslots;            /* [d], [d*d] */
    const double *tlev, *blev;                 /* [n] or NULL (zeros) */
    double comm_factor;
} fp_graph_desc;

typedef struct fp_problem fp_problem;

const char *fp_last_error(void);
int fp_version(void);

/* Upload one graph + cluster to the current CUDA device (once per graph). */
int fp_problem_create(const fp_graph_desc *g, fp_problem **out);
int fp_problem_destroy(fp_problem *p);
/* Shared memory the simulator needs per in-flight episode (bytes). */
int fp_problem_sim_smem(const fp_problem *p, int64_t *bytes_per_episode);

/* Device workspace fp_sim_batch needs for B simulations (0 when every
 * episode's state fits the compact shared-memory core).  Graphs whose state
 * exceeds shared memory (n beyond ~2k at d = 8) run the wide path: a
 * persistent grid with each resident episode's n-sized state in a slice of
 * this caller-owned HBM workspace. */
int fp_sim_workspace_size(const fp_problem *p, int32_t B, int32_t flags, int64_t *bytes);

/* Work-conserving simulation of B assignments (device pointers).
 *   assign   [B][n] int32 device ids
 *   jitter   NULL, or per-task duration factors [n*d + n*d*d] per episode
 *            (exec (v,a) at v*d+a; transfer (v,a,b) at n*d+(v*d+a)*d+b),
 *            episode b reads jitter + b*jitter_stride (stride 0 = shared)
 *   makespan [B] out; status [B] out (FP_EP_*)
 *   trace    NULL, or [B][trace_cap] events out; trace_len [B] out
 *   blocked  NULL, or [B][n] uint8 out: blocked frontier on deadlock
 *   workspace / workspace_bytes: device scratch of fp_sim_workspace_size bytes
 *            (may be NULL / 0 when that size is 0)
 *   flags    FP_FLAG_* */
int fp_sim_batch(const fp_problem *p, const int32_t *assign, int32_t B, int32_t strategy,
                 const double *jitter, int64_t jitter_stride, double *makespan,
                 int32_t *status, fp_event *trace, int32_t trace_cap, int32_t *trace_len,
                 uint8_t *blocked, void *workspace, int64_t workspace_bytes, int32_t flags,
                 void *stream);

/* Drop-in for flowplace/_simcore.pyx:39-45 run_packed: host arrays in, host
 * events out (events[0..*n_events)).  Jitter factors are computed on the host
 * with the reference's splitmix64 + libm recipe (_simcore.pyx:15-36).
 * Returns FP_ERR_DEADLOCK with *makespan = deadlock time and blocked[v] set
 * for the blocked frontier (_simcore.pyx:204-207). */
int fp_run_packed(int32_t n, int32_t d, const int32_t *pred_indptr, const int32_t *pred_indices,
                  const int32_t *succ_indptr, const int32_t *succ_indices,
                  const uint8_t *is_entry, const double *flops, const double *obytes,
                  const int32_t *assign, const double *rates, const double *bw,
                  const int32_t *eslots, const int32_t *tslots, const double *tlev,
                  const double *blev, int32_t strategy, double comm_factor, double sigma,
                  int64_t seed, double *makespan, fp_event *events, int64_t events_cap,
                  int64_t *n_events, uint8_t *blocked);
/* fp_run_packed keeps, per host thread, the device problems of its last 4
 * distinct inputs (keyed by the exact graph / cluster bytes) with grow-only
 * device + pinned buffers and its own stream: repeated calls on one graph do
 * no allocation.  This frees the calling thread's cache. */
int fp_run_packed_cache_clear(void);

/* Static per-vertex features (flowplace/features.py:51-96) on the host in
 * native code, bit-identical to the reference's sweep: matrix [n][5] =
 * (flops, sum of incoming comm costs, comm cost x out-degree, t-level,
 * b-level), and the first-maximum argmax neighbours b_next / t_next (-1 at a
 * path's end).  Host pointers.  FP_ERR_INVALID if the graph has a cycle. */
int fp_static_features(int32_t n, const int32_t *pred_indptr, const int32_t *pred_indices,
                       const int32_t *succ_indptr, const int32_t *succ_indices,
                       const double *flops, const double *obytes, double comm_factor,
                       double *matrix, int32_t *b_next, int32_t *t_next);

/* Host libm jitter tables (the exact reference factors), layout as above. */
int fp_jitter_tables(int32_t n, int32_t d, double sigma, int64_t seed, double *out);

/* ------------------------------------------------------------------------
 * Policy: GNN encoder + SEL/PLC heads (flowplace/policy.py:40-251).
 * Parameters live in ONE flat float64 device vector; param_offsets maps each
 * role to its offset (-1 = absent).  Role index for GNN tensors:
 *   ((enc * 8 + k) * 4 + r), enc 0 = "sel" / shared "enc", 1 = "plc",
 *   r: 0 psi.w, 1 psi.b, 2 phi.w, 3 phi.b;
 * then FP_ROLE_SEL_Z_W .. FP_ROLE_PLC_Y_B below.  Tensors are row-major with
 * the reference's shapes (policy.py:74-98).
 * ------------------------------------------------------------------------ */
#define FP_ROLE_SEL_Z_W 64
#define FP_ROLE_SEL_Z_B 65
#define FP_ROLE_SEL_H1_W 66
#define FP_ROLE_SEL_H1_B 67
#define FP_ROLE_SEL_H2_W 68
#define FP_ROLE_SEL_H2_B 69
#define FP_ROLE_PLC_Z_W 70
#define FP_ROLE_PLC_Z_B 71
#define FP_ROLE_PLC_H1_W 72
#define FP_ROLE_PLC_H1_B 73
#define FP_ROLE_PLC_H2_W 74
#define FP_ROLE_PLC_H2_B 75
#define FP_ROLE_PLC_Y_W 76
#define FP_ROLE_PLC_Y_B 77
#define FP_PARAM_ROLES 78

/* rollout decision modes */
#define FP_MODE_SAMPLE 0  /* epsilon-mixture draws from Philox4x32-10 */
#define FP_MODE_GREEDY 1  /* argmax of the softmax (policy.py:308-309) */
#define FP_MODE_FORCED 2  /* replay given (vertex, device) per step */
#define FP_MODE_TEACHER 3 /* CriticalPathRule actions (heuristics.py:76-91) */

/* device tables readable through fp_policy_table (parity / debugging) */
#define FP_TABLE_H_SEL 0
#define FP_TABLE_H_PLC 1
#define FP_TABLE_SEL_LOGIT 2
#define FP_TABLE_PLC_A 3
#define FP_TABLE_PLC_G 4
#define FP_TABLE_PLC_M 5
#define FP_TABLE_PLC_C 6

typedef struct fp_policy_desc {
    int32_t hidden, k_rounds, shared_encoder;
    double leaky_slope;
    const double *x_static;               /* [n*5] standardized (policy.py:123) */
    const int32_t *adj_ptr, *adj_src;     /* [n+1], [M]: messages INTO each vertex */
    const double *adj_edge;               /* [M] standardized edge cost (policy.py:124-143) */
    const int32_t *bpath_ptr, *bpath_idx; /* [n+1], SEL b-paths (features.py:88-95) */
    const int32_t *tpath_ptr, *tpath_idx; /* [n+1], SEL t-paths */
    const int64_t *param_offsets;         /* [FP_PARAM_ROLES] */
    int64_t n_params;
    /* Forest form of the same paths: path(v) = (v, next[v], next[next[v]], ...),
     * -1 ends a path.  Used when bpath_ptr == NULL (large graphs, where the
     * explicit lists grow like n * depth); path sums are then computed on the
     * GPU by pointer jumping.  Forward only: REINFORCE backward needs the
     * explicit lists. */
    const int32_t *bnext, *tnext;         /* [n] */
} fp_policy_desc;

typedef struct fp_policy fp_policy;

typedef struct fp_rollout_args {
    int32_t B;               /* episodes in the batch */
    int32_t mode;            /* FP_MODE_* */
    double epsilon;          /* exploration mixture weight */
    uint64_t seed;           /* Philox key */
    uint32_t episode_base;   /* Philox counter of episode 0 (rank offset) */
    int32_t strategy;        /* simulator strategy for the reward */
    int32_t simulate;        /* 1: score every episode with the WC simulator */
    const int32_t *forced;   /* [B][n][2] (vertex, device) per step, FORCED */
    int32_t *assign;         /* [B][n] out: device of each vertex */
    int32_t *step_vd;        /* [B][n][2] out or NULL */
    double *step_lp;         /* [B][n][2] out or NULL: (sel, plc) log-prob */
    double *step_ent;        /* [B][n][2] out or NULL: (sel, plc) entropy */
    int32_t *step_argmax;    /* [B][n][2] out or NULL: greedy (vertex, device) */
    int32_t *step_ncand;     /* [B][n] out or NULL: candidate-set size */
    double *makespan;        /* [B] out (simulate = 1) */
    int32_t *status;         /* [B] out: FP_EP_* */
    double *grad_rows;       /* [B][n][fp_grad_rec_stride] out or NULL: REINFORCE
                                decision records (consumed by fp_pg_reduce) */
    double *grad_ep;         /* [B][fp_grad_ep_stride] out (with grad_rows) */
    fp_event *trace;         /* optional simulator trace [B][trace_cap] */
    int32_t trace_cap;
    int32_t *trace_len;
    int32_t flags;           /* FP_FLAG_* */
    void *workspace;         /* device scratch, fp_rollout_workspace_size bytes */
    int64_t workspace_bytes;
} fp_rollout_args;

int fp_policy_create(const fp_problem *p, const fp_policy_desc *desc, fp_policy **out);
int fp_policy_destroy(fp_policy *pol);
/* Encoder implementation: 0 (default) = aggregation kernels + fp64 tensor-core
 * (DMMA) node-MLP kernels when hidden is a multiple of 8 (<= 64); 1 = one
 * fused CUDA-core kernel per round with the reference's per-column FMA order.
 * Both agree with the reference to rounding (1e-11).  2 = bf16 node MLPs on
 * the 5th-gen tensor cores (tcgen05, TMA-fed, split bf16 operands, fp32
 * accumulation in TMEM; ~1e-5 relative, the north star's bf16 MLP mode,
 * forward only, hidden 16 / 32). */
enum { FP_ENCODER_DMMA = 0, FP_ENCODER_FUSED = 1, FP_ENCODER_TC = 2 };
int fp_policy_set_encoder(fp_policy *pol, int32_t mode);
/* GNN encode + head tables for one parameter snapshot (params: device flat). */
int fp_policy_prepare(fp_policy *pol, const double *params, void *stream);
int fp_policy_table(const fp_policy *pol, int32_t which, const double **ptr, int64_t *count);
/* Device workspace fp_rollout_batch needs for B episodes (0 on the compact
 * shared-memory path; graphs beyond it run the wide path, whose per-episode
 * n-sized state lives in this caller-owned HBM scratch).  grad = 1 for a
 * REINFORCE rollout (compact path only; its per-decision records go to
 * grad_rows, not the workspace). */
int fp_rollout_workspace_size(const fp_problem *p, const fp_policy *pol, int32_t B,
                              int32_t flags, int32_t grad, int64_t *bytes);
/* Batched SEL/PLC episodes (+ fused WC simulation) — one warp per episode. */
int fp_rollout_batch(const fp_problem *p, const fp_policy *pol, const fp_rollout_args *args,
                     void *stream);
int fp_grad_ep_stride(const fp_policy *pol, int32_t d, int64_t *stride);
/* doubles per (episode, step) REINFORCE decision record in grad_rows:
 * normalised device features [5d], PLC logits [d], (vertex, device) int2 */
int fp_grad_rec_stride(const fp_policy *pol, int32_t d, int64_t *stride);

/* ------------------------------------------------------------------------
 * Stage-II update (flowplace/training.py:181-216, nn.py:184-277).
 * fp_pg_reduce replays the rollout's REINFORCE decision records with
 * per-episode coefficients alpha[e] (= -advantage_e / B_global for Stage II,
 * -1/B for imitation) and beta (= -entropy_weight / B_global) folded in, and
 * reduces the episodes deterministically (fixed order, no atomics);
 * fp_policy_backward turns the reduced tables into the flat parameter
 * gradient (same layout as the params); fp_sgd_step applies
 * params -= lr * grad (nn.py:271-277).
 * ------------------------------------------------------------------------ */
int fp_pg_reduce(fp_policy *pol, const double *grad_rows, const double *grad_ep,
                 const int32_t *assign, const double *alpha, double beta, int32_t B,
                 void *stream);
int fp_policy_backward(fp_policy *pol, double *grad, void *stream);
/* per_step message passing (reference mp_mode="per_step"): the whole flat
 * gradient of sum_e alpha[e] * sum lp_e + beta * sum ent_e for a per_step
 * REINFORCE rollout (FP_FLAG_PER_STEP with grad_rows), backpropagated
 * through the encode of every step, episodes and steps in order -- replaces
 * fp_pg_reduce + fp_policy_backward for per_step rollouts. */
int fp_pg_reduce_per_step(fp_policy *pol, const double *grad_rows, const double *grad_ep,
                          const double *alpha, double beta, int32_t B, double *grad,
                          void *stream);
int fp_sgd_step(double *params, const double *grad, int64_t count, double lr, void *stream);
/* as fp_sgd_step, skipped on the device when *skip != 0 (skip: device int32,
 * e.g. a sticky "some rollout of this batch failed" flag), so a trainer can
 * keep the step free of host synchronisation and raise afterwards */
int fp_sgd_step_masked(double *params, const double *grad, int64_t count, double lr,
                       const int32_t *skip, void *stream);

/* Measurement hook (bench.py): while enabled, every GNN aggregation launch
 * is bracketed by an event pair on its own stream; fp_agg_timer_read syncs
 * those events, returns the summed kernel time and launch count since the
 * last read / enable, and resets.  No effect on results. */
int fp_agg_timer_enable(int32_t on);
int fp_agg_timer_read(double *total_ms, int64_t *launches);

/* Tensor-core (tcgen05 + TMA) path self test: out[M][N] (fp32) = X . W with
 * X [M][64] given as bf16 hi / lo planes (device, row pitch 128 bytes) and W
 * [64][N] fp64 (device), N in {32, 64}; the three split products accumulate
 * in TMEM.  Test hook for the bf16 encoder's GEMM machinery. */
int fp_tc_gemm_selftest(const void *x_hi, const void *x_lo, const double *W, int32_t N,
                        float *out, int32_t M, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FLOWPLACE_B200_H */
