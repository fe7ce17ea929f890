// Device-side policy state: parameter roles in the flat float64 vector, the
// per-graph encoding constants, and the per-snapshot tables the rollout
// kernel consumes:
//   s[v]          SEL logit of vertex v (static per snapshot in per_episode mode)
//   A[v], G[v]    PLC pre-activation tables: pre(v, d) = A[v] + S_d + xn_d @ M + c,
//                 S_d = sum of G[u] over vertices already placed on d
//   M (5 x h), c  device-feature and bias terms folded through head1
#pragma once

#include <cstdint>

#include "fp_problem.cuh"

namespace fp {

constexpr int kMaxRounds = 8;
constexpr int kMaxHidden = 64;

// Parameter roles.  GNN role index: ((enc * kMaxRounds + k) * 4 + r), enc 0 =
// "sel" (or the shared "enc"), 1 = "plc"; r: 0 psi.w, 1 psi.b, 2 phi.w, 3 phi.b.
enum : int {
    PR_GNN_BASE = 0,
    PR_SEL_Z_W = 2 * kMaxRounds * 4,
    PR_SEL_Z_B,
    PR_SEL_H1_W,
    PR_SEL_H1_B,
    PR_SEL_H2_W,
    PR_SEL_H2_B,
    PR_PLC_Z_W,
    PR_PLC_Z_B,
    PR_PLC_H1_W,
    PR_PLC_H1_B,
    PR_PLC_H2_W,
    PR_PLC_H2_B,
    PR_PLC_Y_W,
    PR_PLC_Y_B,
    PR_COUNT
};

__host__ __device__ inline int gnn_role(int enc, int k, int r) {
    return PR_GNN_BASE + (enc * kMaxRounds + k) * 4 + r;
}

struct DevPolicy {
    int n, h, K, n_enc;  // n_enc = 1 (shared) or 2
    // encoder row batch: rows = batch * n (batch > 1 only for per_step
    // message passing, where row b*n + v is vertex v of episode b and
    // ps_dev[b*n + v] its device so far, -1 = unplaced)
    int rows, batch, D;
    const int *ps_dev;
    double slope;
    const double *params;          // flat float64 (set by prepare)
    double *grad;                  // flat float64 gradient (backward)
    int64_t off[PR_COUNT];
    // per-graph encoding constants
    const double *x;               // [n][5] standardized static features
    const int *adj_ptr, *adj_nbr;  // messages INTO v: source vertices, message order
    const double *adj_e;           // standardized edge cost per message
    const int *bp_ptr, *bp_idx, *tp_ptr, *tp_idx;     // SEL b/t paths
    int n_bpath, n_tpath;                             // their total lengths
    int n_msgs;                                       // adj_ptr[n] (host copy)
    int64_t n_params;                                 // doubles in the flat params
    const int *ibp_ptr, *ibp_idx, *itp_ptr, *itp_idx; // inverse paths (u -> v with u in path(v))
    // forest form (large graphs): next pointers + pointer-jumping buffers
    int forest, jump_rounds;
    const int *nxt[2];             // b_next, t_next
    double *PS[2][2];              // [b/t][ping-pong] partial path sums, [n][h]
    int *PJ[2][2];                 // [b/t][ping-pong] jump pointers
    // workspace (per snapshot)
    double *H[2][kMaxRounds + 1];  // layer inputs/outputs; H[e][0] is [n][7]
    double *Pm[2][kMaxRounds];     // H[e][k] @ psi.w rows [0, d)
    double *Qm[2][kMaxRounds];     // H[e][k] @ psi.w rows [d, 2d)
    double *U[2][kMaxRounds];      // phi pre-activations
    double *AG[2][kMaxRounds];     // aggregated messages (backward)
    double *Zs, *emb, *hidpre, *s; // SEL tables
    double *Zp, *A, *G, *M, *c;    // PLC tables
    // backward workspace
    double *dH[2], *dHn[2], *dU, *Dsrc, *Ddst, *dagg, *De;
    double *dhid, *demb, *dZ;      // SEL head / z backward rows
    double *ds, *dA, *dG, *dsmall; // reduced gradient tables
    // bf16 tensor-core encoder (fp_tc_node.cu): round inputs X_k = [H_k | agg_k]
    // as split bf16 planes (hi, lo), [rows][64], H_k at columns [0, dk),
    // agg_k at [32, 32 + h); zero elsewhere
    int tc;
    uint16_t *Xh[2][kMaxRounds], *Xl[2][kMaxRounds];

    __device__ __forceinline__ const double *W(int role) const { return params + off[role]; }
};

// GNN encode of every row of P (fp_encode.cu): aggregation + DMMA node MLPs
// (+ forest path sums and the SEL head when sel_head).  0 or FP_ERR_*.
int gnn_encode_rows(DevPolicy &P, cudaStream_t st, bool bwd, bool sel_head);
int agg_timer_enable(int on);
int agg_timer_read(double *total_ms, int64_t *launches);

// bf16 tensor-core node MLPs of round k (fp_tc_node.cu); needs P.tc planes.
int tc_node_launch(const DevPolicy &P, int k, bool last, cudaStream_t st);
// bytes of the X planes of a policy / per_step batch with `rows` rows
inline int64_t tc_plane_bytes(int64_t rows, int K, int n_enc) {
    return rows * 64 * 2 * 2 * (int64_t)K * n_enc;
}
void tc_set_planes(DevPolicy &P, void *base, int64_t rows);

}  // namespace fp

struct fp_train_state;
void fp_train_state_free(fp_train_state *);

struct fp_policy {
    fp::DevPolicy dev;
    void *arena = nullptr;
    const fp_problem *problem = nullptr;
    fp_train_state *train = nullptr;  // backward job lists (fp_train.cu)
    int fused_encoder = 0;            // 1: single fused per-vertex kernel (reference order)
    void *tc_planes = nullptr;        // bf16 encoder planes (per-snapshot rows), lazily
    int64_t n_params = 0;
};
