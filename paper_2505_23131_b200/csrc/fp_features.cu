// Static per-vertex features (reference features.py:51-96) as native host
// code, bit-identical to the Python mirror: col 0 flops, col 1 sum of the
// incoming comm costs (pred order), col 2 comm cost x out-degree, col 3
// t-level (longest path toward the exits: max over successors), col 4
// b-level (toward the entries: max over predecessors), with the first-maximum
// argmax neighbours as the t / b next forests.  The two sweeps are one
// topological order (Kahn) walked backward and forward -- O(n + E) and ~10 ms
// at 1M ops, where the Python sweep took seconds and dominated graph setup.
// (A per-graph precompute, not on the per-episode path: the GPU gains
// nothing over a single linear host pass here.)
#include <cmath>
#include <string>
#include <vector>

#include "fp_problem.cuh"

using namespace fp;

extern "C" {

int fp_static_features(int32_t n, const int32_t *pred_indptr, const int32_t *pred_indices,
                       const int32_t *succ_indptr, const int32_t *succ_indices,
                       const double *flops, const double *obytes, double comm_factor,
                       double *matrix, int32_t *b_next, int32_t *t_next) {
    if (n < 0 || !pred_indptr || !succ_indptr || !flops || !obytes || !matrix || !b_next || !t_next) {
        set_error("bad fp_static_features arguments");
        return FP_ERR_INVALID;
    }
    if (n == 0) return FP_OK;
    std::vector<double> cc(n);
    for (int v = 0; v < n; ++v) {
        volatile double c = obytes[v] * comm_factor;  // features.py:66, one rounding
        cc[v] = c;
    }
    // topological order (Kahn, smallest-id-first is not needed: any order
    // in which every predecessor precedes its successors gives the same DP)
    std::vector<int> indeg(n), order;
    order.reserve(n);
    for (int v = 0; v < n; ++v) {
        indeg[v] = pred_indptr[v + 1] - pred_indptr[v];
        if (!indeg[v]) order.push_back(v);
    }
    for (size_t i = 0; i < order.size(); ++i) {
        const int v = order[i];
        for (int j = succ_indptr[v]; j < succ_indptr[v + 1]; ++j)
            if (--indeg[succ_indices[j]] == 0) order.push_back(succ_indices[j]);
    }
    if ((int)order.size() != n) { set_error("graph is not a DAG"); return FP_ERR_INVALID; }
    auto M = [&](int v, int c) -> double & { return matrix[(size_t)v * 5 + c]; };
    for (int v = 0; v < n; ++v) {
        // sum(cc[u] for u in preds): CPython >= 3.12 sums floats with
        // Neumaier compensation (bltinmodule.c builtin_sum), so a plain
        // left-to-right sum would differ in the last bit
        volatile double in = 0.0, comp = 0.0;
        for (int j = pred_indptr[v]; j < pred_indptr[v + 1]; ++j) {
            const double x = cc[pred_indices[j]];
            volatile double t = in + x;
            if (std::fabs(in) >= std::fabs(x)) {
                volatile double d = in - t;
                comp = comp + (d + x);
            } else {
                volatile double d = x - t;
                comp = comp + (d + in);
            }
            in = t;
        }
        if (comp != 0.0 && std::isfinite(comp)) in = in + comp;
        M(v, 0) = flops[v];
        M(v, 1) = in;
        volatile double out = cc[v] * (double)(succ_indptr[v + 1] - succ_indptr[v]);
        M(v, 2) = out;
    }
    // _longest (features.py:38-48): first strict maximum in neighbour order
    for (int i = n - 1; i >= 0; --i) {  // t-level over successors, step cost cc[v]
        const int v = order[i];
        double best = 0.0;
        int arg = -1;
        for (int j = succ_indptr[v]; j < succ_indptr[v + 1]; ++j) {
            const int w = succ_indices[j];
            volatile double cand = cc[v] + M(w, 3);
            if (arg == -1 || cand > best) { best = cand; arg = w; }
        }
        volatile double t = flops[v] + best;
        M(v, 3) = t;
        t_next[v] = arg;
    }
    for (int i = 0; i < n; ++i) {  // b-level over predecessors, step cost cc[u]
        const int v = order[i];
        double best = 0.0;
        int arg = -1;
        for (int j = pred_indptr[v]; j < pred_indptr[v + 1]; ++j) {
            const int u = pred_indices[j];
            volatile double cand = cc[u] + M(u, 4);
            if (arg == -1 || cand > best) { best = cand; arg = u; }
        }
        volatile double b = flops[v] + best;
        M(v, 4) = b;
        b_next[v] = arg;
    }
    return FP_OK;
}

}  // extern "C"
