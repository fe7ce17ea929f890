// C-ABI: problem lifecycle, batched simulator entry, run_packed drop-in.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "fp_problem.cuh"
#include "fp_sim.cuh"

namespace fp {

static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }

#define FP_CUDA(call)                                                                     \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                \
            return FP_ERR_CUDA;                                                           \
        }                                                                                 \
    } while (0)

// Bump allocator over one device arena.
struct Arena {
    std::vector<std::pair<size_t, std::vector<uint8_t>>> parts;
    size_t size = 0;
    template <typename T>
    size_t put(const T *src, size_t count) {
        size = (size + 255) / 256 * 256;
        size_t off = size;
        std::vector<uint8_t> bytes(sizeof(T) * count);
        if (count) std::memcpy(bytes.data(), src, bytes.size());
        parts.emplace_back(off, std::move(bytes));
        size += sizeof(T) * count;
        return off;
    }
};

// One warp per simulation.  Compact path: the whole episode state in the
// warp's shared-memory slice, one wave.  Wide path (state beyond shared
// memory): a persistent grid, each resident warp owning one HBM workspace
// slice of L.gbytes and looping over episodes.
// LEAN: no trace / jitter / blocked-frontier outputs (the makespan-only path:
// batched scoring, brute force) -- smaller code, fewer instruction fetch stalls.
template <int RPL, int WARPS, bool WIDE, bool SM1, bool LEAN = false>
__global__ void __launch_bounds__(WARPS * 32)
sim_batch_kernel(DevProblem P, EpLayout L, const int32_t *__restrict__ assign, int B,
                 int strategy, const double *__restrict__ jit, long long jit_stride,
                 double *__restrict__ makespan, int32_t *__restrict__ status,
                 fp_event *__restrict__ trace, int trace_cap, int32_t *__restrict__ trace_len,
                 uint8_t *__restrict__ blocked, uint8_t *__restrict__ ws) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int warp = threadIdx.x >> 5;
    const int gw = blockIdx.x * WARPS + warp;
    uint8_t *sb = smem + (size_t)warp * L.bytes;
    uint8_t *nb = WIDE ? ws + (size_t)gw * L.gbytes : sb;
    for (int ep = gw; ep < B; ep += gridDim.x * WARPS) {
        uint8_t *as = nb + L.assign;
        const int32_t *row = assign + (size_t)ep * P.n;
        // device ids index per-device arrays and 1u << dev: an id outside
        // [0, d) fails the episode (FP_EP_BAD_ACTION) instead of running
        bool bad = false;
        for (int v = lane_id(); v < P.n; v += 32) {
            const int32_t a = row[v];
            bad |= a < 0 || a >= P.d;
            as[v] = (uint8_t)a;
        }
        if (__any_sync(FP_FULL_MASK, bad)) {
            if (lane_id() == 0) {
                makespan[ep] = 0.0;
                status[ep] = FP_EP_BAD_ACTION;
                if (trace_len) trace_len[ep] = 0;
            }
            continue;
        }
        __syncwarp();
        SimOut o = sim_episode<RPL, WIDE, SM1>(
            P, nb, sb, L, strategy, (!LEAN && jit) ? jit + (size_t)ep * jit_stride : nullptr,
            (!LEAN && trace) ? trace + (size_t)ep * trace_cap : nullptr, trace_cap,
            (!LEAN && blocked) ? blocked + (size_t)ep * P.n : nullptr);
        if (lane_id() == 0) {
            makespan[ep] = o.makespan;
            status[ep] = o.status;
            if (trace_len) trace_len[ep] = o.n_events;
        }
        __syncwarp();
    }
}

constexpr int kSimWarps = 4;

static bool sim_wide(const fp_problem *p, int flags) {
    const EpLayout L = make_layout(p->dev.n, p->dev.W, p->dev.R, p->dev.SM, false);
    return (flags & FP_FLAG_WIDE) || (int64_t)L.bytes * kSimWarps > 227 * 1024;
}

// Resident-episode count of a persistent launch: occupancy x SMs, capped by
// the batch (one workspace slice per resident warp).
int persistent_blocks(const void *kern, int threads, int64_t smem, int64_t blocks_needed) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, (size_t)smem) !=
            cudaSuccess || per_sm < 1)
        per_sm = 1;
    return (int)std::max<int64_t>(1, std::min<int64_t>(blocks_needed, (int64_t)sms * per_sm));
}

template <int RPL>
static int launch_sim_t(const fp_problem *p, const int32_t *assign, int B, int strategy,
                        const double *jit, long long jstride, double *mk, int32_t *st,
                        fp_event *trace, int cap, int32_t *tlen, uint8_t *blocked,
                        void *ws, int64_t ws_bytes, int flags, int64_t *ws_needed,
                        cudaStream_t stream) {
    constexpr int WARPS = kSimWarps;
    const bool wide = sim_wide(p, flags);
    const EpLayout L = make_layout(p->dev.n, p->dev.W, p->dev.R, p->dev.SM, false, 0, wide);
    const int64_t smem = (int64_t)L.bytes * WARPS;
    if (smem > 227 * 1024) {
        set_error("simulator scratch exceeds shared memory (too many devices / slots)");
        return FP_ERR_UNSUPPORTED;
    }
    const bool sm1 = p->dev.SM == 1;
    const bool lean = sm1 && !jit && !trace && !blocked;
    const void *kern =
        wide ? (sm1 ? (lean ? (const void *)sim_batch_kernel<RPL, WARPS, true, true, true>
                            : (const void *)sim_batch_kernel<RPL, WARPS, true, true>)
                    : (const void *)sim_batch_kernel<RPL, WARPS, true, false>)
             : (sm1 ? (lean ? (const void *)sim_batch_kernel<RPL, WARPS, false, true, true>
                            : (const void *)sim_batch_kernel<RPL, WARPS, false, true>)
                    : (const void *)sim_batch_kernel<RPL, WARPS, false, false>);
    FP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t need_blocks = (B + WARPS - 1) / WARPS;
    const int grid = wide ? persistent_blocks(kern, WARPS * 32, smem, need_blocks)
                          : (int)need_blocks;
    const int64_t need = wide ? (int64_t)grid * WARPS * L.gbytes : 0;
    if (ws_needed) { *ws_needed = need; return FP_OK; }
    if (need > 0 && (!ws || ws_bytes < need)) {
        set_error("workspace too small for the HBM-resident simulator (see fp_sim_workspace_size)");
        return FP_ERR_INVALID;
    }
    void *args[] = {(void *)&p->dev, (void *)&L, (void *)&assign, (void *)&B, (void *)&strategy,
                    (void *)&jit, (void *)&jstride, (void *)&mk, (void *)&st, (void *)&trace,
                    (void *)&cap, (void *)&tlen, (void *)&blocked, (void *)&ws};
    FP_CUDA(cudaLaunchKernel(kern, dim3(grid), dim3(WARPS * 32), args, (size_t)smem, stream));
    FP_CUDA(cudaGetLastError());
    return FP_OK;
}

static int launch_sim(const fp_problem *p, const int32_t *assign, int B, int strategy,
                      const double *jit, long long jstride, double *mk, int32_t *st,
                      fp_event *trace, int cap, int32_t *tlen, uint8_t *blocked, void *ws,
                      int64_t ws_bytes, int flags, int64_t *ws_needed, cudaStream_t stream) {
    const int R = p->dev.R;
#define FP_SIM_ARGS p, assign, B, strategy, jit, jstride, mk, st, trace, cap, tlen, blocked, ws, \
                    ws_bytes, flags, ws_needed, stream
    if (R <= 32) return launch_sim_t<1>(FP_SIM_ARGS);
    if (R <= 96) return launch_sim_t<3>(FP_SIM_ARGS);
    if (R <= 288) return launch_sim_t<9>(FP_SIM_ARGS);
    return launch_sim_t<33>(FP_SIM_ARGS);
#undef FP_SIM_ARGS
}

int sim_launch_compact(const fp_problem *p, const int32_t *assign, int B, int strategy,
                       double *makespan, int32_t *status, fp_event *trace, int trace_cap,
                       int32_t *trace_len, cudaStream_t stream) {
    return launch_sim(p, assign, B, strategy, nullptr, 0, makespan, status, trace, trace_cap,
                      trace_len, nullptr, nullptr, 0, 0, nullptr, stream);
}

}  // namespace fp

using namespace fp;

extern "C" {

const char *fp_last_error(void) { return g_err.c_str(); }
int fp_version(void) { return 1; }

int fp_problem_create(const fp_graph_desc *g, fp_problem **out) {
    if (!g || !out) { set_error("null argument"); return FP_ERR_INVALID; }
    const int n = g->n, d = g->d;
    if (n < 0 || d < 1 || d > kMaxDevices) {
        set_error("need n >= 0 and 1 <= d <= 32");
        return FP_ERR_UNSUPPORTED;
    }
    const int E = g->pred_indptr[n];
    if (g->succ_indptr[n] != E) { set_error("pred/succ edge counts differ"); return FP_ERR_INVALID; }
    for (int v = 0; v < E; ++v) {
        if (g->pred_indices[v] < 0 || g->pred_indices[v] >= n || g->succ_indices[v] < 0 ||
            g->succ_indices[v] >= n) {
            set_error("edge endpoint out of range");
            return FP_ERR_INVALID;
        }
    }
    const int R = d + d * d;
    std::vector<int> slots(R, 0);
    for (int a = 0; a < d; ++a) slots[a] = g->eslots[a];
    for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) slots[d + a * d + b] = a == b ? 0 : g->tslots[a * d + b];
    int SM = 1;
    for (int r = 0; r < R; ++r) {
        if (slots[r] < 0) { set_error("negative slot count"); return FP_ERR_INVALID; }
        SM = std::max(SM, slots[r]);
    }
    // a resource can never run more tasks at once than it has candidates
    SM = std::min(SM, std::max(n, 1));
    for (int r = 0; r < R; ++r) slots[r] = std::min(slots[r], SM);
    std::vector<double> tl(n, 0.0), bl(n, 0.0);
    if (g->tlev) std::copy(g->tlev, g->tlev + n, tl.begin());
    if (g->blev) std::copy(g->blev, g->blev + n, bl.begin());
    // strategy orders: fifo = id; depth_first = tlev desc; breadth_first = blev asc; ties by id
    std::vector<int> rpos(3 * n), rvert(3 * n), krank(3 * n, 0);
    for (int s = 0; s < 3; ++s) {
        std::vector<int> ord(n);
        std::iota(ord.begin(), ord.end(), 0);
        if (s == 1)
            std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return tl[x] > tl[y]; });
        if (s == 2)
            std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return bl[x] < bl[y]; });
        int k = 0;
        for (int i = 0; i < n; ++i) {
            const int v = ord[i];
            if (i > 0 && s != 0) {
                const double kv = s == 1 ? tl[v] : bl[v];
                const double ku = s == 1 ? tl[ord[i - 1]] : bl[ord[i - 1]];
                if (kv != ku) ++k;
            }
            rpos[s * n + v] = i;
            rvert[s * n + i] = v;
            krank[s * n + v] = k;
        }
    }
    int nonentry = 0;
    for (int v = 0; v < n; ++v) nonentry += !g->is_entry[v];
    // clean task durations, the reference's exact IEEE expressions
    // (_simcore.pyx:183,189; cluster.py:108-124): computed once per problem
    std::vector<double> edur((size_t)n * d), tdur((size_t)n * d * d, 0.0);
    for (int v = 0; v < n; ++v)
        for (int a = 0; a < d; ++a) {
            volatile double e = g->flops[v] / g->rates[a];
            edur[(size_t)v * d + a] = e;
            for (int b = 0; b < d; ++b) {
                if (a == b) continue;
                volatile double num = g->obytes[v] * g->comm_factor;
                volatile double t = num / g->bw[a * d + b];
                tdur[((size_t)v * d + a) * d + b] = t;
            }
        }

    Arena A;
    const int nn = std::max(n, 1);
    std::vector<uint8_t> entry(g->is_entry, g->is_entry + n);
    entry.resize(nn, 0);
    size_t o_pp = A.put(g->pred_indptr, n + 1), o_pi = A.put(g->pred_indices, E),
           o_sp = A.put(g->succ_indptr, n + 1), o_si = A.put(g->succ_indices, E),
           o_en = A.put(entry.data(), nn), o_fl = A.put(g->flops, n), o_ob = A.put(g->obytes, n),
           o_ra = A.put(g->rates, d), o_bw = A.put(g->bw, (size_t)d * d),
           o_tl = A.put(tl.data(), n), o_bl = A.put(bl.data(), n),
           o_sl = A.put(slots.data(), R), o_ed = A.put(edur.data(), edur.size()),
           o_td = A.put(tdur.data(), tdur.size()),
           o_rp = A.put(rpos.data(), 3 * n), o_rv = A.put(rvert.data(), 3 * n),
           o_kr = A.put(krank.data(), 3 * n);
    fp_problem *p = new fp_problem();
    FP_CUDA(cudaGetDevice(&p->device));
    if (cudaMalloc(&p->arena, std::max<size_t>(A.size, 256)) != cudaSuccess) {
        set_error("cudaMalloc failed for problem arena");
        delete p;
        return FP_ERR_CUDA;
    }
    uint8_t *base = (uint8_t *)p->arena;
    for (auto &part : A.parts)
        if (!part.second.empty())
            FP_CUDA(cudaMemcpy(base + part.first, part.second.data(), part.second.size(),
                               cudaMemcpyHostToDevice));
    DevProblem &D = p->dev;
    D.n = n; D.d = d; D.W = (n + 31) / 32; D.R = R; D.SM = SM; D.P = R * SM;
    D.n_nonentry = nonentry;
    D.comm_factor = g->comm_factor;
    D.pred_ptr = (const int *)(base + o_pp); D.pred_idx = (const int *)(base + o_pi);
    D.succ_ptr = (const int *)(base + o_sp); D.succ_idx = (const int *)(base + o_si);
    D.is_entry = base + o_en;
    D.flops = (const double *)(base + o_fl); D.obytes = (const double *)(base + o_ob);
    D.rates = (const double *)(base + o_ra); D.bw = (const double *)(base + o_bw);
    D.tlev = (const double *)(base + o_tl); D.blev = (const double *)(base + o_bl);
    D.slots = (const int *)(base + o_sl);
    D.edur = (const double *)(base + o_ed);
    D.tdur = (const double *)(base + o_td);
    D.rank_pos = (const int *)(base + o_rp); D.rank_vert = (const int *)(base + o_rv);
    D.krank = (const int *)(base + o_kr);
    p->sim_smem = make_layout(n, D.W, R, SM, false).bytes;
    *out = p;
    return FP_OK;
}

int fp_problem_destroy(fp_problem *p) {
    if (!p) return FP_OK;
    if (p->arena) cudaFree(p->arena);
    delete p;
    return FP_OK;
}

int fp_problem_sim_smem(const fp_problem *p, int64_t *bytes) {
    if (!p || !bytes) { set_error("null argument"); return FP_ERR_INVALID; }
    *bytes = p->sim_smem;
    return FP_OK;
}

int fp_sim_workspace_size(const fp_problem *p, int32_t B, int32_t flags, int64_t *bytes) {
    if (!p || !bytes) { set_error("null argument"); return FP_ERR_INVALID; }
    *bytes = 0;
    if (B <= 0) return FP_OK;
    return launch_sim(p, nullptr, B, 0, nullptr, 0, nullptr, nullptr, nullptr, 0, nullptr,
                      nullptr, nullptr, 0, flags, bytes, 0);
}

int fp_sim_batch(const fp_problem *p, const int32_t *assign, int32_t B, int32_t strategy,
                 const double *jitter, int64_t jitter_stride, double *makespan, int32_t *status,
                 fp_event *trace, int32_t trace_cap, int32_t *trace_len, uint8_t *blocked,
                 void *workspace, int64_t workspace_bytes, int32_t flags, void *stream) {
    if (!p || !assign || !makespan || !status) { set_error("null argument"); return FP_ERR_INVALID; }
    if (strategy < 0 || strategy > 2) { set_error("unknown strategy"); return FP_ERR_INVALID; }
    if (B <= 0) return FP_OK;
    return launch_sim(p, assign, B, strategy, jitter, jitter_stride, makespan, status, trace,
                      trace_cap, trace_len, blocked, workspace, workspace_bytes, flags, nullptr,
                      (cudaStream_t)stream);
}

// ---- fp_run_packed's per-thread problem cache --------------------------------
// The reference's FFI call (_simcore.pyx:39-45) receives the packed graph on
// every call and its callers loop over it (heuristics.py:127-128,
// cli.py:338-340).  Rebuilding the device problem and allocating per call
// would cost more than the simulation, so each host thread keeps the last few
// problems keyed by their exact input bytes (compared, not hashed), plus
// grow-only device / pinned buffers and its own stream: a repeated call does
// a compare, one H2D copy, the kernel and one D2H copy -- no allocation.
struct RunPackedSlot {
    std::vector<uint8_t> key;
    fp_problem *p = nullptr;
    uint8_t *dmem = nullptr, *hpin = nullptr;
    size_t dmem_bytes = 0, hpin_bytes = 0;
    void *ws = nullptr;
    int64_t ws_bytes = 0;
    cudaStream_t stream = nullptr;
    uint64_t used = 0;
    int reserve(size_t dbytes, size_t hbytes) {
        if (!stream) FP_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        if (dbytes > dmem_bytes) {
            if (dmem) cudaFree(dmem);
            dmem = nullptr;
            dmem_bytes = 0;
            FP_CUDA(cudaMalloc(&dmem, dbytes));
            dmem_bytes = dbytes;
        }
        if (hbytes > hpin_bytes) {
            if (hpin) cudaFreeHost(hpin);
            hpin = nullptr;
            hpin_bytes = 0;
            FP_CUDA(cudaMallocHost(&hpin, hbytes));
            hpin_bytes = hbytes;
        }
        return FP_OK;
    }
    int reserve_ws(int64_t bytes) {
        if (bytes > ws_bytes) {
            if (ws) cudaFree(ws);
            ws = nullptr;
            ws_bytes = 0;
            FP_CUDA(cudaMalloc(&ws, bytes));
            ws_bytes = bytes;
        }
        return FP_OK;
    }
    void release() {
        if (stream) cudaStreamSynchronize(stream);
        if (p) fp_problem_destroy(p);
        if (dmem) cudaFree(dmem);
        if (hpin) cudaFreeHost(hpin);
        if (ws) cudaFree(ws);
        if (stream) cudaStreamDestroy(stream);
        *this = RunPackedSlot{};
    }
};

constexpr int kRunPackedSlots = 4;
struct RunPackedCache {
    RunPackedSlot slot[kRunPackedSlots];
    uint64_t clock = 0;
    // no teardown at thread / process exit: the CUDA context may already be
    // gone then, and the driver reclaims everything with the process
};
static thread_local RunPackedCache tl_rp;

static void key_put(std::vector<uint8_t> &k, const void *src, size_t bytes) {
    const size_t o = k.size();
    k.resize(o + bytes);
    if (bytes) std::memcpy(k.data() + o, src, bytes);
}

static std::vector<uint8_t> run_packed_key(const fp_graph_desc &g) {
    const size_t n = (size_t)g.n, d = (size_t)g.d;
    const size_t E = g.n ? (size_t)g.pred_indptr[n] : 0, Es = g.n ? (size_t)g.succ_indptr[n] : 0;
    std::vector<uint8_t> k;
    k.reserve(64 + (n + 1) * 8 + (E + Es) * 4 + n * 33 + d * 16 + d * d * 12);
    key_put(k, &g.n, 4);
    key_put(k, &g.d, 4);
    key_put(k, &g.comm_factor, 8);
    key_put(k, g.pred_indptr, (n + 1) * 4);
    key_put(k, g.succ_indptr, (n + 1) * 4);
    key_put(k, g.pred_indices, E * 4);
    key_put(k, g.succ_indices, Es * 4);
    key_put(k, g.is_entry, n);
    key_put(k, g.flops, n * 8);
    key_put(k, g.obytes, n * 8);
    key_put(k, g.rates, d * 8);
    key_put(k, g.bw, d * d * 8);
    key_put(k, g.eslots, d * 4);
    key_put(k, g.tslots, d * d * 4);
    if (g.tlev) key_put(k, g.tlev, n * 8);
    if (g.blev) key_put(k, g.blev, n * 8);
    return k;
}

static int run_packed_slot(const fp_graph_desc &g, RunPackedSlot **out) {
    RunPackedCache &c = tl_rp;
    std::vector<uint8_t> key = run_packed_key(g);
    RunPackedSlot *victim = &c.slot[0];
    for (auto &s : c.slot) {
        if (s.p && s.key == key) {
            s.used = ++c.clock;
            *out = &s;
            return FP_OK;
        }
        if (!victim->p) continue;
        if (!s.p || s.used < victim->used) victim = &s;
    }
    if (victim->p) {  // evict the least recently used problem, keep its buffers
        if (victim->stream) cudaStreamSynchronize(victim->stream);
        fp_problem_destroy(victim->p);
        victim->p = nullptr;
    }
    fp_problem *p = nullptr;
    const int rc = fp_problem_create(&g, &p);
    if (rc) return rc;
    victim->p = p;
    victim->key = std::move(key);
    victim->used = ++c.clock;
    *out = victim;
    return FP_OK;
}

static void run_packed_cache_clear() {
    for (auto &s : tl_rp.slot) s.release();
}

// ---- host libm jitter (the reference recipe, _simcore.pyx:15-36) ----------
static uint64_t h_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static double h_jitter(uint64_t seed, int kind, int a, int b, int c, double sigma) {
    uint64_t h = h_mix64(seed ^ 0xD1B54A32D192ED03ULL);
    h = h_mix64(h ^ (uint64_t)(int64_t)(kind + 1));
    h = h_mix64(h ^ (uint64_t)(int64_t)(a + 1));
    h = h_mix64(h ^ (uint64_t)(int64_t)(b + 2));
    h = h_mix64(h ^ (uint64_t)(int64_t)(c + 2));
    const double s53 = std::ldexp(1.0, -53);
    volatile double u1 = ((double)(h >> 11) + 0.5) * s53;
    h = h_mix64(h);
    volatile double u2 = ((double)(h >> 11) + 0.5) * s53;
    volatile double two_pi_u2 = 2.0 * M_PI * u2;
    volatile double r = std::sqrt(-2.0 * std::log(u1));
    volatile double z = r * std::cos(two_pi_u2);
    return std::exp(sigma * z);
}

int fp_jitter_tables(int32_t n, int32_t d, double sigma, int64_t seed, double *out) {
    if (!out || n < 0 || d < 1) { set_error("bad jitter table arguments"); return FP_ERR_INVALID; }
    const size_t base = (size_t)n * d;
    for (size_t i = 0; i < base + base * d; ++i) out[i] = 1.0;
    if (sigma <= 0.0) return FP_OK;
    for (int v = 0; v < n; ++v)
        for (int a = 0; a < d; ++a) {
            out[(size_t)v * d + a] = h_jitter((uint64_t)seed, 0, v, a, 0, sigma);
            for (int b = 0; b < d; ++b)
                if (b != a)
                    out[base + ((size_t)v * d + a) * d + b] =
                        h_jitter((uint64_t)seed, 1, v, a, b, sigma);
        }
    return FP_OK;
}

int fp_run_packed(int32_t n, int32_t d, const int32_t *pred_indptr, const int32_t *pred_indices,
                  const int32_t *succ_indptr, const int32_t *succ_indices,
                  const uint8_t *is_entry, const double *flops, const double *obytes,
                  const int32_t *assign, const double *rates, const double *bw,
                  const int32_t *eslots, const int32_t *tslots, const double *tlev,
                  const double *blev, int32_t strategy, double comm_factor, double sigma,
                  int64_t seed, double *makespan, fp_event *events, int64_t events_cap,
                  int64_t *n_events, uint8_t *blocked) {
    if (n < 0 || d < 1) { set_error("need n >= 0 and d >= 1"); return FP_ERR_INVALID; }
    for (int v = 0; v < n; ++v)
        if (assign[v] < 0 || assign[v] >= d) { set_error("assignment names a device outside the cluster"); return FP_ERR_INVALID; }
    fp_graph_desc g{n, d, pred_indptr, pred_indices, succ_indptr, succ_indices, is_entry, flops,
                    obytes, rates, bw, eslots, tslots, tlev, blev, comm_factor};
    RunPackedSlot *slot = nullptr;
    int rc = run_packed_slot(g, &slot);
    if (rc) return rc;
    fp_problem *p = slot->p;
    const size_t jn = sigma > 0.0 ? (size_t)n * d * (d + 1) : 0;
    const int cap = (int)std::min<int64_t>(events_cap, 2LL * (n + (int64_t)n * d) + 2);
    // one device block: assign | jitter | makespan, status, len | blocked | trace
    const size_t off_j = (size_t)fp_align64((int64_t)n * 4, 256);
    const size_t off_m = off_j + (size_t)fp_align64((int64_t)jn * 8, 256);
    const size_t off_b = off_m + 256;
    const size_t off_t = off_b + (size_t)fp_align64(n, 256);
    const size_t total = off_t + (size_t)std::max(cap, 1) * sizeof(fp_event);
    // pinned staging: assign | jitter (upload), the 256-byte result block,
    // then (small traces) the whole event buffer, fetched in the same round
    // trip as the result block -- a second synchronising copy costs more
    // than moving up to 256 KB of unused capacity
    const size_t ev_bytes = events ? (size_t)std::max(cap, 1) * sizeof(fp_event) : 0;
    const bool ev_one_trip = ev_bytes <= (256u << 10);
    const size_t hup = off_m, htotal = hup + 256 + (ev_one_trip ? ev_bytes : 0);
    if ((rc = slot->reserve(total, htotal))) return rc;
    cudaStream_t st = slot->stream;
    uint8_t *h = slot->hpin, *dmem = slot->dmem;
    std::memcpy(h, assign, (size_t)n * 4);
    if (jn) fp_jitter_tables(n, d, sigma, seed, (double *)(h + off_j));
    FP_CUDA(cudaMemcpyAsync(dmem, h, hup, cudaMemcpyHostToDevice, st));
    int64_t ws_need = 0;
    rc = launch_sim(p, nullptr, 1, strategy, nullptr, 0, nullptr, nullptr, nullptr, 0, nullptr,
                    nullptr, nullptr, 0, 0, &ws_need, 0);
    if (rc) return rc;
    if ((rc = slot->reserve_ws(ws_need))) return rc;
    double *d_mk = (double *)(dmem + off_m);
    int32_t *d_st = (int32_t *)(dmem + off_m + 64), *d_len = (int32_t *)(dmem + off_m + 128);
    rc = launch_sim(p, (const int32_t *)dmem, 1, strategy,
                    jn ? (const double *)(dmem + off_j) : nullptr, 0, d_mk, d_st,
                    events ? (fp_event *)(dmem + off_t) : nullptr, cap, d_len, dmem + off_b,
                    slot->ws, slot->ws_bytes, 0, nullptr, st);
    if (rc) return rc;
    uint8_t *hres = h + hup;
    FP_CUDA(cudaMemcpyAsync(hres, dmem + off_m, 256, cudaMemcpyDeviceToHost, st));
    if (events && ev_one_trip)
        FP_CUDA(cudaMemcpyAsync(hres + 256, dmem + off_t, ev_bytes, cudaMemcpyDeviceToHost, st));
    {
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            set_error(std::string("simulator kernel failed: ") + cudaGetErrorString(e));
            return FP_ERR_CUDA;
        }
    }
    double mk;
    int32_t stt, len;
    std::memcpy(&mk, hres, 8);
    std::memcpy(&stt, hres + 64, 4);
    std::memcpy(&len, hres + 128, 4);
    if (events && len > 0) {
        const size_t got = (size_t)std::min(len, cap) * sizeof(fp_event);
        if (ev_one_trip)
            std::memcpy(events, hres + 256, got);
        else
            FP_CUDA(cudaMemcpy(events, dmem + off_t, got, cudaMemcpyDeviceToHost));
    }
    if (blocked && stt == FP_EP_DEADLOCK)
        FP_CUDA(cudaMemcpy(blocked, dmem + off_b, (size_t)n, cudaMemcpyDeviceToHost));
    *makespan = mk;
    if (n_events) *n_events = len;
    if (stt == FP_EP_DEADLOCK) { set_error("deadlock"); return FP_ERR_DEADLOCK; }
    if (stt == FP_EP_TRACE_OVERFLOW) { set_error("event buffer too small"); return FP_ERR_OVERFLOW; }
    return FP_OK;
}

int fp_run_packed_cache_clear(void) {
    run_packed_cache_clear();
    return FP_OK;
}

}  // extern "C"
