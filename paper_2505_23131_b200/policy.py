"""Dual SEL/PLC policy — drop-in for reference ``flowplace/policy.py``.

Same names and semantics as the reference (``PolicyConfig``,
``init_policy_params``, ``GraphEncoding``, ``PolicyContext.rollout`` ->
``(Assignment, EpisodeTrace)``, ``TeacherActionError``), executed by the CUDA
library: ``fp_policy_prepare`` encodes the graph once per parameter snapshot
(GNN + head tables), ``fp_rollout_batch`` runs B episodes — one warp each —
and scores them with the fused WC simulator.

Differences from the reference, by design:
  * sampling draws come from Philox4x32-10 keyed by (seed, episode, step,
    head) instead of numpy PCG64; distributions and the
    recorded mixture log-probs are the reference's;
  * ``EpisodeTrace.logprob_tensors`` / ``entropy_tensors`` stay empty: the
    REINFORCE gradient is produced natively (``training.py``);
  * teachers: ``CriticalPathRule`` runs natively; ``ForcedActions`` replays
    recorded actions; any other object with the reference's select / place
    interface is stepped on the host (``teacher_actions``) and its actions
    replayed in FORCED mode (no per-step Python callbacks inside the kernel).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .cluster import ClusterSpec
from .features import StaticGraphFeatures, static_features
from .graph import DataflowGraph
from .heuristics import Assignment, CriticalPathRule, ForcedActions
from .params import (N_DEVICE_FEATURES, N_DYNAMIC_COLS, N_STATIC_FEATURES, FlatLayout, Param,
                     Params, as_array, encoder_names, init_policy_params)
from .simulate import _STRATEGY_CODE, DeadlockError, SimProblem

MP_MODES = ("per_episode", "per_step")

__all__ = ["PolicyConfig", "init_policy_params", "GraphEncoding", "PolicyContext", "TraceStep",
           "EpisodeTrace", "TeacherActionError", "RolloutBatch", "assign_rollout",
           "N_STATIC_FEATURES", "N_DEVICE_FEATURES", "N_DYNAMIC_COLS"]


@dataclass
class PolicyConfig:
    hidden: int = 32
    k_rounds: int = 2
    mp_mode: str = "per_episode"
    leaky_slope: float = 0.01
    shared_encoder: bool = False

    def __post_init__(self):
        if self.mp_mode not in MP_MODES:
            raise ValueError(f"mp_mode must be one of {MP_MODES}, got {self.mp_mode!r}")
        if self.k_rounds < 1:
            raise ValueError("k_rounds must be >= 1")

    def to_dict(self) -> dict:
        return {"hidden": self.hidden, "k_rounds": self.k_rounds, "mp_mode": self.mp_mode,
                "leaky_slope": self.leaky_slope, "shared_encoder": self.shared_encoder}

    @classmethod
    def from_dict(cls, doc: dict) -> "PolicyConfig":
        return cls(**{k: doc[k] for k in ("hidden", "k_rounds", "mp_mode", "leaky_slope",
                                          "shared_encoder") if k in doc})


def _standardize(mat: np.ndarray):
    """Column standardization with the 1e-12 guard (reference policy.py:101-105)."""
    mean = mat.mean(axis=0) if mat.size else np.zeros(mat.shape[1])
    std = mat.std(axis=0) if mat.size else np.ones(mat.shape[1])
    std = np.where(std < 1e-12, 1.0, std)
    return (mat - mean) / std, mean, std


@dataclass
class GraphEncoding:
    """Per-graph constants (reference policy.py:108-146): standardized static
    features and the two-way message lists with standardized edge costs."""

    graph: DataflowGraph
    features: StaticGraphFeatures
    x_static: np.ndarray
    msg_src: np.ndarray
    msg_dst: np.ndarray
    msg_edge: np.ndarray
    norm_stats: dict

    @classmethod
    def build(cls, graph: DataflowGraph, features: StaticGraphFeatures) -> "GraphEncoding":
        x, mean, std = _standardize(features.matrix)
        m = len(graph.edges)
        src = np.empty(2 * m, dtype=np.intp)
        dst = np.empty(2 * m, dtype=np.intp)
        cost = np.empty(2 * m, dtype=np.float64)
        for i, (u, v) in enumerate(graph.edges):
            c = graph.vertices[u].output_bytes * features.comm_factor
            src[2 * i], dst[2 * i], cost[2 * i] = u, v, c
            src[2 * i + 1], dst[2 * i + 1], cost[2 * i + 1] = v, u, c
        cost = cost.reshape(-1, 1)
        if cost.size:
            e_mean = float(cost.mean())
            e_std = float(cost.std()) or 1.0
        else:
            e_mean, e_std = 0.0, 1.0
        e_std = e_std if e_std >= 1e-12 else 1.0
        return cls(graph, features, x, src, dst, (cost - e_mean) / e_std,
                   {"mean": mean.tolist(), "std": std.tolist(), "edge_mean": e_mean,
                    "edge_std": e_std})

    def csr_into(self):
        """Messages grouped by destination (message order kept): the gather
        layout of the CUDA aggregation kernel."""
        n = len(self.graph)
        order = np.argsort(self.msg_dst, kind="stable")
        ptr = np.zeros(n + 1, dtype=np.int32)
        np.add.at(ptr, self.msg_dst + 1, 1)
        ptr = np.cumsum(ptr).astype(np.int32)
        return (ptr, self.msg_src[order].astype(np.int32),
                np.ascontiguousarray(self.msg_edge.reshape(-1)[order]))

    def paths_csr(self):
        def pack(paths):
            ptr = np.zeros(len(paths) + 1, dtype=np.int32)
            ptr[1:] = np.cumsum([len(p) for p in paths])
            return ptr, np.asarray([u for p in paths for u in p], dtype=np.int32)
        return pack(self.features.b_paths) + pack(self.features.t_paths)


@dataclass
class TraceStep:
    step: int
    candidates: tuple[int, ...]
    vertex: int
    sel_logprob: float
    device: int
    plc_logprob: float
    sel_entropy: float
    plc_entropy: float
    sel_argmax: int = -1
    plc_argmax: int = -1


@dataclass
class EpisodeTrace:
    steps: list[TraceStep] = field(default_factory=list)
    makespan_ms: float | None = None
    encode_invocations: int = 0
    logprob_tensors: list = field(default_factory=list, repr=False)
    entropy_tensors: list = field(default_factory=list, repr=False)


class TeacherActionError(RuntimeError):
    pass


@dataclass
class RolloutBatch:
    """Device tensors of one batched rollout (B episodes)."""

    assign: object                 # [B, n] int32
    status: object                 # [B] int32
    makespan: object | None        # [B] f64
    step_vd: object | None = None  # [B, n, 2] int32 (vertex, device)
    step_lp: object | None = None  # [B, n, 2] f64
    step_ent: object | None = None
    step_argmax: object | None = None
    step_ncand: object | None = None
    grad_rows: object | None = None
    grad_ep: object | None = None
    trace: object | None = None
    trace_len: object | None = None


def is_native_teacher(teacher) -> bool:
    """CriticalPathRule runs inside the rollout kernel (FP_MODE_TEACHER)."""
    return isinstance(teacher, CriticalPathRule) or type(teacher).__name__ == "CriticalPathRule"


def teacher_actions(graph: DataflowGraph, cluster, teacher, episodes: int = 1) -> np.ndarray:
    """Actions of an arbitrary (duck-typed) teacher, stepped on the host the
    way the reference's rollout calls it (policy.py:353-389): at every step
    ``teacher.select(candidates)`` on the ascending candidate list, then
    ``teacher.place(v, timeline)`` on the committed placements so far
    (heuristics.PlacementTimeline, timeline.py:19-58).  Returns [episodes, n,
    2] (vertex, device) for the GPU rollout's FORCED mode, which recomputes the
    log-probs / REINFORCE terms of these actions; one host pass per episode,
    so stochastic teachers get independent episodes.  A vertex outside the
    candidates raises TeacherActionError (reference policy.py:359-363); an
    out-of-range device is reported by the kernel (FP_EP_BAD_ACTION)."""
    from .heuristics import PlacementTimeline

    n = len(graph)
    preds = [len(graph.preds(v)) for v in range(n)]
    out = np.empty((episodes, n, 2), dtype=np.int32)
    for e in range(episodes):
        left = list(preds)
        cands = sorted(v for v in range(n) if left[v] == 0)
        tl = PlacementTimeline(graph, cluster)
        for t in range(n):
            if not cands:
                raise TeacherActionError("no candidate left (cyclic graph)")
            v = int(teacher.select(list(cands)))
            if v not in cands:
                raise TeacherActionError(
                    f"teacher selected vertex {v} outside candidates {cands}")
            d = int(teacher.place(v, tl))
            if not 0 <= d < cluster.device_count:
                raise TeacherActionError(f"teacher placed vertex {v} on device {d}")
            tl.commit(v, d)
            out[e, t] = (v, d)
            cands.remove(v)
            for w in graph.succs(v):
                left[w] -= 1
                if left[w] == 0:
                    cands.append(w)
            cands.sort()
    return out


def _candidate_sets(graph: DataflowGraph, order) -> list[tuple[int, ...]]:
    """The sorted candidate set before each step of a placement order
    (policy.py:338-389) — host reconstruction for TraceStep.candidates."""
    left = [len(graph.preds(v)) for v in range(len(graph))]
    cands = sorted(graph.entry_vertices())
    out = []
    for v in order:
        out.append(tuple(cands))
        cands.remove(v)
        for w in graph.succs(v):
            left[w] -= 1
            if left[w] == 0:
                cands.append(w)
        cands.sort()
    return out


# Graphs above this size hand the SEL paths to the GPU as next-pointer
# forests (path sums by pointer jumping) instead of explicit lists, whose
# total length grows like n * depth.  Matches the compact rollout's limit:
# REINFORCE rows (and so the backward, which needs the lists) stop there.
FOREST_MIN_N = 1024


class PolicyContext:
    """Per-graph rollout machinery on the GPU (reference policy.py:281-402)."""

    def __init__(self, graph: DataflowGraph, cluster: ClusterSpec, config: PolicyConfig,
                 features: StaticGraphFeatures | None = None, forest: bool | None = None):
        if config.mp_mode not in ("per_episode", "per_step"):
            raise ValueError(f"unknown mp_mode {config.mp_mode!r}")
        # per_step (policy.py:353-371): both encoders re-run before every
        # decision with the placement columns -- a B x n-row batched encode per
        # step on the GPU (forward only)
        self.per_step = config.mp_mode == "per_step"
        self.graph = graph
        self.cluster = cluster
        self.config = config
        self.features = features if features is not None else static_features(
            graph, cluster.comm_factor)
        self.enc = GraphEncoding.build(graph, self.features)
        self.encode_count = 0
        self.sim = SimProblem(graph, cluster, self.features)
        self.layout = FlatLayout.for_config(config)
        self.forest = len(graph) > FOREST_MIN_N if forest is None else bool(forest)
        self._make_native()
        self._flat = None          # device flat params of the current snapshot
        self._prepared_key = None

    # ------------------------------------------------------------------ native
    def _make_native(self):
        offs = np.full(N.PARAM_ROLES, -1, dtype=np.int64)
        encs = ["enc"] if self.config.shared_encoder else ["sel", "plc"]
        for e, name in enumerate(encs):
            for k in range(self.config.k_rounds):
                for r, t in enumerate(("psi.w", "psi.b", "phi.w", "phi.b")):
                    offs[N.gnn_role(e, k, r)] = self.layout.offset(f"{name}.gnn{k}.{t}")
        for name, role in N.ROLE_BY_HEAD.items():
            offs[role] = self.layout.offset(name)
        ptr, src, edge = self.enc.csr_into()
        # explicit path lists for graphs the compact kernels (and the REINFORCE
        # backward) handle; the next-pointer forests beyond that
        bnext = np.ascontiguousarray(self.features.b_next, dtype=np.int32)
        tnext = np.ascontiguousarray(self.features.t_next, dtype=np.int32)
        bp = bi = tp = ti = None
        if not self.forest:
            bp, bi, tp, ti = self.enc.paths_csr()
        x = np.ascontiguousarray(self.enc.x_static, dtype=np.float64)
        self._host_keep = (offs, ptr, src, edge, bp, bi, tp, ti, x, bnext, tnext)
        desc = N.FpPolicyDesc(self.config.hidden, self.config.k_rounds,
                              int(self.config.shared_encoder), float(self.config.leaky_slope),
                              *[N.ptr(a).value for a in (x, ptr, src, edge, bp, bi, tp, ti, offs)],
                              self.layout.size, N.ptr(bnext).value, N.ptr(tnext).value)
        h = ctypes.c_void_p()
        N.check(N.lib().fp_policy_create(self.sim.handle, ctypes.byref(desc), ctypes.byref(h)))
        self.handle = h
        self._lib = N.lib()

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self._lib.fp_policy_destroy(h)
            self.handle = None

    def encode_launches(self) -> int:
        """Kernel launches of one prepare: a single fused launch for graphs of
        <= 64 ops; else proj0 + K x (aggregation, node MLPs) + path sums (or
        the pointer-jumping rounds) + SEL head (fp_encode.cu)."""
        K = self.config.k_rounds
        if self.config.hidden in (8, 16, 32, 64):
            if len(self.graph) <= 64 and not self.forest:
                return 1
            return 2 * K + 2 + (self.jump_rounds() if self.forest else 1)
        return K + 1  # fused per-vertex encoder

    def jump_rounds(self) -> int:
        """Pointer-jumping launches per prepare (forest-form paths only)."""
        if not self.forest:
            return 0
        longest = max(int(self.features.path_lengths("b").max(initial=1)),
                      int(self.features.path_lengths("t").max(initial=1)))
        return int(np.ceil(np.log2(longest))) if longest > 1 else 0

    ENCODERS = {"dmma": 0, "fused": 1, "tc": 2}

    def set_encoder(self, mode=None, *, fused: bool | None = None):
        """Encoder implementation: ``"dmma"`` (default: aggregation kernels +
        fp64 tensor-core node MLPs, 1e-11 of the reference), ``"fused"`` (one
        per-vertex kernel in the reference's FMA order) or ``"tc"`` (bf16
        node MLPs on tcgen05 fed by TMA, split-bf16 operands, ~1e-5 relative;
        forward only).  A bool selects fused (True) / dmma (False)."""
        if fused is not None:
            mode = bool(fused)
        if isinstance(mode, bool):
            mode = "fused" if mode else "dmma"
        if mode not in self.ENCODERS:
            raise ValueError(f"encoder must be one of {sorted(self.ENCODERS)}")
        N.check(N.lib().fp_policy_set_encoder(self.handle, ctypes.c_int32(self.ENCODERS[mode])))
        self.encoder = mode
        self._prepared_key = None

    def flat_params(self, params) -> "object":
        """Upload a params dict (or pass through a flat CUDA tensor)."""
        import torch

        if isinstance(params, torch.Tensor):
            if params.dtype != torch.float64 or not params.is_cuda or params.numel() != self.layout.size:
                raise ValueError("flat params must be a CUDA float64 tensor of layout size")
            return params.contiguous()
        return torch.from_numpy(self.layout.flatten(params)).cuda()

    def prepare(self, params, stream=None):
        """Encode the graph for one parameter snapshot (2 encoder passes, as the
        reference's two _encode calls per episode, policy.py:348-350)."""
        flat = self.flat_params(params)
        self._flat = flat
        N.check(N.lib().fp_policy_prepare(self.handle, N.ptr(flat), N.stream_ptr(stream)))
        if not self.per_step:  # per_step encodes are counted by the rollout
            self.encode_count += 2
        return flat

    def read_table(self, name: str) -> np.ndarray:
        """Copy one device table (H_sel, H_plc, sel_logit, A, G, M, c) to host."""
        import torch

        p = ctypes.c_void_p()
        cnt = ctypes.c_int64()
        N.check(N.lib().fp_policy_table(self.handle, N.TABLE[name], ctypes.byref(p),
                                        ctypes.byref(cnt)))
        torch.cuda.synchronize()
        host = _DevPtrTensor.view(p.value, cnt.value).cpu().numpy().copy()
        n, h = len(self.graph), self.config.hidden
        return host.reshape(n, h) if name in ("H_sel", "H_plc", "A", "G") else host

    # ----------------------------------------------------------------- rollout
    def rollout_batch(self, params, B: int, epsilon: float, seed: int = 0, *,
                      mode: str = "sample", forced=None, simulate: bool = True,
                      strategy: str = "fifo", trace_steps: bool = False, grad: bool = False,
                      sim_trace: bool = False, episode_base: int = 0, prepare: bool = True,
                      stream=None, out: RolloutBatch | None = None,
                      wide: bool = False, tie_random: bool = False) -> RolloutBatch:
        import torch

        if mode not in N.MODE:
            raise ValueError(f"unknown mode {mode!r}")
        if strategy not in _STRATEGY_CODE:
            raise ValueError(f"unknown strategy {strategy!r}")
        if prepare:
            self.prepare(params, stream)
        n, d, h = len(self.graph), self.cluster.device_count, self.config.hidden
        dev = torch.device("cuda")
        if out is None:
            out = self.alloc_batch(B, trace_steps=trace_steps, grad=grad, simulate=simulate,
                                   sim_trace=sim_trace)
        ft = None
        if mode == "forced":
            ft = torch.as_tensor(np.asarray(forced, dtype=np.int32).reshape(B, n, 2),
                                 device=dev) if not isinstance(forced, torch.Tensor) else forced
            ft = ft.to(dtype=torch.int32).contiguous()
        flags = ((N.FLAG_WIDE if wide else 0) | (N.FLAG_TIE_RANDOM if tie_random else 0) |
                 (N.FLAG_PER_STEP if self.per_step else 0))
        # the argument block is cached on the output batch (its pointers are
        # fixed); per call only the scalars and the forced-action pointer change
        key = (B, mode, simulate, strategy, flags)
        args = getattr(out, "_args", None)
        if args is None or out._args_key != key:
            args = N.FpRolloutArgs(
                B, N.MODE[mode], 0.0, 0, 0, _STRATEGY_CODE[strategy], int(simulate),
                *[N.ptr(t).value for t in (None, out.assign, out.step_vd, out.step_lp,
                                           out.step_ent, out.step_argmax, out.step_ncand,
                                           out.makespan, out.status, out.grad_rows,
                                           out.grad_ep, out.trace)],
                out.trace.shape[1] // 16 if out.trace is not None else 0,
                N.ptr(out.trace_len).value, flags)
            ws = self.workspace(B, wide=wide, grad=out.grad_rows is not None)
            args.workspace = N.ptr(ws).value
            args.workspace_bytes = 0 if ws is None else ws.numel()
            out._args, out._args_key, out._ws = args, key, ws
        args.epsilon = float(epsilon)
        args.seed = int(seed) & ((1 << 64) - 1)
        args.episode_base = int(episode_base) & 0xFFFFFFFF
        args.forced = N.ptr(ft).value
        N.check(N.lib().fp_rollout_batch(self.sim.handle, self.handle, ctypes.byref(args),
                                         N.stream_ptr(stream)))
        if self.per_step:
            self.encode_count += 2 * n * B
        out._forced = ft
        return out

    def workspace(self, B: int, *, wide: bool = False, grad: bool = False):
        """Device scratch of the wide (HBM-resident) rollout for ``B`` episodes;
        None when the compact shared-memory kernel applies.  Cached, grown on
        demand."""
        import torch

        need = ctypes.c_int64()
        flags = (N.FLAG_WIDE if wide else 0) | (N.FLAG_PER_STEP if self.per_step else 0)
        N.check(N.lib().fp_rollout_workspace_size(
            self.sim.handle, self.handle, ctypes.c_int32(B), ctypes.c_int32(flags),
            ctypes.c_int32(int(grad)), ctypes.byref(need)))
        if need.value == 0:
            return None
        ws = getattr(self, "_ws", None)
        if ws is None or ws.numel() < need.value:
            self._ws = ws = torch.empty(need.value, dtype=torch.uint8, device="cuda")
        return ws

    def policy_gradient(self, batch: RolloutBatch, alpha, beta: float, grad=None, stream=None):
        """Flat parameter gradient of sum_e alpha_e * sum lp_e + beta * sum ent_e
        for a rollout made with ``grad=True`` (fp_pg_reduce + fp_policy_backward)."""
        import torch

        B = batch.assign.shape[0]
        alpha = torch.as_tensor(alpha, dtype=torch.float64, device="cuda").reshape(B).contiguous()
        if grad is None:
            grad = torch.empty(self.layout.size, dtype=torch.float64, device="cuda")
        self.reduce_gradient(batch.grad_rows, batch.grad_ep, batch.assign, alpha, beta, B, grad,
                             stream)
        batch._alpha = alpha
        return grad

    def reduce_gradient(self, grad_rows, grad_ep, assign, alpha, beta: float, B: int, grad,
                        stream=None) -> None:
        """Flat gradient of a REINFORCE rollout's decision records: the
        replay + episode reduction + backward (per_episode), or the
        backpropagation through every step's encode (per_step)."""
        if self.per_step:
            N.check(N.lib().fp_pg_reduce_per_step(
                self.handle, N.ptr(grad_rows), N.ptr(grad_ep), N.ptr(alpha),
                ctypes.c_double(beta), ctypes.c_int32(B), N.ptr(grad), N.stream_ptr(stream)))
            return
        N.check(N.lib().fp_pg_reduce(self.handle, N.ptr(grad_rows), N.ptr(grad_ep), N.ptr(assign),
                                     N.ptr(alpha), ctypes.c_double(beta), ctypes.c_int32(B),
                                     N.stream_ptr(stream)))
        N.check(N.lib().fp_policy_backward(self.handle, N.ptr(grad), N.stream_ptr(stream)))

    def grad_rec_stride(self) -> int:
        s = ctypes.c_int64()
        N.check(N.lib().fp_grad_rec_stride(self.handle, ctypes.c_int32(self.cluster.device_count),
                                           ctypes.byref(s)))
        return s.value

    def grad_ep_stride(self) -> int:
        s = ctypes.c_int64()
        N.check(N.lib().fp_grad_ep_stride(self.handle, ctypes.c_int32(self.cluster.device_count),
                                          ctypes.byref(s)))
        return s.value

    def alloc_batch(self, B: int, *, trace_steps=False, grad=False, simulate=True,
                    sim_trace=False) -> RolloutBatch:
        import torch

        n, d, h = len(self.graph), self.cluster.device_count, self.config.hidden
        dev = torch.device("cuda")
        i32, f64 = torch.int32, torch.float64
        rb = RolloutBatch(assign=torch.empty((B, n), dtype=i32, device=dev),
                          status=torch.empty(B, dtype=i32, device=dev),
                          makespan=torch.empty(B, dtype=f64, device=dev) if simulate else None)
        if trace_steps:
            rb.step_vd = torch.empty((B, n, 2), dtype=i32, device=dev)
            rb.step_lp = torch.empty((B, n, 2), dtype=f64, device=dev)
            rb.step_ent = torch.empty((B, n, 2), dtype=f64, device=dev)
            rb.step_argmax = torch.empty((B, n, 2), dtype=i32, device=dev)
            rb.step_ncand = torch.empty((B, n), dtype=i32, device=dev)
        if grad:
            # per-decision REINFORCE records (fp_grad_rec_stride doubles each)
            rb.grad_rows = torch.empty((B, n, self.grad_rec_stride()), dtype=f64, device=dev)
            rb.grad_ep = torch.empty((B, self.grad_ep_stride()), dtype=f64, device=dev)
        if sim_trace:
            cap = 2 * (n + n * d) + 2
            rb.trace = torch.empty((B, cap * 16), dtype=torch.uint8, device=dev)
            rb.trace_len = torch.empty(B, dtype=i32, device=dev)
        return rb

    def rollout(self, params, epsilon: float, seed: int, greedy: bool = False,
                teacher=None) -> tuple[Assignment, EpisodeTrace]:
        """One episode (reference policy.py:324-402): batch of one on the GPU."""
        n = len(self.graph)
        mode, forced = ("greedy" if greedy else "sample"), None
        if teacher is not None:
            if is_native_teacher(teacher):
                mode = "teacher"
            elif isinstance(teacher, ForcedActions):
                mode, forced = "forced", teacher.actions.reshape(1, n, 2)
            else:  # any object with select(candidates) / place(v, timeline)
                mode, forced = "forced", teacher_actions(self.graph, self.cluster, teacher)
        start = self.encode_count
        rb = self.rollout_batch(params, 1, epsilon, seed, mode=mode, forced=forced,
                                simulate=False, trace_steps=True)
        st = int(rb.status.cpu()[0])
        if st == N.EP_BAD_ACTION:
            raise TeacherActionError("teacher action outside the candidates / devices")
        if st != N.EP_OK:
            raise RuntimeError(f"rollout failed with status {st}")
        vd = rb.step_vd.cpu().numpy()[0]
        lp = rb.step_lp.cpu().numpy()[0]
        ent = rb.step_ent.cpu().numpy()[0]
        am = rb.step_argmax.cpu().numpy()[0]
        order = vd[:, 0].tolist()
        cands = _candidate_sets(self.graph, order)
        trace = EpisodeTrace()
        for t in range(n):
            trace.steps.append(TraceStep(
                step=t, candidates=cands[t], vertex=int(vd[t, 0]),
                sel_logprob=float(lp[t, 0]), device=int(vd[t, 1]),
                plc_logprob=float(lp[t, 1]), sel_entropy=float(ent[t, 0]),
                plc_entropy=float(ent[t, 1]), sel_argmax=int(am[t, 0]),
                plc_argmax=int(am[t, 1])))
        trace.encode_invocations = self.encode_count - start
        assign = rb.assign.cpu().numpy()[0]
        return Assignment(tuple(int(x) for x in assign), "doppler"), trace


class _DevPtrTensor:
    """Wrap a raw device pointer as a torch tensor (no copy)."""

    @staticmethod
    def view(ptr: int, count: int):
        import torch

        class _Holder:
            __cuda_array_interface__ = {"shape": (count,), "typestr": "<f8",
                                        "data": (ptr, False), "version": 3, "strides": None}
        return torch.as_tensor(_Holder(), device="cuda")


def assign_rollout(graph, cluster, params, config, epsilon, seed, greedy=False):
    return PolicyContext(graph, cluster, config).rollout(params, epsilon, seed, greedy=greedy)
