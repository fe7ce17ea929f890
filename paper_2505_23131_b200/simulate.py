"""Work-conserving simulator API — drop-in for reference ``flowplace/simulate.py``.

``exec_time`` keeps the reference signature and result
(``simulate.py:251-266``): ``(makespan_ms, Schedule)``, raising
``DeadlockError(time_ms, blocked)`` on an inconsistent graph/assignment and
``ValueError`` on a bad assignment or strategy.  The core is the CUDA
simulator (``csrc/fp_sim.cuh``) behind the C ABI; ``backend_name()`` reports
``"cuda"`` and there is no CPU fallback.

Beyond the reference: ``SimProblem`` keeps one graph + cluster resident on the
GPU and simulates batches of assignments (``exec_time_batch``) — the
throughput form every batched consumer (RL rollouts, brute force, critical
path trials) uses.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .cluster import ClusterSpec
from .features import StaticGraphFeatures, static_features
from .graph import DataflowGraph

STRATEGIES = ("fifo", "depth_first", "breadth_first")
_STRATEGY_CODE = {"fifo": 0, "depth_first": 1, "breadth_first": 2}


class DeadlockError(RuntimeError):
    """Nothing in flight yet vertices remain (reference ``_simpy.py:21-28``)."""

    def __init__(self, time_ms: float, blocked: list[int]):
        self.time_ms = time_ms
        self.blocked = blocked
        super().__init__(f"no pending events at t={time_ms} ms with unfinished vertices; "
                         f"blocked frontier: {blocked}")


def backend_name() -> str:
    forced = os.environ.get("FLOWPLACE_SIM_BACKEND", "auto")
    if forced not in ("auto", "cuda"):
        raise RuntimeError(f"FLOWPLACE_SIM_BACKEND={forced!r}: this build only has the CUDA core")
    return "cuda"


@dataclass(frozen=True)
class Task:
    kind: str
    vertex: int
    device: int | None = None
    src: int | None = None
    dst: int | None = None

    @staticmethod
    def exec_(vertex: int, device: int) -> "Task":
        return Task("exec", vertex, device=device)

    @staticmethod
    def transfer(vertex: int, src: int, dst: int) -> "Task":
        return Task("transfer", vertex, src=src, dst=dst)


@dataclass(frozen=True)
class Event:
    task: Task
    time_ms: float
    type: str


@dataclass
class Schedule:
    events: tuple[Event, ...]
    makespan_ms: float


def _check_strategy(strategy: str) -> int:
    if strategy not in _STRATEGY_CODE:
        raise ValueError(f"unknown strategy {strategy!r}; expected one of {STRATEGIES}")
    return _STRATEGY_CODE[strategy]


def _check_assignment(assign: np.ndarray, n: int, d: int) -> np.ndarray:
    if assign.shape[-1:] != (n,):
        raise ValueError(f"assignment must map all {n} vertices")
    if n and (assign.min() < 0 or assign.max() >= d):
        raise ValueError("assignment names a device outside the cluster")
    return assign


def _pack(graph: DataflowGraph, assignment, cluster: ClusterSpec,
          features: StaticGraphFeatures | None, strategy: str, seed: int):
    """The reference's packed tuple (``simulate.py:194-237``), from the graph's
    cached CSR."""
    n = len(graph)
    d = cluster.device_count
    assign = _check_assignment(np.asarray(list(assignment), dtype=np.int32), n, d)
    code = _check_strategy(strategy)
    if features is None and strategy != "fifo":
        features = static_features(graph, cluster.comm_factor)
    c = graph.csr()
    cp = cluster.packed()
    if features is not None:
        tlev = np.ascontiguousarray(features.t_level)
        blev = np.ascontiguousarray(features.b_level)
    else:
        tlev = np.zeros(n)
        blev = np.zeros(n)
    return (n, d, c["pred_indptr"], c["pred_indices"], c["succ_indptr"], c["succ_indices"],
            c["is_entry"], c["flops"], c["obytes"], assign, cp["rates"], cp["bw"],
            cp["eslots"], cp["tslots"], tlev, blev, code, float(cluster.comm_factor),
            float(cluster.jitter_sigma), int(seed))


def run_packed(n, d, pred_indptr, pred_indices, succ_indptr, succ_indices, is_entry, flops,
               obytes, assign, rates, bw, eslots, tslots, tlev, blev, strategy, comm_factor,
               sigma, seed):
    """Drop-in for ``flowplace._simcore.run_packed`` (``_simcore.pyx:39-45``):
    same arguments, returns ``(makespan, [(tkind, v, a, b, time, etype)])``."""
    arrs = [np.ascontiguousarray(x, dtype=t) for x, t in (
        (pred_indptr, np.int32), (pred_indices, np.int32), (succ_indptr, np.int32),
        (succ_indices, np.int32), (is_entry, np.uint8), (flops, np.float64),
        (obytes, np.float64), (assign, np.int32), (rates, np.float64), (bw, np.float64),
        (eslots, np.int32), (tslots, np.int32), (tlev, np.float64), (blev, np.float64))]
    cap = 2 * (n + n * d) + 2
    events = np.zeros(cap, dtype=N.EVENT_DTYPE)
    blocked = np.zeros(max(n, 1), dtype=np.uint8)
    mk = ctypes.c_double(0.0)
    ne = ctypes.c_int64(0)
    rc = N.lib().fp_run_packed(
        ctypes.c_int32(n), ctypes.c_int32(d), *[N.ptr(a) for a in arrs], ctypes.c_int32(strategy),
        ctypes.c_double(comm_factor), ctypes.c_double(sigma), ctypes.c_int64(seed),
        ctypes.byref(mk), N.ptr(events), ctypes.c_int64(cap), ctypes.byref(ne), N.ptr(blocked))
    if rc == N.FP_ERR_DEADLOCK:
        raise DeadlockError(mk.value, [int(v) for v in np.nonzero(blocked[:n])[0]])
    N.check(rc)
    ev = events[: ne.value]
    raw = list(zip(ev["kind"].tolist(), ev["v"].tolist(), ev["a"].tolist(), ev["b"].tolist(),
                   ev["time"].tolist(), ev["etype"].tolist()))
    return mk.value, raw


def _assemble(makespan: float, raw_events) -> Schedule:
    out = []
    for kind, v, a, b, time, etype in raw_events:
        task = Task.exec_(v, a) if kind == 0 else Task.transfer(v, a, b)
        out.append(Event(task, time, "beg" if etype == 0 else "end"))
    return Schedule(tuple(out), makespan)


def exec_time(graph: DataflowGraph, assignment, cluster: ClusterSpec,
              strategy: str = "fifo", seed: int = 0,
              features: StaticGraphFeatures | None = None) -> tuple[float, Schedule]:
    """Simulate one assignment on the GPU core; ``(makespan_ms, Schedule)``."""
    backend_name()
    makespan, raw = run_packed(*_pack(graph, assignment, cluster, features, strategy, seed))
    return makespan, _assemble(makespan, raw)


class SimProblem:
    """One graph + cluster resident on the current CUDA device (``fp_problem``)."""

    def __init__(self, graph: DataflowGraph, cluster: ClusterSpec,
                 features: StaticGraphFeatures | None = None):
        self.graph = graph
        self.cluster = cluster
        self.n = len(graph)
        self.d = cluster.device_count
        self.features = features if features is not None else static_features(
            graph, cluster.comm_factor)
        c = graph.csr()
        cp = cluster.packed()
        self._keep = dict(c, **cp, tlev=np.ascontiguousarray(self.features.t_level),
                          blev=np.ascontiguousarray(self.features.b_level))
        k = self._keep
        desc = N.FpGraphDesc(self.n, self.d, *[N.ptr(k[x]).value or None for x in (
            "pred_indptr", "pred_indices", "succ_indptr", "succ_indices", "is_entry", "flops",
            "obytes", "rates", "bw", "eslots", "tslots", "tlev", "blev")],
                             float(cluster.comm_factor))
        handle = ctypes.c_void_p()
        N.check(N.lib().fp_problem_create(ctypes.byref(desc), ctypes.byref(handle)))
        self.handle = handle
        self._lib = N.lib()

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self._lib.fp_problem_destroy(h)
            self.handle = None

    def jitter_table(self, seed: int):
        """Reference-exact jitter factors for one seed (host libm), or None."""
        if self.cluster.jitter_sigma <= 0.0:
            return None
        out = np.empty(self.n * self.d * (self.d + 1), dtype=np.float64)
        N.check(N.lib().fp_jitter_tables(ctypes.c_int32(self.n), ctypes.c_int32(self.d),
                                         ctypes.c_double(self.cluster.jitter_sigma),
                                         ctypes.c_int64(seed), N.ptr(out)))
        return out

    def workspace(self, B: int, wide: bool = False):
        """Device scratch for ``B`` simulations (None on the compact shared-memory
        path); cached and grown on demand."""
        import torch

        need = ctypes.c_int64()
        N.check(N.lib().fp_sim_workspace_size(self.handle, ctypes.c_int32(B),
                                              ctypes.c_int32(N.FLAG_WIDE if wide else 0),
                                              ctypes.byref(need)))
        if need.value == 0:
            return None
        ws = getattr(self, "_ws", None)
        if ws is None or ws.numel() < need.value:
            self._ws = ws = torch.empty(need.value, dtype=torch.uint8, device="cuda")
        return ws

    def simulate(self, assign, strategy: str = "fifo", *, jitter=None, trace: bool = False,
                 stream=None, wide: bool = False):
        """Batched simulation of device-resident int32 assignments [B, n].

        Returns a dict of device tensors: makespan [B] f64, status [B] i32 and,
        with ``trace``, events [B, cap] (uint8 view of fp_event records) and
        trace_len [B]."""
        import torch

        code = _check_strategy(strategy)
        if assign.dtype != torch.int32 or not assign.is_cuda or assign.dim() != 2:
            raise ValueError("assign must be a CUDA int32 tensor [B, n]")
        assign = assign.contiguous()
        B = assign.shape[0]
        dev = assign.device
        out = {"makespan": torch.empty(B, dtype=torch.float64, device=dev),
               "status": torch.empty(B, dtype=torch.int32, device=dev)}
        cap = 2 * (self.n + self.n * self.d) + 2 if trace else 0
        if trace:
            out["events"] = torch.empty((B, cap * 16), dtype=torch.uint8, device=dev)
            out["trace_len"] = torch.empty(B, dtype=torch.int32, device=dev)
            out["blocked"] = torch.zeros((B, max(self.n, 1)), dtype=torch.uint8, device=dev)
        jstride = 0
        if jitter is not None:
            jitter = jitter.contiguous()
            jstride = jitter.shape[-1] if jitter.dim() == 2 else 0
        ws = self.workspace(B, wide)
        N.check(N.lib().fp_sim_batch(
            self.handle, N.ptr(assign), ctypes.c_int32(B), ctypes.c_int32(code), N.ptr(jitter),
            ctypes.c_int64(jstride), N.ptr(out["makespan"]), N.ptr(out["status"]),
            N.ptr(out.get("events")), ctypes.c_int32(cap), N.ptr(out.get("trace_len")),
            N.ptr(out.get("blocked")), N.ptr(ws), ctypes.c_int64(0 if ws is None else ws.numel()),
            ctypes.c_int32(N.FLAG_WIDE if wide else 0), N.stream_ptr(stream)))
        return out


def decode_events(events_u8, length: int) -> list[tuple]:
    """Raw (tkind, v, a, b, time, etype) records from one trace row."""
    arr = np.frombuffer(np.ascontiguousarray(events_u8).tobytes(), dtype=N.EVENT_DTYPE)[:length]
    return list(zip(arr["kind"].tolist(), arr["v"].tolist(), arr["a"].tolist(),
                    arr["b"].tolist(), arr["time"].tolist(), arr["etype"].tolist()))


def exec_time_batch(graph: DataflowGraph, assignments, cluster: ClusterSpec,
                    strategy: str = "fifo", features: StaticGraphFeatures | None = None,
                    seed: int = 0, schedules: bool = False):
    """Makespans of many assignments of one graph in one GPU launch.
    Returns ``np.ndarray[B]`` (and the Schedules when ``schedules``)."""
    import torch

    prob = SimProblem(graph, cluster, features)
    a = _check_assignment(np.asarray(assignments, dtype=np.int32).reshape(-1, len(graph)),
                          len(graph), cluster.device_count)
    at = torch.from_numpy(a).cuda()
    jit = prob.jitter_table(seed)
    jt = torch.from_numpy(jit).cuda() if jit is not None else None
    out = prob.simulate(at, strategy, jitter=jt, trace=schedules)
    st = out["status"].cpu().numpy()
    mk = out["makespan"].cpu().numpy()
    if (st == N.EP_DEADLOCK).any():
        b = int(np.nonzero(st == N.EP_DEADLOCK)[0][0])
        blocked = out["blocked"][b].cpu().numpy() if schedules else None
        raise DeadlockError(float(mk[b]), [] if blocked is None else
                            [int(v) for v in np.nonzero(blocked[: len(graph)])[0]])
    if not schedules:
        return mk
    ev = out["events"].cpu().numpy()
    tl = out["trace_len"].cpu().numpy()
    return mk, [_assemble(float(mk[b]), decode_events(ev[b], int(tl[b]))) for b in range(len(mk))]


def schedule_to_dict(schedule: Schedule) -> dict:
    return {"makespan_ms": schedule.makespan_ms,
            "events": [{"task": {"kind": e.task.kind, "vertex": e.task.vertex,
                                 "src": e.task.src, "dst": e.task.dst,
                                 "device": e.task.device},
                        "time_ms": e.time_ms, "type": e.type} for e in schedule.events]}


def schedule_from_dict(doc: dict) -> Schedule:
    evs = []
    for rec in doc["events"]:
        t = rec["task"]
        task = (Task.exec_(t["vertex"], t["device"]) if t["kind"] == "exec"
                else Task.transfer(t["vertex"], t["src"], t["dst"]))
        evs.append(Event(task, rec["time_ms"], rec["type"]))
    return Schedule(tuple(evs), doc["makespan_ms"])
