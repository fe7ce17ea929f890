"""ORACLE — test infrastructure only (tests/, __graft_entry__.smoke(),
bench.py's cpu_baseline / --impl reference leg).  Never imported by the
product package.

ctypes front end of ``oracle/wc_sim.c``, the C restatement of the reference
simulator core ``flowplace/_simcore.pyx:39-248``.  ``run_packed`` keeps the
reference signature and return shape ``(makespan, [(tkind, v, a, b, time,
etype), ...])`` (``_simpy.py:7-9``); ``pack`` restates ``simulate._pack``
(``simulate.py:194-237``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB = None

STRATEGY_CODE = {"fifo": 0, "depth_first": 1, "breadth_first": 2}


class OracleDeadlock(RuntimeError):
    def __init__(self, time_ms: float, blocked: list[int]):
        self.time_ms = time_ms
        self.blocked = blocked
        super().__init__(f"no pending events at t={time_ms} ms with unfinished vertices; "
                         f"blocked frontier: {blocked}")


class _Event(ctypes.Structure):
    _fields_ = [("time", ctypes.c_double), ("v", ctypes.c_int32), ("kind", ctypes.c_int8),
                ("etype", ctypes.c_int8), ("a", ctypes.c_int8), ("b", ctypes.c_int8)]


def build() -> Path:
    so = _HERE / "liboracle.so"
    src = _HERE / "wc_sim.c"
    if not so.exists() or so.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return so


def lib():
    global _LIB
    if _LIB is None:
        _LIB = ctypes.CDLL(str(build()))
        _LIB.oracle_run_packed.restype = ctypes.c_int
        _LIB.oracle_jitter_factor.restype = ctypes.c_double
        _LIB.oracle_jitter_factor.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_int, ctypes.c_double]
    return _LIB


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def pack(graph, assignment, cluster, features=None, strategy="fifo", seed=0):
    """The reference's packed problem tuple for ``run_packed``."""
    n = len(graph)
    d = cluster.device_count
    assign = np.asarray(list(assignment), dtype=np.int32)
    if assign.shape != (n,):
        raise ValueError(f"assignment must map all {n} vertices")
    if n and (assign.min() < 0 or assign.max() >= d):
        raise ValueError("assignment names a device outside the cluster")
    if strategy not in STRATEGY_CODE:
        raise ValueError(f"unknown strategy {strategy!r}")
    pi = np.zeros(n + 1, dtype=np.int32)
    si = np.zeros(n + 1, dtype=np.int32)
    for v in range(n):
        pi[v + 1] = pi[v] + len(graph.preds(v))
        si[v + 1] = si[v] + len(graph.succs(v))
    pv = np.asarray([u for v in range(n) for u in graph.preds(v)], dtype=np.int32)
    sv = np.asarray([w for v in range(n) for w in graph.succs(v)], dtype=np.int32)
    entry = np.asarray([1 if graph.is_entry(v) else 0 for v in range(n)], dtype=np.uint8)
    flops = np.asarray([x.flops for x in graph.vertices], dtype=np.float64)
    obytes = np.asarray([x.output_bytes for x in graph.vertices], dtype=np.float64)
    if features is not None:
        tlev = np.ascontiguousarray(features.matrix[:, 3], dtype=np.float64)
        blev = np.ascontiguousarray(features.matrix[:, 4], dtype=np.float64)
    else:
        tlev = np.zeros(n)
        blev = np.zeros(n)
    return (n, d, pi, pv, si, sv, entry, flops, obytes, assign,
            np.asarray(cluster.rates, dtype=np.float64),
            np.asarray(cluster.bandwidth, dtype=np.float64).reshape(d * d),
            np.asarray(cluster.exec_slots, dtype=np.int32),
            np.asarray(cluster.transfer_slots, dtype=np.int32).reshape(d * d),
            tlev, blev, STRATEGY_CODE[strategy], float(cluster.comm_factor),
            float(cluster.jitter_sigma), int(seed))


def run_packed(n, d, pred_indptr, pred_indices, succ_indptr, succ_indices, is_entry,
               flops, obytes, assign, rates, bw, eslots, tslots, tlev, blev, strategy,
               comm_factor, sigma, seed, want_events=True):
    arrs = [np.ascontiguousarray(x, dtype=t) for x, t in (
        (pred_indptr, np.int32), (pred_indices, np.int32), (succ_indptr, np.int32),
        (succ_indices, np.int32), (is_entry, np.uint8), (flops, np.float64),
        (obytes, np.float64), (assign, np.int32), (rates, np.float64), (bw, np.float64),
        (eslots, np.int32), (tslots, np.int32), (tlev, np.float64), (blev, np.float64))]
    cap = 2 * (n + n * d) + 2
    ev = (_Event * cap)() if want_events else None
    mk = ctypes.c_double(0.0)
    ne = ctypes.c_int64(0)
    dl = ctypes.c_double(0.0)
    blocked = np.zeros(max(n, 1), dtype=np.uint8)
    rc = lib().oracle_run_packed(
        ctypes.c_int(n), ctypes.c_int(d), *[_p(a) for a in arrs], ctypes.c_int(strategy),
        ctypes.c_double(comm_factor), ctypes.c_double(sigma), ctypes.c_int64(seed),
        ctypes.byref(mk), ev, ctypes.c_int64(cap), ctypes.byref(ne), ctypes.byref(dl),
        _p(blocked))
    if rc == 1:
        raise OracleDeadlock(dl.value, [int(v) for v in np.nonzero(blocked[:n])[0]])
    if rc != 0:
        raise RuntimeError(f"oracle_run_packed failed rc={rc}")
    events = []
    if want_events:
        for i in range(ne.value):
            e = ev[i]
            events.append((int(e.kind), int(e.v), int(e.a), int(e.b), float(e.time), int(e.etype)))
    return mk.value, events


def exec_time(graph, assignment, cluster, strategy="fifo", seed=0, features=None):
    """(makespan, raw events) of one assignment through the C oracle core."""
    if features is None and strategy != "fifo":
        from paper_2505_23131_b200.features import static_features
        features = static_features(graph, cluster.comm_factor)
    return run_packed(*pack(graph, assignment, cluster, features, strategy, seed))


def sim_batch(packed, assigns: np.ndarray) -> np.ndarray:
    """Makespans of B x n assignments (no trace) through ``oracle_sim_batch``."""
    (n, d, pi, pv, si, sv, entry, flops, obytes, _a, rates, bw, es, ts, tl, bl, strat,
     cf, _s, _seed) = packed
    assigns = np.ascontiguousarray(assigns, dtype=np.int32)
    B = assigns.shape[0]
    mk = np.zeros(B)
    st = np.zeros(B, dtype=np.int32)
    arrs = [np.ascontiguousarray(x) for x in (pi, pv, si, sv, entry, flops, obytes)]
    lib().oracle_sim_batch(ctypes.c_int(n), ctypes.c_int(d), *[_p(a) for a in arrs],
                           _p(assigns), ctypes.c_int(B),
                           *[_p(np.ascontiguousarray(a)) for a in (rates, bw, es, ts, tl, bl)],
                           ctypes.c_int(strat), ctypes.c_double(cf), _p(mk), _p(st))
    return mk
