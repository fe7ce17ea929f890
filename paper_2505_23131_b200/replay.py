"""Schedule checks and reports over simulator traces (reference
``simulate.py:300-420``: ``utilization_report``, ``replay_violations``).

``replay_violations`` checks the same invariants as the reference -- every
begun task was enumerable with a free slot, slot capacities are never
exceeded, readiness never resets, times never decrease, no startable task
existed whenever time advanced (work conservation), every vertex ends ready
on its device, the recorded makespan is the last end -- but event-driven:
the reference re-enumerates all O(n*d) tasks at every event, this keeps the
per-resource counts of enumerable tasks up to date as readiness changes, so a
trace of a 100k-op episode (~10^6 events) is checked in seconds.  That is the
size-independent parity check for schedules far beyond the CPU oracle's reach.

Inputs are raw ``(tkind, v, a, b, time, etype)`` records (``decode_events``)
or a ``Schedule``.
"""

from __future__ import annotations

from .cluster import ClusterSpec
from .graph import DataflowGraph

_EPS = 1e-12


def _records(schedule_or_events):
    ev = getattr(schedule_or_events, "events", schedule_or_events)
    for e in ev:
        if isinstance(e, tuple):
            yield e
        else:  # simulate.Event
            t = e.task
            if t.kind == "exec":
                yield (0, t.vertex, t.device, -1, e.time_ms, 0 if e.type == "beg" else 1)
            else:
                yield (1, t.vertex, t.src, t.dst, e.time_ms, 0 if e.type == "beg" else 1)


def replay_violations(graph: DataflowGraph, assignment, cluster: ClusterSpec, schedule_or_events,
                      makespan_ms: float | None = None) -> list[str]:
    n, D = len(graph), cluster.device_count
    A = [int(x) for x in assignment]
    entry = [graph.is_entry(v) for v in range(n)]
    succs = [graph.succs(v) for v in range(n)]
    cons = [set(A[w] for w in succs[v]) - {A[v]} for v in range(n)]
    rdy = [set(range(D)) if entry[v] else set() for v in range(n)]
    missing = [sum(1 for p in graph.preds(v) if not entry[p]) for v in range(n)]
    begun_x = [False] * n
    begun_t: set[tuple[int, int]] = set()
    exec_free = list(cluster.exec_slots)
    tr_free = [list(r) for r in cluster.transfer_slots]
    pend_x = [0] * D                        # enumerable execs per device
    pend_t = [[0] * D for _ in range(D)]    # enumerable transfers per link
    for v in range(n):
        if not entry[v] and missing[v] == 0:
            pend_x[A[v]] += 1
    open_tasks: set[tuple] = set()
    out: list[str] = []
    t = 0.0
    max_end = 0.0

    def startable() -> bool:
        if any(exec_free[d] > 0 and pend_x[d] > 0 for d in range(D)):
            return True
        return any(tr_free[a][b] > 0 and pend_t[a][b] > 0 for a in range(D) for b in range(D))

    def became_ready(v: int, dev: int):
        rdy[v].add(dev)
        if dev == A[v]:  # its transfers to the consumer devices become enumerable
            for b in cons[v]:
                if b not in rdy[v] and (v, b) not in begun_t:
                    pend_t[dev][b] += 1
        for w in succs[v]:
            if A[w] == dev and not entry[v]:
                missing[w] -= 1
                if missing[w] == 0 and not begun_x[w]:
                    pend_x[dev] += 1

    for kind, v, a, b, time, etype in _records(schedule_or_events):
        if time < t - _EPS:
            out.append(f"time-order: event at {time} after time {t}")
        if time > t + _EPS:
            if startable():
                out.append(f"work-conservation: idle advance from t={t} to t={time} "
                           f"with a startable task")
            t = time
        if etype == 0:  # beg
            if kind == 0:
                ok = (not entry[v]) and a == A[v] and not begun_x[v] and missing[v] == 0
                if ok:
                    pend_x[a] -= 1
                begun_x[v] = True
                exec_free[a] -= 1
                if exec_free[a] < 0:
                    out.append(f"resource-overflow: exec slots on device {a} at t={t}")
            else:
                ok = (a == A[v] and a in rdy[v] and b in cons[v] and b not in rdy[v]
                      and (v, b) not in begun_t)
                if ok:
                    pend_t[a][b] -= 1
                begun_t.add((v, b))
                tr_free[a][b] -= 1
                if tr_free[a][b] < 0:
                    out.append(f"resource-overflow: transfer slots {a}->{b} at t={t}")
            if not ok:
                out.append(f"invalid-start: {('exec', 'transfer')[kind]} {(v, a, b)} not "
                           f"enumerable at t={t}")
            open_tasks.add((kind, v, a, b))
        else:  # end
            if (kind, v, a, b) not in open_tasks:
                out.append(f"dangling-end: {(kind, v, a, b)} ends at t={t} without a beg")
            else:
                open_tasks.discard((kind, v, a, b))
            dev = a if kind == 0 else b
            if kind == 0:
                exec_free[a] += 1
            else:
                tr_free[a][b] += 1
            if dev in rdy[v]:
                out.append(f"readiness-reset: vertex {v} already ready on device {dev} at t={t}")
            else:
                became_ready(v, dev)
            max_end = max(max_end, time)
    for v in range(n):
        if A[v] not in rdy[v]:
            out.append(f"incomplete: vertex {v} never became ready on its device")
    mk = getattr(schedule_or_events, "makespan_ms", makespan_ms)
    if mk is not None and abs(mk - max_end) > 1e-9:
        out.append(f"makespan-mismatch: recorded {mk}, max end {max_end}")
    return out


def _union_length(intervals):
    total, last = 0.0, None
    for beg, end in sorted(intervals):
        if last is None or beg > last:
            total += end - beg
            last = end
        elif end > last:
            total += end - last
            last = end
    return total


def utilization_report(schedule_or_events, cluster: ClusterSpec,
                       makespan_ms: float | None = None) -> dict:
    """Per-device busy fraction of [0, makespan] and per-link transfer
    intervals (reference ``simulate.py:314-343``)."""
    mk = getattr(schedule_or_events, "makespan_ms", makespan_ms)
    D = cluster.device_count
    exec_iv = {d: [] for d in range(D)}
    link_iv: dict[tuple[int, int], list] = {}
    opened = {}
    for kind, v, a, b, time, etype in _records(schedule_or_events):
        key = (kind, v, a, b)
        if etype == 0:
            opened[key] = time
            continue
        beg = opened.pop(key)
        if kind == 0:
            exec_iv[a].append((beg, time))
        else:
            link_iv.setdefault((a, b), []).append((beg, time))
    devices = []
    for d in range(D):
        busy = _union_length(exec_iv[d])
        devices.append({"device": d, "busy_ms": busy,
                        "busy_fraction": busy / mk if mk and mk > 0 else 0.0,
                        "intervals": [[x, y] for x, y in sorted(exec_iv[d])]})
    links = [{"src": s, "dst": t, "intervals": [[x, y] for x, y in sorted(iv)]}
             for (s, t), iv in sorted(link_iv.items())]
    return {"makespan_ms": mk, "devices": devices, "links": links}
