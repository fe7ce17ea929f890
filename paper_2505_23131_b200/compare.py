"""Clean-vs-jittered comparison of placements: the evaluation core of the
reference's ``compare`` command (``cli.py:316-366``) and its correlation
metrics (``metrics.py:8-40``), without the CLI / manifest plumbing (out of
scope).

The reference evaluates each assignment with one clean ``exec_time`` plus
``trials`` jittered ones (seeds ``seed + t``), one Python call after another.
Here every (assignment, run) pair is one episode of a single batched GPU
simulation launch (``fp_sim_batch``), each jittered episode carrying the
reference-exact host jitter table of its seed, so the makespans -- and the
row statistics computed from them with the reference's own numpy reductions
-- are identical to the per-call loop.
"""

from __future__ import annotations

import numpy as np

from .cluster import ClusterSpec
from .graph import DataflowGraph

ENGINES = ("critical_path", "enumopt", "random", "single", "doppler")


def pearson(x, y) -> float:
    """Pearson correlation (reference ``metrics.py:8-20``, same errors)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if x.shape != y.shape or x.ndim != 1:
        raise ValueError(f"need two equal-length 1-D series, got {x.shape} and {y.shape}")
    if x.size < 2:
        raise ValueError("need at least two points")
    cx, cy = x - x.mean(), y - y.mean()
    denom = np.sqrt((cx * cx).sum() * (cy * cy).sum())
    if denom == 0.0:
        raise ValueError("a constant series has no defined correlation")
    return float((cx * cy).sum() / denom)


def average_ranks(x) -> np.ndarray:
    """1-based ranks, ties sharing the mean of the ranks they span
    (reference ``metrics.py:23-34``)."""
    x = np.asarray(x, dtype=np.float64)
    order = np.argsort(x, kind="stable")
    xs = x[order]
    # run boundaries of equal values in sorted order
    starts = np.flatnonzero(np.r_[True, xs[1:] != xs[:-1]])
    ends = np.r_[starts[1:], x.size] - 1
    ranks = np.empty(x.size, dtype=np.float64)
    ranks[order] = np.repeat((starts + ends) / 2.0 + 1.0, ends - starts + 1)
    return ranks


def spearman(x, y) -> float:
    """Spearman rank correlation (reference ``metrics.py:37-40``)."""
    return pearson(average_ranks(x), average_ranks(y))


def compare_assignments(graph: DataflowGraph, cluster: ClusterSpec, assignments,
                        trials: int, jitter_sigma: float, seed: int = 0,
                        strategy: str = "fifo", features=None) -> dict:
    """``assignments``: ordered ``(name, assignment)`` pairs.  Returns the
    reference's ``compare.json`` document ``{"rows", "pearson", "spearman"}``
    (rows: engine, clean_ms, noisy_mean_ms, noisy_std_ms)."""
    import torch

    from . import _native as N
    from .simulate import DeadlockError, SimProblem, _check_assignment

    names = [name for name, _ in assignments]
    A = len(names)
    n = len(graph)
    if trials < 0:
        raise ValueError("trials must be >= 0")
    assign = _check_assignment(
        np.asarray([list(a) for _, a in assignments], dtype=np.int32).reshape(A, n), n,
        cluster.device_count)
    jittered = ClusterSpec.from_dict({**cluster.to_dict(), "jitter_sigma": jitter_sigma})
    clean_prob = SimProblem(graph, cluster, features)
    noisy_prob = SimProblem(graph, jittered, clean_prob.features)

    def run(prob, a_rows, seeds):
        at = torch.from_numpy(np.ascontiguousarray(a_rows)).cuda()
        jt = None
        if prob.cluster.jitter_sigma > 0:
            tabs = {sd: prob.jitter_table(sd) for sd in set(seeds)}
            jt = torch.from_numpy(np.stack([tabs[sd] for sd in seeds])).cuda()
        out = prob.simulate(at, strategy, jitter=jt)
        st = out["status"].cpu().numpy()
        mk = out["makespan"].cpu().numpy()
        if (st == N.EP_DEADLOCK).any():
            b = int(np.flatnonzero(st == N.EP_DEADLOCK)[0])
            raise DeadlockError(float(mk[b]), [])
        return mk

    clean = run(clean_prob, assign, [0] * A)  # exec_time(..., seed=0), cli.py:339
    if trials:
        # episode (i, t) = assignment i under seed + t, cli.py:340-341
        rows = np.repeat(assign, trials, axis=0)
        noisy = run(noisy_prob, rows, [seed + t for _ in range(A) for t in range(trials)])
        noisy = noisy.reshape(A, trials)
    out_rows, clean_series, noisy_series = [], [], []
    for i, name in enumerate(names):
        series = [float(x) for x in noisy[i]] if trials else []
        mean = float(np.mean(series))
        out_rows.append({"engine": name, "clean_ms": float(clean[i]), "noisy_mean_ms": mean,
                         "noisy_std_ms": float(np.std(series))})
        clean_series.append(float(clean[i]))
        noisy_series.append(mean)
    return {"rows": out_rows, "pearson": pearson(clean_series, noisy_series),
            "spearman": spearman(clean_series, noisy_series)}


def engine_assignment(engine: str, graph: DataflowGraph, cluster: ClusterSpec, *,
                      trials: int = 50, seed: int = 0, strategy: str = "fifo",
                      params=None, pconfig=None):
    """The assignment an engine proposes (reference ``cli.py:191-210``)."""
    from . import heuristics as H

    if engine == "critical_path":
        return H.critical_path_assign(graph, cluster, trials=trials, seed=seed, strategy=strategy)
    if engine == "random":
        return H.random_assign(graph, cluster.device_count, seed=seed)
    if engine == "single":
        return H.single_device_assign(graph)
    if engine == "doppler":
        if params is None or pconfig is None:
            raise ValueError("engine doppler requires a checkpoint (params, pconfig)")
        from .policy import PolicyContext

        assignment, _ = PolicyContext(graph, cluster, pconfig).rollout(params, 0.0, seed,
                                                                       greedy=True)
        return assignment
    if engine == "enumopt":
        raise ValueError("engine enumopt (the enumerative optimizer) is outside this "
                         "package's scope (DESIGN.md section 7)")
    raise ValueError(f"unknown engine {engine!r}")


def compare(graph: DataflowGraph, cluster: ClusterSpec, engines=("critical_path", "random"),
            trials: int = 10, probe_assignments: int = 0, jitter_sigma: float = 0.1,
            seed: int = 0, strategy: str = "fifo", params=None, pconfig=None) -> dict:
    """``cmd_compare`` without the output directory: engines' assignments,
    then ``probe_assignments`` random probes (seeds ``seed + 1000 + k``),
    all evaluated in one batched simulation."""
    for e in engines:
        if e not in ENGINES:
            raise ValueError(f"unknown engine {e!r}")
    from .heuristics import random_assign

    pairs = [(e, engine_assignment(e, graph, cluster, trials=trials, seed=seed,
                                   strategy=strategy, params=params, pconfig=pconfig))
             for e in engines]
    pairs += [(f"probe_{k}", random_assign(graph, cluster.device_count, seed=seed + 1000 + k))
              for k in range(probe_assignments)]
    return compare_assignments(graph, cluster, pairs, trials, jitter_sigma, seed, strategy)
