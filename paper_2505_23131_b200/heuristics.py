"""Assignments and the critical-path rule (mirror of reference
``heuristics.py:35-91``).  ``CriticalPathRule`` is the imitation teacher; the
CUDA rollout executes it natively (FP_MODE_TEACHER), so here it only carries
identity and the host-side reference semantics for single calls."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Assignment:
    device_of: tuple[int, ...]
    engine: str = ""

    def __getitem__(self, v: int) -> int:
        return self.device_of[v]

    def __iter__(self):
        return iter(self.device_of)

    def __len__(self) -> int:
        return len(self.device_of)


def validate_assignment(graph, assignment, device_count: int) -> list[str]:
    devs = list(assignment)
    if len(devs) != len(graph):
        return [f"not-total: {len(devs)} entries for {len(graph)} vertices"]
    return [f"bad-device: vertex {v} on device {d} of {device_count}"
            for v, d in enumerate(devs) if not 0 <= d < device_count]


def single_device_assign(graph) -> Assignment:
    return Assignment((0,) * len(graph), "single")


def random_assign(graph, devices: int, seed: int = 0) -> Assignment:
    rng = np.random.default_rng(seed)
    return Assignment(tuple(int(d) for d in rng.integers(0, devices, size=len(graph))), "random")


class CriticalPathRule:
    """Select the candidate with the largest t-level (ties: smallest id);
    place on the earliest-start device (ties: smallest id).  Executed on the
    GPU inside the rollout kernel when passed as ``teacher``."""

    def __init__(self, graph, cluster, features):
        self.graph = graph
        self.cluster = cluster
        self.features = features

    def select(self, candidates, rng=None) -> int:
        tlev = self.features.t_level
        best = max(tlev[v] for v in candidates)
        top = [v for v in candidates if tlev[v] == best]
        if rng is None or len(top) == 1:
            return top[0]
        return top[int(rng.integers(len(top)))]

    def place(self, v: int, timeline: "PlacementTimeline") -> int:
        """Earliest-start device, smallest id on ties (heuristics.py:83-91).
        The GPU teacher computes the same argmin from its device features."""
        starts = [timeline.earliest_start(v, d) for d in range(self.cluster.device_count)]
        return min(range(len(starts)), key=starts.__getitem__)


class PlacementTimeline:
    """Host model of committed placements for ``CriticalPathRule.place``
    (reference ``timeline.py:19-58``).  The rollout kernel keeps the same
    per-episode state on chip; this mirror serves host callers.  Inputs
    (entry vertices) cost nothing and are ready everywhere at t = 0."""

    def __init__(self, graph, cluster):
        self.graph, self.cluster = graph, cluster
        n, nd = len(graph), cluster.device_count
        self.device = [-1] * n
        self.start, self.end = [0.0] * n, [0.0] * n
        self.device_avail, self.assigned_flops = [0.0] * nd, [0.0] * nd

    def arrival_time(self, pred: int, device: int) -> float:
        if self.graph.is_entry(pred):
            return 0.0
        if self.device[pred] < 0:
            raise ValueError(f"predecessor {pred} is not assigned yet")
        nbytes = self.graph.vertices[pred].output_bytes
        return self.end[pred] + self.cluster.transfer_duration(nbytes, self.device[pred], device)

    def inputs_ready_time(self, v: int, device: int) -> float:
        ready = [self.arrival_time(u, device) for u in self.graph.preds(v)]
        return max(ready) if ready else 0.0

    def earliest_start(self, v: int, device: int) -> float:
        return max(self.device_avail[device], self.inputs_ready_time(v, device))

    def commit(self, v: int, device: int) -> None:
        if self.device[v] >= 0:
            raise ValueError(f"vertex {v} is already placed")
        fl = self.graph.vertices[v].flops
        self.device[v] = device
        self.assigned_flops[device] += fl
        if not self.graph.is_entry(v):
            t0 = self.earliest_start(v, device)
            self.start[v], self.end[v] = t0, t0 + self.cluster.exec_duration(fl, device)
            self.device_avail[device] = self.end[v]


def critical_path_assign(graph, cluster, trials: int = 50, seed: int = 0,
                         strategy: str = "fifo", features=None, return_all: bool = False):
    """List scheduling with randomised selection tie-breaks, best of ``trials``
    (reference heuristics.py:94-131): every trial is one critical-path-teacher
    episode inside the rollout kernel (largest t-level, ties broken uniformly
    at random by Philox keyed on (seed, trial, step); earliest-start device,
    first on ties), all trials run as one batch with the fused simulator, and
    the first trial with the smallest makespan wins.  The reference draws its
    tie-breaks from numpy PCG64 streams, so individual trials match it in
    distribution, not draw for draw; without ties every trial is the
    deterministic CriticalPathRule episode."""
    if trials < 1:
        raise ValueError("trials must be >= 1")
    from .params import init_policy_params
    from .policy import PolicyConfig, PolicyContext

    # the teacher's actions do not depend on the policy; a minimal policy
    # provides the tables the kernel reads
    pc = PolicyConfig(hidden=8, k_rounds=1)
    ctx = PolicyContext(graph, cluster, pc, features)
    rb = ctx.rollout_batch(init_policy_params(pc, seed=0), trials, 0.0, seed, mode="teacher",
                           simulate=True, strategy=strategy, tie_random=True)
    st = rb.status.cpu().numpy()
    if (st != 0).any():
        raise RuntimeError(f"critical-path trial failed with status {int(st[st != 0][0])}")
    mk = rb.makespan.cpu().numpy()
    assign = rb.assign.cpu().numpy()
    i = int(np.argmin(mk))  # first minimum (strict < over trials in order)
    best = Assignment(tuple(int(x) for x in assign[i]), "critical_path")
    if return_all:
        return best, float(mk[i]), assign, mk
    return best


class ForcedActions:
    """Teacher that replays a recorded (vertex, device) sequence — the
    teacher-forced parity harness of north_star (one list per episode, or a
    [B, n, 2] array for batches)."""

    def __init__(self, actions):
        self.actions = np.asarray(actions, dtype=np.int32)


class BruteForceCapError(ValueError):
    pass


def brute_force_optimal(graph, cluster, strategy: str = "fifo", cap: int = 1 << 20,
                        features=None, batch: int = 65536):
    """Exhaustive oracle (reference heuristics.py:183-212) as batched GPU
    simulations: every assignment of the non-entry vertices (entries pinned to
    device 0), argmin makespan, ties to the lexicographically smallest."""
    import itertools

    from .simulate import SimProblem

    n, d = len(graph), cluster.device_count
    if d ** n > cap:
        raise BruteForceCapError(f"{d}**{n} assignments exceed the cap of {cap}")
    import torch

    prob = SimProblem(graph, cluster, features)
    free = [v for v in range(n) if not graph.is_entry(v)]
    combos = np.array(list(itertools.product(range(d), repeat=len(free))), dtype=np.int32)
    combos = combos.reshape(-1, len(free))
    best, best_mk = None, None
    for s in range(0, len(combos), batch):
        part = combos[s:s + batch]
        a = np.zeros((len(part), n), dtype=np.int32)
        a[:, free] = part
        out = prob.simulate(torch.from_numpy(a).cuda(), strategy)
        mk = out["makespan"].cpu().numpy()
        i = int(np.argmin(mk))  # first minimum = lexicographically smallest
        if best_mk is None or mk[i] < best_mk:
            best_mk, best = float(mk[i]), tuple(int(x) for x in a[i])
    return Assignment(best, "brute_force"), best_mk
