"""Dump golden vectors from the REFERENCE implementation (run in the build
container, where /root/reference exists; the outputs are committed so the
GPU box never needs the reference).

    python tests/golden/make_golden.py [--ref /root/reference/pkg]

Writes tests/golden/sim_cases.json (simulator event streams) and
tests/golden/policy_cases.json (policy encodings, traces, gradients).
The reference's pure-Python simulator backend is used (bit-identical to its
Cython core by the reference's own tests/test_backends.py).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def _ref_imports(ref: Path):
    sys.path.insert(0, str(ref / "src"))
    sys.path.insert(0, str(ref / "tests"))
    os.environ["FLOWPLACE_SIM_BACKEND"] = "python"
    import flowplace  # noqa: F401
    return ref


def sim_cases():
    from flowplace import builders, graph as G
    from flowplace.cluster import ClusterSpec
    from flowplace.features import static_features
    from flowplace.simulate import exec_time
    from flowplace._simpy import DeadlockError
    import util

    cases = []

    def add(tag, g, cl, assign, strategy="fifo", seed=0):
        feats = static_features(g, cl.comm_factor)
        try:
            mk, sched = exec_time(g, assign, cl, strategy, seed, feats)
            ev = [[0 if e.task.kind == "exec" else 1, e.task.vertex,
                   e.task.device if e.task.kind == "exec" else e.task.src,
                   -1 if e.task.kind == "exec" else e.task.dst, e.time_ms,
                   0 if e.type == "beg" else 1] for e in sched.events]
            res = {"makespan": mk, "events": ev}
        except DeadlockError as exc:
            res = {"deadlock": {"time": exc.time_ms, "blocked": exc.blocked}}
        cases.append({"tag": tag, "graph": G.graph_to_dict(g), "cluster": cl.to_dict(),
                      "assign": [int(x) for x in assign], "strategy": strategy,
                      "seed": seed, **res})

    strategies = ("fifo", "depth_first", "breadth_first")
    # tests/test_backends.py:53-62 pattern, plus slot / device-count variations
    rng = np.random.default_rng(2)
    for dev, es, ts in ((2, 1, 1), (2, 2, 1), (3, 1, 2), (4, 2, 2)):
        cl = ClusterSpec.uniform(dev, rate=100.0, bandwidth=64.0, exec_slots=es,
                                 transfer_slots=ts)
        for k in range(12):
            g = util.random_dag(rng)
            assign = [int(x) for x in rng.integers(0, dev, size=len(g))]
            for s in strategies:
                add(f"random_dag[{dev},{es},{ts}]#{k}", g, cl, assign, s)
    # jitter (tests/test_backends.py:65-73)
    clj = util.cluster2(rate=100.0, bandwidth=64.0, jitter_sigma=0.2)
    for seed in range(10):
        add("fixture6_jitter", util.fixture6(), clj, [0, 0, 1, 0, 1, 0], "fifo", seed)
    # fig2_unit locality / alternating (tests/test_simulator.py:254-276)
    g = util.fig2_unit()
    cl = ClusterSpec.uniform(2, rate=1.0, bandwidth=4.0)
    alt = [0] * len(g)
    for i, v in enumerate(range(8, 16)):
        alt[v] = i % 2
    for i, v in enumerate(range(16, 20)):
        alt[v] = i % 2
    loc = [0] * len(g)
    for b in range(4):
        loc[8 + 2 * b] = loc[8 + 2 * b + 1] = loc[16 + b] = b % 2
    for s in strategies:
        add("fig2_alt", g, cl, alt, s)
        add("fig2_loc", g, cl, loc, s)
    # arithmetic pins (tests/test_simulator.py:26-57)
    add("chain30", util.chain_graph((1000, 2000)), util.cluster2(rate=100.0), [0, 0, 0])
    add("chain30.5", util.chain_graph((1000, 2000), bytes_=100),
        util.cluster2(rate=100.0, bandwidth=800.0), [0, 0, 1])
    # deadlock (tests/test_simulator.py:220-227)
    cyc = G.DataflowGraph((G.Vertex(0, G.OpKind.OTHER, 10, 8, ""),
                           G.Vertex(1, G.OpKind.OTHER, 10, 8, "")), ((0, 1), (1, 0)))
    cases.append({"tag": "deadlock_cycle", "graph": G.graph_to_dict(cyc),
                  "cluster": util.cluster2().to_dict(), "assign": [0, 0], "strategy": "fifo",
                  "seed": 0, "deadlock": {"time": 0.0, "blocked": [0, 1]}})
    # bench-config graphs
    rng = np.random.default_rng(7)
    c4 = ClusterSpec.uniform(4, rate=1e6, bandwidth=1e5, comm_factor=4)
    c8 = ClusterSpec.uniform(8, rate=1e6, bandwidth=1e5, comm_factor=4)
    for tag, g, cl in (("chainmm60", builders.build_chainmm(64, 2), c4),
                       ("ffnn64", builders.build_ffnn(8, 4, 16, 4, 2), c8)):
        for k in range(3):
            assign = [int(x) for x in rng.integers(0, cl.device_count, size=len(g))]
            for s in strategies:
                add(f"{tag}#{k}", g, cl, assign, s)
    return cases


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    ap.add_argument("--only", default="sim,policy")
    args = ap.parse_args()
    _ref_imports(Path(args.ref))
    only = set(args.only.split(","))
    if "sim" in only:
        cases = sim_cases()
        (HERE / "sim_cases.json").write_text(json.dumps({"cases": cases}) + "\n")
        print(f"sim_cases.json: {len(cases)} cases")
    if "policy" in only:
        from policy_golden import policy_cases  # noqa: E402  (sibling module)
        doc = policy_cases()
        (HERE / "policy_cases.json").write_text(json.dumps(doc) + "\n")
        print(f"policy_cases.json: {len(doc['cases'])} cases")


if __name__ == "__main__":
    sys.path.insert(0, str(HERE))
    main()
