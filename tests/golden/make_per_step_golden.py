"""Golden vectors for per_step message passing (reference policy.py:353-371,
mp_mode="per_step": both encoders re-run before every decision with the
dynamic columns dyn[v] = (1, (d+1)/D) of the vertices placed so far), dumped
from the REFERENCE in the build container:

    python tests/golden/make_per_step_golden.py [--ref /root/reference/pkg]

Writes tests/golden/policy_per_step.json: per case the graph, cluster, policy
config, and the traces of a teacher-forced, a greedy and two sampled
episodes (sampled actions are FORCED on the GPU; log-probs / entropies must
agree) plus the encoder invocation count (2n per episode).
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

from make_golden import _ref_imports  # noqa: E402
from policy_golden import _trace  # noqa: E402


def per_step_cases():
    from flowplace import builders, graph as G
    from flowplace.cluster import ClusterSpec
    from flowplace.heuristics import CriticalPathRule
    from flowplace.policy import PolicyConfig, PolicyContext, init_policy_params
    from flowplace.training import TrainConfig, _episode_seeds
    import util

    specs = [
        ("fixture6_h8_per_step", util.fixture6(), util.cluster2(),
         dict(hidden=8, k_rounds=2, mp_mode="per_step")),
        ("ffnn64_h32_per_step", builders.build_ffnn(8, 4, 16, 4, 2),
         ClusterSpec.uniform(8, rate=1e6, bandwidth=1e5),
         dict(hidden=32, k_rounds=2, mp_mode="per_step")),
        ("chainmm60_h16_shared_per_step", builders.build_chainmm(64, 2),
         ClusterSpec.uniform(4, rate=1e6, bandwidth=1e5),
         dict(hidden=16, k_rounds=1, shared_encoder=True, mp_mode="per_step")),
    ]
    seeds = _episode_seeds(TrainConfig(seed=0, episodes=2), "sim_rl")
    cases = []
    for tag, g, cl, pc_kw in specs:
        pc = PolicyConfig(**pc_kw)
        params = init_policy_params(pc, seed=0)
        ctx = PolicyContext(g, cl, pc)
        teacher = CriticalPathRule(g, cl, ctx.features)
        _, t_teacher = ctx.rollout(params, epsilon=0.2, seed=0, teacher=teacher)
        _, t_greedy = ctx.rollout(params, epsilon=0.0, seed=0, greedy=True)
        sampled = []
        for eps, sd in ((0.2, seeds[0]), (1.0, seeds[1])):
            a, tr = ctx.rollout(params, epsilon=eps, seed=sd)
            sampled.append(dict(epsilon=eps, seed=int(sd), assign=list(a), trace=_trace(tr),
                                encode_invocations=tr.encode_invocations))
        cases.append(dict(tag=tag, graph=G.graph_to_dict(g), cluster=cl.to_dict(),
                          policy=pc.to_dict(),
                          teacher=dict(epsilon=0.2, trace=_trace(t_teacher),
                                       encode_invocations=t_teacher.encode_invocations),
                          greedy=dict(epsilon=0.0, trace=_trace(t_greedy)),
                          sampled=sampled))
    return dict(cases=cases)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    a = ap.parse_args()
    _ref_imports(Path(a.ref))
    out = HERE / "policy_per_step.json"
    out.write_text(json.dumps(per_step_cases()))
    print("wrote", out, out.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
