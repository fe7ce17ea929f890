"""Golden REINFORCE / imitation gradients for per_step message passing
(reference policy.py:353-371 with mp_mode="per_step", training.py:181-216,
nn.py autodiff through one encode per step), dumped from the REFERENCE in the
build container:

    python tests/golden/make_per_step_grad_golden.py [--ref /root/reference/pkg]

Writes tests/golden/per_step_grad.json: per case the graph, cluster, policy
config, one sampled Stage-II episode (actions, makespan, advantage = -makespan
with a zero baseline, entropy weight 1e-2) with the full parameter gradient of
its loss, and one teacher-forced imitation episode with its gradient.
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


def cases():
    from flowplace import builders, graph as G, nn
    from flowplace.cluster import ClusterSpec
    from flowplace.heuristics import CriticalPathRule
    from flowplace.policy import PolicyConfig, PolicyContext, init_policy_params
    from flowplace.simulate import exec_time
    from flowplace.training import TrainConfig, _episode_seeds, _sum_tensors
    import util

    specs = [
        ("fixture6_h8_per_step", util.fixture6(), util.cluster2(),
         dict(hidden=8, k_rounds=2, mp_mode="per_step")),
        ("ffnn16_h16_per_step", builders.build_ffnn(4, 2, 8, 2, 2),
         ClusterSpec.uniform(4, rate=1e6, bandwidth=1e5),
         dict(hidden=16, k_rounds=2, mp_mode="per_step")),
        ("chainmm_h16_shared_per_step", builders.build_chainmm(16, 2),
         ClusterSpec.uniform(4, rate=1e6, bandwidth=1e5),
         dict(hidden=16, k_rounds=1, shared_encoder=True, mp_mode="per_step")),
    ]
    seeds = _episode_seeds(TrainConfig(seed=0, episodes=1), "sim_rl")
    out = []
    for tag, g, cl, pc_kw in specs:
        pc = PolicyConfig(**pc_kw)
        params = init_policy_params(pc, seed=0)
        ctx = PolicyContext(g, cl, pc)
        a, tr = ctx.rollout(params, epsilon=0.2, seed=int(seeds[0]))
        mk, _ = exec_time(g, a, cl, "fifo", seed=0, features=ctx.features)
        adv = -mk
        obj = nn.add(nn.scalar_mul(_sum_tensors(tr.logprob_tensors), adv),
                     nn.scalar_mul(_sum_tensors(tr.entropy_tensors), 1e-2))
        loss = nn.scalar_mul(obj, -1.0)
        nn.zero_grad(params)
        nn.backward(loss)
        rl = dict(epsilon=0.2, seed=int(seeds[0]), makespan=mk, advantage=adv,
                  entropy_weight=1e-2, loss=loss.item(), trace=_trace(tr),
                  grads={k: v.grad.reshape(-1).tolist() for k, v in params.items()
                         if v.grad is not None})
        teacher = CriticalPathRule(g, cl, ctx.features)
        _, tt = ctx.rollout(params, epsilon=0.0, seed=0, teacher=teacher)
        loss = nn.scalar_mul(_sum_tensors(tt.logprob_tensors), -1.0)
        nn.zero_grad(params)
        nn.backward(loss)
        im = dict(loss=loss.item(), trace=_trace(tt),
                  grads={k: v.grad.reshape(-1).tolist() for k, v in params.items()
                         if v.grad is not None})
        out.append(dict(tag=tag, graph=G.graph_to_dict(g), cluster=cl.to_dict(),
                        policy=pc.to_dict(), rl_grad=rl, imitation_grad=im))
    return dict(cases=out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    a = ap.parse_args()
    _ref_imports(Path(a.ref))
    dst = HERE / "per_step_grad.json"
    dst.write_text(json.dumps(cases()))
    print("wrote", dst, dst.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
