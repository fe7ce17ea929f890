"""Policy golden vectors from the REFERENCE (imported by make_golden.py in the
build container; needs /root/reference).  Output: tests/golden/policy_cases.json.

Per case: graph + cluster + policy config, the reference's static features
(matrix, b/t paths), x_static / edge encoding, GNN outputs H_sel / H_plc,
params hashes (init parity), and traces of teacher-forced, greedy and sampled
episodes (the sampled actions are later FORCED on the GPU/oracle and the
recorded log-probs / entropies must agree), plus full parameter gradients of
one REINFORCE episode and one imitation episode (training.py:144, 200-216).
"""

from __future__ import annotations

import hashlib

import numpy as np


def _trace(tr):
    return [dict(candidates=list(s.candidates), vertex=s.vertex, device=s.device,
                 sel_logprob=s.sel_logprob, plc_logprob=s.plc_logprob,
                 sel_entropy=s.sel_entropy, plc_entropy=s.plc_entropy,
                 sel_argmax=s.sel_argmax, plc_argmax=s.plc_argmax) for s in tr.steps]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def policy_cases():
    from flowplace import builders, graph as G, nn
    from flowplace.cluster import ClusterSpec
    from flowplace.heuristics import CriticalPathRule
    from flowplace.policy import PolicyConfig, PolicyContext, gnn_encode, init_policy_params
    from flowplace.simulate import exec_time
    from flowplace.training import TrainConfig, _episode_seeds, _sum_tensors
    import util

    specs = [
        ("fixture6_h8", util.fixture6(), util.cluster2(), dict(hidden=8, k_rounds=2), True),
        ("ffnn64_h32", builders.build_ffnn(8, 4, 16, 4, 2),
         ClusterSpec.uniform(8, rate=1e6, bandwidth=1e5), dict(hidden=32, k_rounds=2), True),
        ("chainmm60_h16_shared", builders.build_chainmm(64, 2),
         ClusterSpec.uniform(4, rate=1e6, bandwidth=1e5),
         dict(hidden=16, k_rounds=1, shared_encoder=True), True),
    ]
    try:  # Llama-block from the new builder (built by OUR package, fed to the reference)
        import sys
        from pathlib import Path
        sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
        from paper_2505_23131_b200 import builders as ours
        from paper_2505_23131_b200.graph import graph_to_dict
        lb = G.graph_from_dict(graph_to_dict(ours.build_llama_block()))
        specs.append(("llama_block_h32", lb, ClusterSpec.uniform(8, rate=1e9, bandwidth=1e7),
                      dict(hidden=32, k_rounds=2), False))
    except ImportError:
        pass

    seeds = _episode_seeds(TrainConfig(seed=0, episodes=4), "sim_rl")
    cases = []
    for tag, g, cl, pc_kw, grads in specs:
        pc = PolicyConfig(**pc_kw)
        params = init_policy_params(pc, seed=0)
        ctx = PolicyContext(g, cl, pc)
        dyn = np.zeros((len(g), 2))
        Hs = gnn_encode(params, pc, ctx.enc, "sel", dyn).data
        Hp = gnn_encode(params, pc, ctx.enc, "plc", dyn).data
        teacher = CriticalPathRule(g, cl, ctx.features)
        _, t_teacher = ctx.rollout(params, epsilon=0.2, seed=0, teacher=teacher)
        _, t_greedy = ctx.rollout(params, epsilon=0.0, seed=0, greedy=True)
        sampled = []
        for eps, sd in ((0.2, seeds[0]), (0.2, seeds[1]), (1.0, seeds[2]), (0.0, seeds[3])):
            a, tr = ctx.rollout(params, epsilon=eps, seed=sd)
            mk, _ = exec_time(g, a, cl, "fifo", seed=0, features=ctx.features)
            sampled.append(dict(epsilon=eps, seed=int(sd), makespan=mk, assign=list(a),
                                trace=_trace(tr)))
        case = dict(
            tag=tag, graph=G.graph_to_dict(g), cluster=cl.to_dict(), policy=pc.to_dict(),
            features=dict(matrix=ctx.features.matrix.tolist(),
                          b_paths=[list(p) for p in ctx.features.b_paths],
                          t_paths=[list(p) for p in ctx.features.t_paths]),
            x_static=ctx.enc.x_static.tolist(), msg_edge=ctx.enc.msg_edge.reshape(-1).tolist(),
            H_sel=Hs.tolist(), H_plc=Hp.tolist(),
            param_sha={k: _sha(v.data) for k, v in params.items()},
            teacher=dict(epsilon=0.2, trace=_trace(t_teacher)),
            greedy=dict(epsilon=0.0, trace=_trace(t_greedy)),
            sampled=sampled,
        )
        if grads:
            # one Stage-II episode (training.py:193-208): baseline 0 -> adv = -mk
            s0 = sampled[0]
            a, tr = ctx.rollout(params, epsilon=0.2, seed=s0["seed"])
            adv = -s0["makespan"]
            obj = nn.add(nn.scalar_mul(_sum_tensors(tr.logprob_tensors), adv),
                         nn.scalar_mul(_sum_tensors(tr.entropy_tensors), 1e-2))
            loss = nn.scalar_mul(obj, -1.0)
            nn.zero_grad(params)
            nn.backward(loss)
            case["rl_grad"] = dict(epsilon=0.2, seed=s0["seed"], advantage=adv,
                                   entropy_weight=1e-2, loss=loss.item(),
                                   grads={k: v.grad.reshape(-1).tolist()
                                          for k, v in params.items() if v.grad is not None})
            # one imitation episode (training.py:142-147)
            _, tr = ctx.rollout(params, epsilon=0.0, seed=0, teacher=teacher)
            loss = nn.scalar_mul(_sum_tensors(tr.logprob_tensors), -1.0)
            nn.zero_grad(params)
            nn.backward(loss)
            case["imitation_grad"] = dict(loss=loss.item(),
                                          grads={k: v.grad.reshape(-1).tolist()
                                                 for k, v in params.items()
                                                 if v.grad is not None})
        cases.append(case)
    return dict(cases=cases, episode_seeds=[int(s) for s in seeds])
