"""Round-2 golden vectors from the REFERENCE (run in the build container, where
/root/reference exists; outputs committed, the GPU box never needs the
reference).  Pins parity at the BASELINE configs' own scale:

* ``scale_ffnn1024.npz`` -- config 2: 1024 reference episodes of the
  FFNN-64 / 8-device / h32 policy (epsilon 0.2 / 0 / 1 sampled, greedy and
  critical-path-teacher episodes mixed), with every step's (vertex, device),
  log-probs, entropies, argmaxes and the episode makespan.  The GPU replays
  all 1024 as ONE forced launch.
* ``r2_cases.json``:
  - ``llama_layer_grad`` -- config 4: the Llama-layer (248-op) Stage-II
    REINFORCE gradient of one reference episode (training.py:193-208);
  - ``executor`` -- Stage-III ``SimulatorExecutor`` (training.py:81-102)
    makespans over its per-call seed stream (jitter 0.1) for fixed
    assignments;
  - ``checkpoint`` -- a reference-written ``save_checkpoint`` file + sidecar
    (nn.py:283-309, training.py:309-326);
  - ``imitation`` -- ``imitation_stage`` curve (per-episode loss, makespan)
    and final params of a short run (training.py:129-155);
  - ``teacher_agreement`` -- ``measure_teacher_agreement`` (training.py:162-178).

    python tests/golden/make_r2_golden.py [--ref /root/reference/pkg]
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
N_SCALE = 1024


def _setup(ref: str):
    sys.path.insert(0, str(Path(ref) / "src"))
    sys.path.insert(0, str(ROOT))
    os.environ["FLOWPLACE_SIM_BACKEND"] = "python"


def _ffnn():
    from flowplace import builders
    from flowplace.cluster import ClusterSpec
    return builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, rate=1e6, bandwidth=1e5)


def _episode_plan(i: int):
    """Episode i of the 1024: (kind, epsilon, seed)."""
    if i % 64 == 5:
        return "teacher", 0.2, i
    if i % 64 == 9:
        return "greedy", 0.0, i
    eps = (0.2, 0.2, 0.2, 0.0, 1.0)[i % 5]
    return "sample", eps, 10_000 + i


def _scale_worker(args):
    ref, lo, hi = args
    _setup(ref)
    from flowplace.heuristics import CriticalPathRule
    from flowplace.policy import PolicyConfig, PolicyContext, init_policy_params
    from flowplace.simulate import exec_time
    g, cl = _ffnn()
    pc = PolicyConfig(hidden=32, k_rounds=2)
    params = init_policy_params(pc, seed=0)
    ctx = PolicyContext(g, cl, pc)
    teacher = CriticalPathRule(g, cl, ctx.features)
    n = len(g)
    out = []
    for i in range(lo, hi):
        kind, eps, seed = _episode_plan(i)
        a, tr = ctx.rollout(params, epsilon=eps, seed=seed, greedy=kind == "greedy",
                            teacher=teacher if kind == "teacher" else None)
        mk, _ = exec_time(g, a, cl, "fifo", seed=0, features=ctx.features)
        rec = np.zeros((n, 8))
        for t, s in enumerate(tr.steps):
            rec[t] = (s.vertex, s.device, s.sel_logprob, s.plc_logprob, s.sel_entropy,
                      s.plc_entropy, s.sel_argmax, s.plc_argmax)
        out.append((i, eps, mk, rec))
    return out


def scale_ffnn(ref: str):
    with mp.get_context("spawn").Pool(os.cpu_count()) as pool:
        chunks = [(ref, k, min(N_SCALE, k + 32)) for k in range(0, N_SCALE, 32)]
        res = [r for part in pool.map(_scale_worker, chunks) for r in part]
    res.sort(key=lambda r: r[0])
    rec = np.stack([r[3] for r in res])
    kinds = np.array([("sample", "greedy", "teacher").index(_episode_plan(i)[0])
                      for i in range(N_SCALE)], dtype=np.int8)
    np.savez_compressed(
        HERE / "scale_ffnn1024.npz",
        vd=rec[..., :2].astype(np.uint8), lp=rec[..., 2:4], ent=rec[..., 4:6],
        argmax=rec[..., 6:8].astype(np.uint8), makespan=np.array([r[2] for r in res]),
        epsilon=np.array([r[1] for r in res]), kind=kinds)
    print(f"scale_ffnn1024.npz: {N_SCALE} episodes")


def r2_cases():
    from flowplace import graph as G, nn
    from flowplace.cluster import ClusterSpec
    from flowplace.heuristics import CriticalPathRule
    from flowplace.policy import PolicyConfig, PolicyContext, init_policy_params
    from flowplace.simulate import exec_time
    from flowplace.training import (SimulatorExecutor, TrainConfig, _episode_seeds,
                                    _sum_tensors, imitation_stage, measure_teacher_agreement,
                                    save_checkpoint)
    from paper_2505_23131_b200 import builders as ours
    from paper_2505_23131_b200.graph import graph_to_dict

    doc = {}
    # ---- config 4: Llama-layer REINFORCE gradient ----
    g = G.graph_from_dict(graph_to_dict(ours.build_llama_layer()))
    cl = ClusterSpec.uniform(8, rate=1e9, bandwidth=1e7)
    pc = PolicyConfig(hidden=32, k_rounds=2)
    params = init_policy_params(pc, seed=0)
    ctx = PolicyContext(g, cl, pc)
    seed = _episode_seeds(TrainConfig(seed=0, episodes=1), "sim_rl")[0]
    a, tr = ctx.rollout(params, epsilon=0.2, seed=seed)
    mk, _ = exec_time(g, a, cl, "fifo", seed=0, features=ctx.features)
    adv = -mk
    obj = nn.add(nn.scalar_mul(_sum_tensors(tr.logprob_tensors), adv),
                 nn.scalar_mul(_sum_tensors(tr.entropy_tensors), 1e-2))
    loss = nn.scalar_mul(obj, -1.0)
    nn.zero_grad(params)
    nn.backward(loss)
    doc["llama_layer_grad"] = dict(
        graph=G.graph_to_dict(g), cluster=cl.to_dict(), policy=pc.to_dict(), epsilon=0.2,
        makespan=mk, advantage=adv, entropy_weight=1e-2, loss=loss.item(),
        actions=[[s.vertex, s.device] for s in tr.steps],
        lp=[[s.sel_logprob, s.plc_logprob] for s in tr.steps],
        ent=[[s.sel_entropy, s.plc_entropy] for s in tr.steps],
        grads={k: v.grad.reshape(-1).tolist() for k, v in params.items() if v.grad is not None})

    # ---- Stage-III executor seed stream ----
    gf, cf = _ffnn()
    rng = np.random.default_rng(11)
    assigns = [[int(x) for x in rng.integers(0, 8, size=len(gf))] for _ in range(24)]
    ex = SimulatorExecutor(cf, "fifo", jitter_sigma=0.1, base_seed=123)
    doc["executor"] = dict(graph=G.graph_to_dict(gf), cluster=cf.to_dict(), strategy="fifo",
                           jitter_sigma=0.1, base_seed=123, assign=assigns,
                           makespan=[float(ex(gf, a)) for a in assigns])

    # ---- checkpoint written by the reference ----
    pc8 = PolicyConfig(hidden=8, k_rounds=1)
    p8 = init_policy_params(pc8, seed=3)
    with tempfile.TemporaryDirectory() as td:
        path = Path(td) / "ck.json"
        save_checkpoint(path, p8, pc8, TrainConfig(episodes=7, seed=5),
                        norm_stats={"mean": [1.0, 2.0]})
        doc["checkpoint"] = dict(params_json=path.read_text(),
                                 sidecar_json=Path(str(path) + ".sidecar.json").read_text())

    # ---- imitation stage (B = 1 semantics) + teacher agreement ----
    pci = PolicyConfig(hidden=32, k_rounds=2)
    pi = init_policy_params(pci, seed=0)
    ctxi = PolicyContext(gf, cf, pci)
    teacher = CriticalPathRule(gf, cf, ctxi.features)
    agree0 = measure_teacher_agreement(ctxi, pi, teacher, rollouts=3, seed=0)
    res = imitation_stage(gf, cf, TrainConfig(episodes=3, lr0=1e-2, lr1=1e-3), pci, pi,
                          context=ctxi)
    agree1 = measure_teacher_agreement(ctxi, res.params, teacher, rollouts=3, seed=0)
    doc["imitation"] = dict(
        graph=G.graph_to_dict(gf), cluster=cf.to_dict(), policy=pci.to_dict(),
        train=dict(episodes=3, lr0=1e-2, lr1=1e-3), curve=res.curve,
        final_loss=res.final_loss, agreement_before=agree0, agreement_after=agree1,
        final_params={k: v.data.reshape(-1).tolist() for k, v in res.params.items()})
    return doc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    ap.add_argument("--only", default="scale,cases")
    args = ap.parse_args()
    only = set(args.only.split(","))
    _setup(args.ref)
    if "scale" in only:
        scale_ffnn(args.ref)
    if "cases" in only:
        doc = r2_cases()
        (HERE / "r2_cases.json").write_text(json.dumps(doc) + "\n")
        print("r2_cases.json:", sorted(doc))


if __name__ == "__main__":
    main()
