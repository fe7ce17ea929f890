"""GPU: per_step message passing (reference policy.py:353-371) — a B x n-row
batched encode before every decision.  Pinned to the reference's own per_step
traces (tests/golden/policy_per_step.json: teacher actions exact, forced
replays' log-probs / entropies within 1e-9, 2n encoder invocations per
episode) and to the numpy oracle under the same Philox draws."""
import json

import numpy as np
import pytest

from conftest import GOLDEN
from helpers import graph_from_golden
from oracle import policy as OP
from oracle import sim as osim
from paper_2505_23131_b200 import builders
from paper_2505_23131_b200.cluster import ClusterSpec
from paper_2505_23131_b200.heuristics import CriticalPathRule, ForcedActions
from paper_2505_23131_b200.params import init_policy_params
from paper_2505_23131_b200.policy import PolicyConfig, PolicyContext

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _close(a, b, tol=TOL):
    return abs(a - b) <= tol * max(1.0, abs(b))


def _check(trace, want, actions=True):
    assert len(trace.steps) == len(want)
    for s, w in zip(trace.steps, want):
        if actions:
            assert list(s.candidates) == w["candidates"]
            assert (s.vertex, s.device) == (w["vertex"], w["device"])
        for k in ("sel_logprob", "plc_logprob", "sel_entropy", "plc_entropy"):
            assert _close(getattr(s, k), w[k]), (k, getattr(s, k), w[k])


def test_per_step_matches_reference_golden():
    doc = json.loads((GOLDEN / "policy_per_step.json").read_text())
    for case in doc["cases"]:
        g = graph_from_golden(case["graph"])
        cl = ClusterSpec.from_dict(case["cluster"])
        pc = PolicyConfig.from_dict(case["policy"])
        ctx = PolicyContext(g, cl, pc)
        params = init_policy_params(pc, seed=0)
        a, tr = ctx.rollout(params, case["teacher"]["epsilon"], 0,
                            teacher=CriticalPathRule(g, cl, ctx.features))
        _check(tr, case["teacher"]["trace"])
        assert tr.encode_invocations == case["teacher"]["encode_invocations"] == 2 * len(g)
        for run in [case["greedy"]] + case["sampled"]:
            acts = [(x["vertex"], x["device"]) for x in run["trace"]]
            a, tr = ctx.rollout(params, run["epsilon"], 0, teacher=ForcedActions(acts))
            _check(tr, run["trace"])
            if "assign" in run:
                assert list(a) == run["assign"]


@pytest.mark.parametrize("which", ["ffnn", "chainmm_shared"])
def test_per_step_sampled_batch_matches_oracle_draws(which):
    if which == "ffnn":
        g, cl = builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, 1e6, 1e5)
        pc = PolicyConfig(mp_mode="per_step")
    else:
        g, cl = builders.build_chainmm(64, 2), ClusterSpec.uniform(4, 1e6, 1e5)
        pc = PolicyConfig(hidden=16, k_rounds=1, shared_encoder=True, mp_mode="per_step")
    params = init_policy_params(pc, seed=2)
    ctx = PolicyContext(g, cl, pc)
    B, seed = 32, 77
    rb = ctx.rollout_batch(params, B, 0.2, seed, trace_steps=True)
    st = rb.status.cpu().numpy()
    assert (st == 0).all()
    vd, lp = rb.step_vd.cpu().numpy(), rb.step_lp.cpu().numpy()
    ent, mk = rb.step_ent.cpu().numpy(), rb.makespan.cpu().numpy()
    assign = rb.assign.cpu().numpy()
    octx = OP.Ctx(g, cl, pc.hidden, pc.k_rounds, pc.leaky_slope, pc.shared_encoder, ctx.features)
    P = OP.leaves(params, need=False)
    for b in (0, 5, 31):
        ro = OP.rollout(P, octx, 0.2, mode="uniform", seed=seed, episode=b, per_step=True)
        assert [(int(x), int(y)) for x, y in vd[b]] == \
            [(s["vertex"], s["device"]) for s in ro["steps"]], (which, b)
        for t, s in enumerate(ro["steps"]):
            assert _close(lp[b, t, 0], s["sel_logprob"]) and _close(lp[b, t, 1], s["plc_logprob"])
            assert _close(ent[b, t, 0], s["sel_entropy"]) and _close(ent[b, t, 1], s["plc_entropy"])
        assert list(assign[b]) == ro["assign"]
        omk, _ = osim.exec_time(g, assign[b], cl)
        assert mk[b] == omk


def test_per_step_bad_action_and_failed_episodes_skip_gradient():
    g, cl = builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, 1e6, 1e5)
    pc = PolicyConfig(mp_mode="per_step")
    ctx = PolicyContext(g, cl, pc)
    params = init_policy_params(pc, seed=0)
    ref = ctx.rollout_batch(params, 2, 0.0, 0, mode="teacher", trace_steps=True)
    acts = ref.step_vd.cpu().numpy().copy()
    acts[0, 10, 1] = 99
    acts[1, 20, 0] = 10 ** 6
    rb = ctx.rollout_batch(params, 2, 0.0, 0, mode="forced", forced=acts)
    assert rb.status.cpu().numpy().tolist() == [3, 3]
    # per_step REINFORCE rollouts are supported; failed episodes contribute nothing
    rb = ctx.rollout_batch(params, 2, 0.0, 0, mode="forced", forced=acts, grad=True)
    assert rb.status.cpu().numpy().tolist() == [3, 3]
    grad = ctx.policy_gradient(rb, [1.0, 1.0], 0.0)
    assert float(grad.abs().max()) == 0.0
