"""CPU: pin the numpy policy oracle (and the host-side features / params /
encoding it shares with the product) to vectors dumped from the reference
(tests/golden/policy_cases.json)."""
import hashlib

import numpy as np
import pytest

from helpers import graph_from_golden
from oracle import policy as OP
from paper_2505_23131_b200.cluster import ClusterSpec
from paper_2505_23131_b200.features import static_features
from paper_2505_23131_b200.params import init_policy_params


class PC:
    def __init__(self, d):
        self.hidden, self.k_rounds = d["hidden"], d["k_rounds"]
        self.shared_encoder, self.leaky_slope = d["shared_encoder"], d["leaky_slope"]


def _setup(case):
    g = graph_from_golden(case["graph"])
    cl = ClusterSpec.from_dict(case["cluster"])
    pc = PC(case["policy"])
    ctx = OP.Ctx(g, cl, pc.hidden, pc.k_rounds, pc.leaky_slope, pc.shared_encoder)
    return g, cl, pc, ctx


def _cases(policy_golden):
    return policy_golden["cases"]


def test_static_features_match_reference(policy_golden):
    for case in _cases(policy_golden):
        g = graph_from_golden(case["graph"])
        cl = ClusterSpec.from_dict(case["cluster"])
        f = static_features(g, cl.comm_factor)
        assert np.array_equal(f.matrix, np.asarray(case["features"]["matrix"])), case["tag"]
        assert [list(p) for p in f.b_paths] == case["features"]["b_paths"]
        assert [list(p) for p in f.t_paths] == case["features"]["t_paths"]


def test_encoding_and_init_match_reference(policy_golden):
    for case in _cases(policy_golden):
        g, cl, pc, ctx = _setup(case)
        assert np.array_equal(ctx.x, np.asarray(case["x_static"])), case["tag"]
        assert np.array_equal(ctx.edge.reshape(-1), np.asarray(case["msg_edge"]))
        params = init_policy_params(pc, seed=0)
        got = {k: hashlib.sha256(np.ascontiguousarray(v.data).tobytes()).hexdigest()
               for k, v in params.items()}
        assert got == case["param_sha"], case["tag"]


def test_oracle_gnn_matches_reference(policy_golden):
    for case in _cases(policy_golden):
        g, cl, pc, ctx = _setup(case)
        P = OP.leaves(init_policy_params(pc, seed=0), need=False)
        for head, key in (("sel", "H_sel"), ("plc", "H_plc")):
            H = OP.encode(P, ctx, head).v
            np.testing.assert_allclose(H, np.asarray(case[key]), rtol=1e-12, atol=1e-13)


def _check_trace(got, want, tol=1e-10, actions=True):
    assert len(got) == len(want)
    for s, w in zip(got, want):
        if actions:
            assert list(s["candidates"]) == w["candidates"]
            assert (s["vertex"], s["device"]) == (w["vertex"], w["device"])
        for k in ("sel_logprob", "plc_logprob", "sel_entropy", "plc_entropy"):
            assert abs(s[k] - w[k]) <= tol * max(1.0, abs(w[k])), (k, s[k], w[k])
        assert s["sel_argmax"] == w["sel_argmax"] and s["plc_argmax"] == w["plc_argmax"]


def test_oracle_teacher_greedy_and_forced_replays(policy_golden):
    for case in _cases(policy_golden):
        g, cl, pc, ctx = _setup(case)
        P = OP.leaves(init_policy_params(pc, seed=0), need=False)
        ro = OP.rollout(P, ctx, case["teacher"]["epsilon"], mode="teacher")
        _check_trace(ro["steps"], case["teacher"]["trace"])
        ro = OP.rollout(P, ctx, 0.0, mode="greedy")
        _check_trace(ro["steps"], case["greedy"]["trace"])
        for s in case["sampled"]:
            forced = [(x["vertex"], x["device"]) for x in s["trace"]]
            ro = OP.rollout(P, ctx, s["epsilon"], mode="forced", forced=forced)
            assert ro["assign"] == s["assign"]
            _check_trace(ro["steps"], s["trace"])


def test_oracle_gradients_match_reference(policy_golden):
    for case in _cases(policy_golden):
        if "rl_grad" not in case:
            continue
        g, cl, pc, ctx = _setup(case)
        params = init_policy_params(pc, seed=0)
        rg = case["rl_grad"]
        s0 = case["sampled"][0]
        forced = [(x["vertex"], x["device"]) for x in s0["trace"]]
        grads, _ = OP.rl_gradients(params, ctx, rg["epsilon"], rg["advantage"],
                                   rg["entropy_weight"], mode="forced", forced=forced)
        for k, want in rg["grads"].items():
            np.testing.assert_allclose(grads[k].reshape(-1), want, rtol=1e-9, atol=1e-12,
                                       err_msg=f"{case['tag']} {k}")
        ig = case["imitation_grad"]
        grads, _ = OP.rl_gradients(params, ctx, 0.0, 1.0, 0.0, mode="teacher")
        for k, want in ig["grads"].items():
            np.testing.assert_allclose(grads[k].reshape(-1), want, rtol=1e-9, atol=1e-12,
                                       err_msg=f"imitation {case['tag']} {k}")


def test_philox_known_answers():
    # Random123 kat_vectors for philox4x32-10
    assert OP.philox4x32_10((0, 0, 0, 0), (0, 0)) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C,
                                                      0x9B00DBD8]
    assert OP.philox4x32_10((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2) == [
        0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]


def test_oracle_per_step_matches_reference_golden():
    """per_step message passing (reference policy.py:353-371): the oracle's
    forced replays of the reference's teacher / greedy / sampled episodes give
    the recorded log-probs and entropies (1e-10)."""
    import json
    from conftest import GOLDEN
    from helpers import graph_from_golden
    from oracle import policy as OP
    from paper_2505_23131_b200.cluster import ClusterSpec
    from paper_2505_23131_b200.params import init_policy_params
    from paper_2505_23131_b200.policy import PolicyConfig

    doc = json.loads((GOLDEN / "policy_per_step.json").read_text())
    for case in doc["cases"]:
        g = graph_from_golden(case["graph"])
        cl = ClusterSpec.from_dict(case["cluster"])
        pc = PolicyConfig.from_dict(case["policy"])
        assert pc.mp_mode == "per_step"
        ctx = OP.Ctx(g, cl, pc.hidden, pc.k_rounds, pc.leaky_slope, pc.shared_encoder)
        P = OP.leaves(init_policy_params(pc, seed=0), need=False)
        assert case["teacher"]["encode_invocations"] == 2 * len(g)
        runs = [case["teacher"], case["greedy"]] + case["sampled"]
        for run in runs:
            want = run["trace"]
            ro = OP.rollout(P, ctx, run["epsilon"], mode="forced",
                            forced=[(w["vertex"], w["device"]) for w in want], per_step=True)
            for s, w in zip(ro["steps"], want):
                assert list(s["candidates"]) == w["candidates"]
                for k in ("sel_logprob", "plc_logprob", "sel_entropy", "plc_entropy"):
                    assert abs(s[k] - w[k]) <= 1e-10 * max(1.0, abs(w[k])), (case["tag"], k)
        # the teacher episode itself: CriticalPathRule actions from the oracle
        ro = OP.rollout(P, ctx, 0.2, mode="teacher", per_step=True)
        assert [(s["vertex"], s["device"]) for s in ro["steps"]] == \
            [(w["vertex"], w["device"]) for w in case["teacher"]["trace"]]
