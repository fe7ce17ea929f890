"""CPU: host-side drop-in pieces against reference-written goldens
(tests/golden/r2_cases.json, policy_cases.json): checkpoint JSON interop both
ways, and the host CriticalPathRule.place / PlacementTimeline replaying the
reference's teacher episodes."""
import json

import numpy as np

from helpers import graph_from_golden
from paper_2505_23131_b200.cluster import ClusterSpec
from paper_2505_23131_b200.heuristics import CriticalPathRule, PlacementTimeline
from paper_2505_23131_b200.params import init_policy_params, load_params
from paper_2505_23131_b200.policy import PolicyConfig
from paper_2505_23131_b200.training import TrainConfig, load_checkpoint, save_checkpoint

GOLDEN = __import__("pathlib").Path(__file__).resolve().parent / "golden"


def test_checkpoint_interop_with_reference_files(tmp_path):
    """A checkpoint the reference wrote (nn.py:283-309, training.py:309-326)
    loads here; saving the same params + configs reproduces both files byte
    for byte."""
    ck = json.loads((GOLDEN / "r2_cases.json").read_text())["checkpoint"]
    ref = tmp_path / "ref.json"
    ref.write_text(ck["params_json"])
    (tmp_path / "ref.json.sidecar.json").write_text(ck["sidecar_json"])
    params, pc, sidecar = load_checkpoint(ref)
    assert pc == PolicyConfig(hidden=8, k_rounds=1)
    want = init_policy_params(pc, seed=3)
    assert set(params) == set(want)
    for k in want:
        assert np.array_equal(params[k].data, want[k].data), k
    out = tmp_path / "ours.json"
    save_checkpoint(out, params, pc, TrainConfig.from_dict(sidecar["train"]),
                    norm_stats=sidecar["feature_norm"])
    assert out.read_text() == ck["params_json"]
    assert (tmp_path / "ours.json.sidecar.json").read_text() == ck["sidecar_json"]
    # and a file we write loads as the same tensors
    again = load_params(out)
    for k in want:
        assert np.array_equal(again[k].data, want[k].data), k


def test_host_critical_path_rule_replays_reference_teacher(policy_golden):
    """CriticalPathRule.select / place over the host PlacementTimeline
    reproduce the reference teacher's (vertex, device) sequence."""
    for case in policy_golden["cases"]:
        g = graph_from_golden(case["graph"])
        cl = ClusterSpec.from_dict(case["cluster"])
        from paper_2505_23131_b200.features import static_features
        rule = CriticalPathRule(g, cl, static_features(g, cl.comm_factor))
        tl = PlacementTimeline(g, cl)
        left = [len(g.preds(v)) for v in range(len(g))]
        cands = sorted(g.entry_vertices())
        got = []
        for _ in range(len(g)):
            v = rule.select(cands)
            d = rule.place(v, tl)
            tl.commit(v, d)
            got.append((v, d))
            cands.remove(v)
            for w in g.succs(v):
                left[w] -= 1
                if left[w] == 0:
                    cands.append(w)
            cands.sort()
        want = [(s["vertex"], s["device"]) for s in case["teacher"]["trace"]]
        assert got == want, case["tag"]


class _DuckTeacher:
    """Any object with the reference teacher interface (select / place)."""

    def __init__(self, rule):
        self.rule = rule

    def select(self, candidates):
        return self.rule.select(candidates)

    def place(self, v, timeline):
        return self.rule.place(v, timeline)


def test_duck_teacher_actions_replay_reference_teacher(policy_golden):
    """policy.teacher_actions steps an arbitrary select / place teacher the
    way the reference rollout does (policy.py:353-389): wrapping the rule
    reproduces the reference teacher's (vertex, device) sequence."""
    import pytest

    from paper_2505_23131_b200.features import static_features
    from paper_2505_23131_b200.policy import TeacherActionError, teacher_actions
    for case in policy_golden["cases"]:
        g = graph_from_golden(case["graph"])
        cl = ClusterSpec.from_dict(case["cluster"])
        duck = _DuckTeacher(CriticalPathRule(g, cl, static_features(g, cl.comm_factor)))
        acts = teacher_actions(g, cl, duck, episodes=2)
        want = [(s["vertex"], s["device"]) for s in case["teacher"]["trace"]]
        assert acts.shape == (2, len(g), 2)
        for e in range(2):
            assert [tuple(map(int, a)) for a in acts[e]] == want, case["tag"]

    class Bad:
        def select(self, candidates):
            return max(candidates) + 1

        def place(self, v, timeline):
            return 0

    with pytest.raises(TeacherActionError):
        teacher_actions(g, cl, Bad())
