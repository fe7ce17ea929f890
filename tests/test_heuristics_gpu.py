"""GPU: critical_path_assign (reference heuristics.py:94-131) — best of
randomised-tie critical-path trials, run as one teacher-mode batch with the
fused simulator.  The reference's PCG64 tie-break stream is not reproduced,
so each trial is pinned by the rule itself (largest t-level, then the first
earliest-start device on the oracle timeline) and the winner by bit-exact
oracle makespans."""
import numpy as np
import pytest

from oracle import policy as OP
from oracle import sim as osim
from paper_2505_23131_b200 import builders
from paper_2505_23131_b200.cluster import ClusterSpec
from paper_2505_23131_b200.heuristics import critical_path_assign
from paper_2505_23131_b200.params import init_policy_params
from paper_2505_23131_b200.policy import PolicyConfig, PolicyContext, _candidate_sets

pytestmark = pytest.mark.gpu


def _check_cp_trial(g, cl, tlev, order_devs):
    order = [v for v, _ in order_devs]
    cands = _candidate_sets(g, order)
    tl = OP.Timeline(g, cl)
    for t, (v, d) in enumerate(order_devs):
        best = max(tlev[u] for u in cands[t])
        assert tlev[v] == best, (t, v)
        starts = [tl.earliest(v, dd) for dd in range(cl.device_count)]
        assert d == int(np.argmin(starts)), (t, v, d, starts)
        tl.commit(v, d)


@pytest.mark.parametrize("wide", [False, True])
def test_tie_random_trials_follow_the_rule(wide):
    g, cl = builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, 1e6, 1e5)
    pc = PolicyConfig(hidden=8, k_rounds=1)
    ctx = PolicyContext(g, cl, pc)
    tlev = ctx.features.t_level
    B = 24
    rb = ctx.rollout_batch(init_policy_params(pc, 0), B, 0.0, 5, mode="teacher",
                           trace_steps=True, tie_random=True, wide=wide)
    assert (rb.status.cpu().numpy() == 0).all()
    vd = rb.step_vd.cpu().numpy()
    for b in range(B):
        _check_cp_trial(g, cl, tlev, [(int(x), int(y)) for x, y in vd[b]])
    # FFNN's symmetric shards tie on t-level: the trials must not all agree
    assert len({tuple(vd[b, :, 0]) for b in range(B)}) > 1
    # deterministic teacher = the tie-free first choice
    det = ctx.rollout_batch(init_policy_params(pc, 0), 1, 0.0, 5, mode="teacher",
                            trace_steps=True, wide=wide).step_vd.cpu().numpy()[0]
    _check_cp_trial(g, cl, tlev, [(int(x), int(y)) for x, y in det])


def test_critical_path_assign_best_of_trials():
    g, cl = builders.build_chainmm(64, 2), ClusterSpec.uniform(4, 1e6, 1e5)
    best, mk, assign, mks = critical_path_assign(g, cl, trials=32, seed=3, return_all=True)
    for b in (0, 7, 31):
        omk, _ = osim.exec_time(g, assign[b], cl)
        assert mks[b] == omk
    assert mk == mks.min() and list(best) == list(assign[int(np.argmin(mks))])
    assert critical_path_assign(g, cl, trials=1, seed=0).engine == "critical_path"
    with pytest.raises(ValueError):
        critical_path_assign(g, cl, trials=0)


class _DuckRule:
    """A teacher the kernel does not know: the reference select / place API."""

    def __init__(self, rule):
        self.rule = rule

    def select(self, candidates):
        return self.rule.select(candidates)

    def place(self, v, timeline):
        return self.rule.place(v, timeline)


def test_duck_teacher_matches_native_teacher_mode():
    """An arbitrary teacher object is stepped on the host and replayed in
    FORCED mode: the same actions and log-probs as the native CriticalPathRule
    teacher, and imitation training with it gives the same parameters."""
    import torch

    from paper_2505_23131_b200.heuristics import CriticalPathRule
    from paper_2505_23131_b200.training import TrainConfig, imitation_stage, measure_teacher_agreement
    g, cl = builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, 1e6, 1e5)
    pc = PolicyConfig()
    params = init_policy_params(pc, seed=0)
    ctx = PolicyContext(g, cl, pc)
    rule = CriticalPathRule(g, cl, ctx.features)
    duck = _DuckRule(rule)
    a1, t1 = ctx.rollout(params, 0.0, 3, teacher=rule)
    a2, t2 = ctx.rollout(params, 0.0, 3, teacher=duck)
    assert tuple(a1) == tuple(a2)
    assert [(s.vertex, s.device) for s in t1.steps] == [(s.vertex, s.device) for s in t2.steps]
    assert np.allclose([s.sel_logprob for s in t1.steps], [s.sel_logprob for s in t2.steps],
                       rtol=0, atol=1e-12)
    assert np.allclose([s.plc_logprob for s in t1.steps], [s.plc_logprob for s in t2.steps],
                       rtol=0, atol=1e-12)
    assert measure_teacher_agreement(ctx, params, duck, rollouts=4) == \
        measure_teacher_agreement(ctx, params, rule, rollouts=4)
    cfg = TrainConfig(episodes=8, lr0=1e-3, lr1=1e-3)
    r1 = imitation_stage(g, cl, cfg, pc, init_policy_params(pc, seed=0), teacher=rule,
                         batch_size=4)
    r2 = imitation_stage(g, cl, cfg, pc, init_policy_params(pc, seed=0), teacher=duck,
                         batch_size=4)
    for k in r1.params:
        assert np.allclose(r1.params[k].data, r2.params[k].data, rtol=0, atol=1e-12), k
    assert r1.final_loss == pytest.approx(r2.final_loss, rel=1e-12)
    torch.cuda.synchronize()
