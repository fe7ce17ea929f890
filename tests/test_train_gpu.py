"""GPU: REINFORCE gradient of the CUDA path vs the reference's autodiff
(golden, one Stage-II episode and one imitation episode at B = 1) and vs the
numpy tape oracle for a batch; trainer semantics (baseline, zero lr)."""
import numpy as np
import pytest

from helpers import graph_from_golden
from oracle import policy as OP
from paper_2505_23131_b200 import builders
from paper_2505_23131_b200.cluster import ClusterSpec
from paper_2505_23131_b200.params import init_policy_params
from paper_2505_23131_b200.policy import PolicyConfig, PolicyContext

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


def _ctx(case):
    g = graph_from_golden(case["graph"])
    cl = ClusterSpec.from_dict(case["cluster"])
    pc = PolicyConfig.from_dict(case["policy"])
    return g, cl, pc, PolicyContext(g, cl, pc)


def _compare(ctx, grad, want, rtol=1e-8):
    got = ctx.layout.unflatten(grad.cpu().numpy())
    for name, vals in want.items():
        np.testing.assert_allclose(got[name].data.reshape(-1), vals, rtol=rtol, atol=1e-12,
                                   err_msg=name)


def test_rl_gradient_matches_reference(policy_golden, torch_cuda):
    for case in policy_golden["cases"]:
        if "rl_grad" not in case:
            continue
        g, cl, pc, ctx = _ctx(case)
        params = init_policy_params(pc, seed=0)
        rg = case["rl_grad"]
        acts = [(x["vertex"], x["device"]) for x in case["sampled"][0]["trace"]]
        rb = ctx.rollout_batch(params, 1, rg["epsilon"], 0, mode="forced",
                               forced=np.asarray(acts).reshape(1, -1, 2), grad=True)
        assert int(rb.status.cpu()[0]) == 0
        assert float(rb.makespan.cpu()[0]) == case["sampled"][0]["makespan"]
        grad = ctx.policy_gradient(rb, [-rg["advantage"]], -rg["entropy_weight"])
        _compare(ctx, grad, rg["grads"])


def test_imitation_gradient_matches_reference(policy_golden, torch_cuda):
    for case in policy_golden["cases"]:
        if "imitation_grad" not in case:
            continue
        g, cl, pc, ctx = _ctx(case)
        rb = ctx.rollout_batch(init_policy_params(pc, seed=0), 1, 0.0, 0, mode="teacher",
                               grad=True)
        grad = ctx.policy_gradient(rb, [-1.0], 0.0)
        _compare(ctx, grad, case["imitation_grad"]["grads"])


def test_batched_gradient_matches_oracle_sum(torch_cuda):
    g, cl = builders.build_chainmm(64, 2), ClusterSpec.uniform(4, 1e6, 1e5)
    pc = PolicyConfig(hidden=16, k_rounds=2)
    params = init_policy_params(pc, seed=4)
    ctx = PolicyContext(g, cl, pc)
    B = 6
    rb = ctx.rollout_batch(params, B, 0.3, 77, grad=True, trace_steps=True)
    mk = rb.makespan.cpu().numpy()
    alpha = (mk - mk.mean()) / B
    beta = -0.01 / B
    grad = ctx.policy_gradient(rb, alpha, beta).cpu().numpy()
    vd = rb.step_vd.cpu().numpy()
    octx = OP.Ctx(g, cl, pc.hidden, pc.k_rounds, pc.leaky_slope, pc.shared_encoder,
                  ctx.features)
    want = np.zeros_like(grad)
    for b in range(B):
        forced = [(int(v), int(d)) for v, d in vd[b]]
        # oracle grads of -(adv*sum lp + w*sum ent) = alpha*sum lp + beta*sum ent with
        # adv = -alpha*B, w = -beta*B, scaled by 1/B
        gr, _ = OP.rl_gradients(params, octx, 0.3, -alpha[b] * B, -beta * B, mode="forced",
                                forced=forced)
        want += ctx.layout.flatten({k: v / B for k, v in gr.items()})
    np.testing.assert_allclose(grad, want, rtol=1e-8, atol=1e-13)


def test_trainer_zero_lr_keeps_params_and_baseline(torch_cuda):
    from paper_2505_23131_b200.training import BatchedTrainer, TrainConfig
    g, cl = builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, 1e6, 1e5)
    pc = PolicyConfig()
    params = init_policy_params(pc, seed=0)
    ctx = PolicyContext(g, cl, pc)
    tr = BatchedTrainer(ctx, params, TrainConfig(episodes=64, lr0=0.0, lr1=0.0), batch_size=16)
    before = tr.flat.clone()
    st1 = tr.step(seed=1, record=True)
    st2 = tr.step(seed=2, record=True)
    assert (tr.flat == before).all()
    assert np.allclose(st1["advantage"], -st1["makespan"])          # baseline 0 first
    base = -st1["makespan"].mean()
    assert np.allclose(st2["advantage"], -st2["makespan"] - base)   # mean of previous returns
    assert tr.upd.count == 32


def test_sim_rl_stage_improves_on_fixture(torch_cuda):
    from helpers import cluster2, fixture6
    from paper_2505_23131_b200.training import TrainConfig, sim_rl_stage
    pc = PolicyConfig(hidden=16, k_rounds=1)
    params = init_policy_params(pc, seed=0)
    cfg = TrainConfig(episodes=2048, lr0=1e-3, lr1=1e-4, seed=0)
    # reference acceptance criterion 6 (tests/test_acceptance.py:148-164)
    from paper_2505_23131_b200.heuristics import brute_force_optimal, random_assign
    from paper_2505_23131_b200.simulate import exec_time, exec_time_batch
    g, cl = fixture6(), cluster2()
    res = sim_rl_stage(g, cl, cfg, pc, params, batch_size=128)
    mks = [r["makespan_ms"] for r in res.curve]
    assert len(mks) == 2048
    assert res.best_makespan == min(mks)
    assert res.curve[0]["advantage"] == -res.curve[0]["makespan_ms"]
    rand = exec_time_batch(g, [list(random_assign(g, 2, seed=s)) for s in range(100)], cl)
    _, oracle = brute_force_optimal(g, cl)
    assert res.best_makespan <= rand.mean()
    assert res.best_makespan <= 1.10 * oracle
    assert exec_time(g, res.best_assignment, cl)[0] == res.best_makespan


def test_system_rl_batched_executor_matches_per_call():
    """Stage III (training.py:235-248) with the jittered simulator executor:
    the batched path (one simulation launch per update, per-episode seeds in
    call order) gives the same rewards and updates as per-episode calls."""
    from paper_2505_23131_b200.training import SimulatorExecutor, TrainConfig, system_rl_stage
    g, cl = builders.build_chainmm(64, 2), ClusterSpec.uniform(4, 1e6, 1e5)
    pc = PolicyConfig(hidden=16, k_rounds=1)
    cfg = TrainConfig(episodes=8, seed=0)
    batched = SimulatorExecutor(cl, jitter_sigma=0.1, base_seed=5)
    per_call = SimulatorExecutor(cl, jitter_sigma=0.1, base_seed=5)
    r1 = system_rl_stage(g, cl, batched, cfg, pc, init_policy_params(pc, 0), batch_size=4)
    r2 = system_rl_stage(g, cl, lambda gg, a: per_call(gg, a), cfg, pc,
                         init_policy_params(pc, 0), batch_size=4)
    m1 = [row["makespan_ms"] for row in r1.curve]
    m2 = [row["makespan_ms"] for row in r2.curve]
    assert m1 == m2 and len(m1) == 8


def test_trainer_failed_rollout_masks_update_and_raises(torch_cuda):
    """A failed episode (status != 0) is counted on the device: that step's
    SGD update (and every later one) is skipped without a host sync inside
    the step, and the trainer raises at its next check."""
    from paper_2505_23131_b200.training import BatchedTrainer, TrainConfig
    g, cl = builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, 1e6, 1e5)
    pc = PolicyConfig()
    ctx = PolicyContext(g, cl, pc)
    tr = BatchedTrainer(ctx, init_policy_params(pc, seed=0), TrainConfig(episodes=64),
                        batch_size=16)
    tr.step(seed=1)
    tr.check()                      # clean step: nothing to raise
    before = tr.flat.clone()
    real = ctx.rollout_batch

    def failing(*a, **kw):          # the rollout reports a deadlock for episode 3
        out = real(*a, **kw)
        kw["out"].status[3] = 1
        return out

    ctx.rollout_batch = failing
    tr.step(seed=2)
    ctx.rollout_batch = real
    assert (tr.flat == before).all()   # masked on the device
    with pytest.raises(RuntimeError, match="rollout failed"):
        tr.check()


@pytest.fixture(scope="module")
def per_step_grad_golden():
    import json
    from pathlib import Path
    return json.loads((Path(__file__).parent / "golden" / "per_step_grad.json").read_text())


def test_per_step_rl_gradient_matches_reference(per_step_grad_golden, torch_cuda):
    """per_step REINFORCE: the reference's sampled per_step episode, forced on
    the GPU, gives the reference's full parameter gradient (backpropagated
    through one encode per step, reference autodiff) within 1e-8."""
    for case in per_step_grad_golden["cases"]:
        g, cl, pc, ctx = _ctx(case)
        assert ctx.per_step
        params = init_policy_params(pc, seed=0)
        rg = case["rl_grad"]
        acts = [(x["vertex"], x["device"]) for x in rg["trace"]]
        rb = ctx.rollout_batch(params, 1, rg["epsilon"], 0, mode="forced",
                               forced=np.asarray(acts).reshape(1, -1, 2), grad=True,
                               trace_steps=True)
        assert int(rb.status.cpu()[0]) == 0, case["tag"]
        assert float(rb.makespan.cpu()[0]) == rg["makespan"], case["tag"]
        lp = rb.step_lp.cpu().numpy()[0]
        np.testing.assert_allclose(lp[:, 0], [x["sel_logprob"] for x in rg["trace"]],
                                   rtol=0, atol=1e-9)
        grad = ctx.policy_gradient(rb, [-rg["advantage"]], -rg["entropy_weight"])
        _compare(ctx, grad, rg["grads"])


def test_per_step_imitation_gradient_matches_reference(per_step_grad_golden, torch_cuda):
    for case in per_step_grad_golden["cases"]:
        g, cl, pc, ctx = _ctx(case)
        rb = ctx.rollout_batch(init_policy_params(pc, seed=0), 1, 0.0, 0, mode="teacher",
                               grad=True)
        assert int(rb.status.cpu()[0]) == 0, case["tag"]
        grad = ctx.policy_gradient(rb, [-1.0], 0.0)
        _compare(ctx, grad, case["imitation_grad"]["grads"])


def test_per_step_sim_rl_stage_trains(torch_cuda):
    """sim_rl_stage with mp_mode="per_step" (the reference's acceptance
    criterion 8 setup): trains, n x the encoder invocations of per_episode."""
    from helpers import cluster2, fixture6
    from paper_2505_23131_b200.training import TrainConfig, sim_rl_stage
    g, cl = fixture6(), cluster2()
    res = {}
    for mode in ("per_episode", "per_step"):
        pc = PolicyConfig(hidden=16, k_rounds=2, mp_mode=mode)
        res[mode] = sim_rl_stage(g, cl, TrainConfig(episodes=8, seed=0), pc,
                                 init_policy_params(pc, seed=0), batch_size=1)
        assert np.isfinite(res[mode].best_makespan)
    # reference criterion 8's counts at one episode per update
    assert res["per_episode"].encoder_invocations == 2 * 8
    assert res["per_step"].encoder_invocations == len(g) * res["per_episode"].encoder_invocations
