"""GPU: CUDA policy path (encode + fused rollout/simulation) vs the reference
(golden traces, teacher-forced actions bit-exact) and the numpy oracle
(same Philox draws -> same sampled actions; log-probs within 1e-9)."""
import numpy as np
import pytest

from helpers import graph_from_golden
from oracle import policy as OP
from oracle import sim as osim
from paper_2505_23131_b200 import builders
from paper_2505_23131_b200.cluster import ClusterSpec
from paper_2505_23131_b200.heuristics import CriticalPathRule, ForcedActions
from paper_2505_23131_b200.params import init_policy_params
from paper_2505_23131_b200.policy import PolicyConfig, PolicyContext, TeacherActionError

pytestmark = pytest.mark.gpu
TOL = 1e-9


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


def _close(a, b, tol=TOL):
    return abs(a - b) <= tol * max(1.0, abs(b))


def _oracle_probs(ctx, params, want):
    """Per-step (sel, plc) probability vectors of a forced replay (oracle)."""
    octx = _oracle_ctx(ctx)
    ro = OP.rollout(OP.leaves(params, need=False), octx, 0.0, mode="forced",
                    forced=[(w["vertex"], w["device"]) for w in want])
    return [(s["candidates"], s["sel_probs"], s["plc_probs"]) for s in ro["steps"]]


def _check_steps(trace, want, probs=None, actions=True):
    """Actions exact; log-probs / entropies within TOL; greedy argmax exact
    unless the two candidates are a near-tie (|dp| <= 1e-9 p), where the
    winner is decided by rounding noise in either implementation."""
    assert len(trace.steps) == len(want)
    for t, (s, w) in enumerate(zip(trace.steps, want)):
        if actions:
            assert list(s.candidates) == w["candidates"]
            assert (s.vertex, s.device) == (w["vertex"], w["device"])
        for k in ("sel_logprob", "plc_logprob", "sel_entropy", "plc_entropy"):
            assert _close(getattr(s, k), w[k]), (k, getattr(s, k), w[k])
        if (s.sel_argmax, s.plc_argmax) != (w["sel_argmax"], w["plc_argmax"]):
            assert probs is not None, (t, s.sel_argmax, w["sel_argmax"])
            cands, ps, pp = probs[t]
            a, b = cands.index(s.sel_argmax), cands.index(w["sel_argmax"])
            assert abs(ps[a] - ps[b]) <= 1e-9 * ps[b], (t, ps[a], ps[b])
            assert abs(pp[s.plc_argmax] - pp[w["plc_argmax"]]) <= 1e-9 * pp[w["plc_argmax"]]


def test_encoder_tables_match_reference(policy_golden, torch_cuda):
    for case in policy_golden["cases"]:
        g, cl, pc, ctx = _ctx(case)
        ctx.prepare(init_policy_params(pc, seed=0))
        for name, key in (("H_sel", "H_sel"), ("H_plc", "H_plc")):
            np.testing.assert_allclose(ctx.read_table(name), np.asarray(case[key]),
                                       rtol=1e-11, atol=1e-12, err_msg=case["tag"])


def test_teacher_greedy_and_forced_match_reference(policy_golden, torch_cuda):
    for case in policy_golden["cases"]:
        g, cl, pc, ctx = _ctx(case)
        params = init_policy_params(pc, seed=0)
        teacher = CriticalPathRule(g, cl, ctx.features)
        want = case["teacher"]["trace"]
        a, tr = ctx.rollout(params, case["teacher"]["epsilon"], 0, teacher=teacher)
        _check_steps(tr, want, _oracle_probs(ctx, params, want))
        assert tr.encode_invocations == 2
        # greedy: the reference's greedy actions replayed (its argmax is decided
        # by BLAS rounding on near-ties, so the episode itself is replayed)
        want = case["greedy"]["trace"]
        acts = [(x["vertex"], x["device"]) for x in want]
        a, tr = ctx.rollout(params, 0.0, 0, teacher=ForcedActions(acts))
        _check_steps(tr, want, _oracle_probs(ctx, params, want))
        for s in case["sampled"]:
            acts = [(x["vertex"], x["device"]) for x in s["trace"]]
            a, tr = ctx.rollout(params, s["epsilon"], 0, teacher=ForcedActions(acts))
            assert list(a) == s["assign"]
            _check_steps(tr, s["trace"], _oracle_probs(ctx, params, s["trace"]))


def test_bad_forced_action_raises(policy_golden, torch_cuda):
    case = policy_golden["cases"][0]
    g, cl, pc, ctx = _ctx(case)
    acts = [(999, 0)] * len(g)
    with pytest.raises(TeacherActionError):
        ctx.rollout(init_policy_params(pc, seed=0), 0.0, 0, teacher=ForcedActions(acts))


def _oracle_ctx(ctx):
    pc = ctx.config
    return OP.Ctx(ctx.graph, ctx.cluster, pc.hidden, pc.k_rounds, pc.leaky_slope,
                  pc.shared_encoder, ctx.features)


@pytest.mark.parametrize("which", ["ffnn", "chainmm", "llama"])
def test_sampled_batch_matches_oracle_draws(which, torch_cuda):
    if which == "ffnn":
        g, cl, pc = builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, 1e6, 1e5), \
            PolicyConfig()
    elif which == "chainmm":
        g, cl, pc = builders.build_chainmm(64, 2), ClusterSpec.uniform(4, 1e6, 1e5), \
            PolicyConfig(hidden=16, k_rounds=1, shared_encoder=True)
    else:
        g, cl, pc = builders.build_llama_block(), ClusterSpec.uniform(8, 1e9, 1e7), PolicyConfig()
    params = init_policy_params(pc, seed=3)
    ctx = PolicyContext(g, cl, pc)
    B, seed, base = 64, 1234, 7
    rb = ctx.rollout_batch(params, B, 0.2, seed, trace_steps=True, episode_base=base)
    st = rb.status.cpu().numpy()
    assert (st == 0).all()
    vd = rb.step_vd.cpu().numpy()
    lp = rb.step_lp.cpu().numpy()
    ent = rb.step_ent.cpu().numpy()
    mk = rb.makespan.cpu().numpy()
    assign = rb.assign.cpu().numpy()
    octx = _oracle_ctx(ctx)
    P = OP.leaves(params, need=False)
    check = range(B) if which != "llama" else range(0, B, 16)
    for b in check:
        ro = OP.rollout(P, octx, 0.2, mode="uniform", seed=seed, episode=base + b)
        got = [(int(vd[b, t, 0]), int(vd[b, t, 1])) for t in range(len(g))]
        want = [(s["vertex"], s["device"]) for s in ro["steps"]]
        assert got == want, (which, b)
        for t, s in enumerate(ro["steps"]):
            assert _close(lp[b, t, 0], s["sel_logprob"]) and _close(lp[b, t, 1], s["plc_logprob"])
            assert _close(ent[b, t, 0], s["sel_entropy"]) and _close(ent[b, t, 1], s["plc_entropy"])
        assert list(assign[b]) == ro["assign"]
        omk, _ = osim.exec_time(g, assign[b], cl)
        assert mk[b] == omk


def test_fused_simulation_trace_bit_exact(torch_cuda):
    from paper_2505_23131_b200.simulate import decode_events
    g, cl = builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, 1e6, 1e5)
    pc = PolicyConfig()
    ctx = PolicyContext(g, cl, pc)
    for strat in ("fifo", "depth_first", "breadth_first"):
        rb = ctx.rollout_batch(init_policy_params(pc, 0), 32, 0.5, 99, strategy=strat,
                               sim_trace=True)
        assign = rb.assign.cpu().numpy()
        tr = rb.trace.cpu().numpy()
        tl = rb.trace_len.cpu().numpy()
        mk = rb.makespan.cpu().numpy()
        for b in range(32):
            omk, oev = osim.exec_time(g, assign[b], cl, strat)
            assert mk[b] == omk
            assert decode_events(tr[b], int(tl[b])) == oev


def test_epsilon_one_is_uniform(torch_cuda):
    from paper_2505_23131_b200.graph import DataflowGraph, OpKind, Vertex
    g = DataflowGraph((Vertex(0, OpKind.MATMUL, 10, 8, "a"), Vertex(1, OpKind.MATMUL, 10, 8, "b")),
                      ())
    cl = ClusterSpec.uniform(2, 1000.0, 256.0)
    pc = PolicyConfig(hidden=8)
    ctx = PolicyContext(g, cl, pc)
    B = 20000
    rb = ctx.rollout_batch(init_policy_params(pc, 0), B, 1.0, 5, trace_steps=True)
    a = rb.assign.cpu().numpy()
    counts = np.zeros((2, 2))
    np.add.at(counts, (a[:, 0], a[:, 1]), 1)
    sigma = np.sqrt(B * 0.25 * 0.75)
    assert np.all(np.abs(counts - B / 4) <= 4 * sigma)
    lp = rb.step_lp.cpu().numpy()
    assert np.allclose(lp[:, :, 1], np.log(0.5), atol=1e-12)


# ---- wide (HBM-resident) rollout path --------------------------------------
def _rollout_np(rb):
    return {k: getattr(rb, k).cpu().numpy() for k in (
        "assign", "status", "makespan", "step_vd", "step_lp", "step_ent", "step_argmax",
        "step_ncand")}


@pytest.mark.parametrize("which", ["ffnn", "llama"])
def test_wide_rollout_matches_compact(which, torch_cuda):
    """The candidate-tree / HBM-state kernel forced onto graphs the compact
    kernel also runs: identical actions, assignments and makespans under the
    same Philox draws; log-probs and entropies within 1e-12 (the tree sums
    candidates in a different order)."""
    if which == "ffnn":
        g, cl = builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, 1e6, 1e5)
    else:
        g, cl = builders.build_llama_block(), ClusterSpec.uniform(8, 1e9, 1e7)
    pc = PolicyConfig()
    params = init_policy_params(pc, seed=5)
    ctx = PolicyContext(g, cl, pc)
    for mode, eps in (("sample", 0.2), ("sample", 0.9), ("teacher", 0.0), ("greedy", 0.0)):
        a = _rollout_np(ctx.rollout_batch(params, 48, eps, 77, mode=mode, trace_steps=True))
        b = _rollout_np(ctx.rollout_batch(params, 48, eps, 77, mode=mode, trace_steps=True,
                                          wide=True))
        assert (a["status"] == 0).all() and (b["status"] == 0).all()
        for k in ("assign", "step_vd", "step_ncand", "makespan"):
            assert np.array_equal(a[k], b[k]), (which, mode, k)
        np.testing.assert_allclose(b["step_lp"], a["step_lp"], rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(b["step_ent"], a["step_ent"], rtol=1e-12, atol=1e-14)
        assert np.array_equal(a["step_argmax"], b["step_argmax"]), (which, mode)
        # forced replay of the same actions through the wide kernel
        f = _rollout_np(ctx.rollout_batch(params, 48, eps, 0, mode="forced",
                                          forced=a["step_vd"], trace_steps=True, wide=True))
        assert np.array_equal(f["assign"], a["assign"]) and np.array_equal(f["makespan"],
                                                                           a["makespan"])
        np.testing.assert_allclose(f["step_lp"], a["step_lp"], rtol=1e-12, atol=1e-14)


def test_wide_bad_actions_terminate(torch_cuda):
    """A bad forced device far beyond the hand-off ring depth must release the
    producer warp (no hang) and report FP_EP_BAD_ACTION."""
    g, cl = builders.build_llama_block(), ClusterSpec.uniform(8, 1e9, 1e7)
    pc = PolicyConfig()
    params = init_policy_params(pc, seed=0)
    ctx = PolicyContext(g, cl, pc)
    ref = ctx.rollout_batch(params, 2, 0.0, 0, mode="teacher", trace_steps=True)
    acts = ref.step_vd.cpu().numpy().copy()
    acts[0, 3, 1] = 99        # bad device early: SEL warp is blocked on a full ring
    acts[1, 150, 0] = 10 ** 6  # bad vertex late
    rb = ctx.rollout_batch(params, 2, 0.0, 0, mode="forced", forced=acts, wide=True)
    assert rb.status.cpu().numpy().tolist() == [3, 3]


def test_wide_large_dag_matches_oracle_draws(torch_cuda):
    """A 2k-op sparse DAG (beyond the compact kernel): sampled episodes equal
    the numpy oracle's under the same Philox draws; makespans bit-exact."""
    g, cl = builders.sparse_dag(2000, seed=3), ClusterSpec.uniform(8, 1e9, 1e7)
    pc = PolicyConfig()
    params = init_policy_params(pc, seed=1)
    ctx = PolicyContext(g, cl, pc)
    assert ctx.workspace(4) is not None
    B, seed = 4, 31
    rb = ctx.rollout_batch(params, B, 0.2, seed, trace_steps=True)
    r = _rollout_np(rb)
    assert (r["status"] == 0).all()
    octx = _oracle_ctx(ctx)
    P = OP.leaves(params, need=False)
    for b in (0, 3):
        ro = OP.rollout(P, octx, 0.2, mode="uniform", seed=seed, episode=b)
        got = [(int(r["step_vd"][b, t, 0]), int(r["step_vd"][b, t, 1])) for t in range(len(g))]
        assert got == [(s["vertex"], s["device"]) for s in ro["steps"]], b
        for t in range(0, len(g), 97):
            s = ro["steps"][t]
            assert _close(r["step_lp"][b, t, 0], s["sel_logprob"])
            assert _close(r["step_ent"][b, t, 0], s["sel_entropy"])
            assert _close(r["step_lp"][b, t, 1], s["plc_logprob"])
        omk, _ = osim.exec_time(g, r["assign"][b], cl)
        assert r["makespan"][b] == omk


def test_forest_path_sums_match_path_lists(torch_cuda):
    """SEL logits from pointer-jumped path sums (large-graph form) equal the
    explicit path-list sums to rounding."""
    for g, cl in ((builders.build_llama_block(), ClusterSpec.uniform(8, 1e9, 1e7)),
                  (builders.sparse_dag(900, seed=4), ClusterSpec.uniform(8, 1e9, 1e7))):
        pc = PolicyConfig()
        params = init_policy_params(pc, seed=2)
        a = PolicyContext(g, cl, pc)
        b = PolicyContext(g, cl, pc, forest=True)
        a.prepare(params)
        b.prepare(params)
        np.testing.assert_allclose(b.read_table("sel_logit"), a.read_table("sel_logit"),
                                   rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("which", ["ffnn", "chainmm_h16", "fixture_h8"])
def test_dmma_encoder_matches_fused_encoder(which, torch_cuda):
    """The split encoder (aggregation + fp64 tensor-core node MLPs) against the
    fused CUDA-core encoder that keeps the reference's FMA order: every
    head table within 1e-12 relative."""
    from helpers import fixture6
    if which == "ffnn":
        g, cl, pc = builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, 1e6, 1e5), \
            PolicyConfig()
    elif which == "chainmm_h16":
        g, cl, pc = builders.build_chainmm(64, 2), ClusterSpec.uniform(4, 1e6, 1e5), \
            PolicyConfig(hidden=16, k_rounds=3, shared_encoder=True)
    else:
        g, cl, pc = fixture6(), ClusterSpec.uniform(2, 1000.0, 256.0), PolicyConfig(hidden=8)
    params = init_policy_params(pc, seed=9)
    a = PolicyContext(g, cl, pc)
    b = PolicyContext(g, cl, pc)
    b.set_encoder(fused=True)
    a.prepare(params)
    b.prepare(params)
    for name in ("H_sel", "H_plc", "sel_logit", "A", "G", "M", "c"):
        x, y = a.read_table(name), b.read_table(name)
        np.testing.assert_allclose(x, y, rtol=1e-12, atol=1e-13 * max(1.0, np.abs(y).max()),
                                   err_msg=f"{which}:{name}")


def test_wide_tree_underflow_fallback(torch_cuda):
    """Logits spread over thousands of nats: candidate weights exp(s - max s)
    underflow to zero and the wide kernel takes its max-shifted slow pass;
    actions and log-probs still match the compact kernel."""
    g, cl = builders.build_llama_block(), ClusterSpec.uniform(8, 1e9, 1e7)
    pc = PolicyConfig()
    params = init_policy_params(pc, seed=4)
    params["sel.head2.w"].data = params["sel.head2.w"].data * 4000.0
    ctx = PolicyContext(g, cl, pc)
    ctx.prepare(params)
    s = ctx.read_table("sel_logit")
    assert s.max() - s.min() > 1000.0
    a = _rollout_np(ctx.rollout_batch(params, 32, 0.2, 5, trace_steps=True))
    b = _rollout_np(ctx.rollout_batch(params, 32, 0.2, 5, trace_steps=True, wide=True))
    assert (a["status"] == 0).all() and (b["status"] == 0).all()
    assert np.array_equal(a["step_vd"], b["step_vd"]) and np.array_equal(a["makespan"], b["makespan"])
    np.testing.assert_allclose(b["step_lp"], a["step_lp"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("wide", [False, True])
def test_multi_slot_cluster_rollouts_match_oracle(wide, torch_cuda):
    """Clusters with several exec / transfer slots per resource take the
    shared-memory in-flight pool (not the single-slot register path) in the
    overlapped (compact) and wide simulators; sampled episodes and their
    makespans still match the oracle."""
    rng = np.random.default_rng(3)
    d = 4
    bw = rng.uniform(1e4, 1e5, size=(d, d))
    cl = ClusterSpec(d, tuple(rng.uniform(5e5, 2e6, size=d)), tuple(map(tuple, bw)),
                     (2, 1, 3, 2), tuple(tuple(int(x) for x in r)
                                         for r in rng.integers(1, 3, size=(d, d))))
    g = builders.build_chainmm(64, 2)
    pc = PolicyConfig(hidden=16, k_rounds=2)
    params = init_policy_params(pc, seed=6)
    ctx = PolicyContext(g, cl, pc)
    B, seed = 24, 9
    rb = ctx.rollout_batch(params, B, 0.3, seed, trace_steps=True, wide=wide, sim_trace=True)
    assert (rb.status.cpu().numpy() == 0).all()
    vd, mk = rb.step_vd.cpu().numpy(), rb.makespan.cpu().numpy()
    assign = rb.assign.cpu().numpy()
    from paper_2505_23131_b200.simulate import decode_events
    tr, tl = rb.trace.cpu().numpy(), rb.trace_len.cpu().numpy()
    octx = _oracle_ctx(ctx)
    P = OP.leaves(params, need=False)
    for b in (0, 11, 23):
        ro = OP.rollout(P, octx, 0.3, mode="uniform", seed=seed, episode=b)
        assert [(int(x), int(y)) for x, y in vd[b]] == [(s["vertex"], s["device"])
                                                        for s in ro["steps"]]
        omk, oev = osim.exec_time(g, assign[b], cl)
        assert mk[b] == omk
        assert decode_events(tr[b], int(tl[b])) == oev


@pytest.mark.parametrize("d", [3, 6, 12])
def test_odd_device_counts_match_oracle(d, torch_cuda):
    """Device counts that are not powers of two (true division in the
    standardisation, padded device lanes in the PLC reductions)."""
    g = builders.build_ffnn(8, 4, 16, 4, 2)
    cl = ClusterSpec.uniform(d, 1e6, 1e5)
    pc = PolicyConfig(hidden=16, k_rounds=2)
    params = init_policy_params(pc, seed=8)
    ctx = PolicyContext(g, cl, pc)
    B, seed = 16, 21
    rb = ctx.rollout_batch(params, B, 0.2, seed, trace_steps=True)
    assert (rb.status.cpu().numpy() == 0).all()
    vd, lp, mk = rb.step_vd.cpu().numpy(), rb.step_lp.cpu().numpy(), rb.makespan.cpu().numpy()
    octx = _oracle_ctx(ctx)
    P = OP.leaves(params, need=False)
    for b in (0, 15):
        ro = OP.rollout(P, octx, 0.2, mode="uniform", seed=seed, episode=b)
        assert [(int(x), int(y)) for x, y in vd[b]] == [(s["vertex"], s["device"])
                                                        for s in ro["steps"]]
        for t, s in enumerate(ro["steps"]):
            assert _close(lp[b, t, 1], s["plc_logprob"])
        omk, _ = osim.exec_time(g, rb.assign.cpu().numpy()[b], cl)
        assert mk[b] == omk
    # per_step on the same odd cluster
    pc2 = PolicyConfig(hidden=16, k_rounds=1, mp_mode="per_step")
    ctx2 = PolicyContext(g, cl, pc2)
    p2 = init_policy_params(pc2, seed=8)
    rb2 = ctx2.rollout_batch(p2, 4, 0.2, seed, trace_steps=True)
    ro = OP.rollout(OP.leaves(p2, need=False), _oracle_ctx(ctx2), 0.2, mode="uniform", seed=seed,
                    episode=1, per_step=True)
    assert [(int(x), int(y)) for x, y in rb2.step_vd.cpu().numpy()[1]] == \
        [(s["vertex"], s["device"]) for s in ro["steps"]]
