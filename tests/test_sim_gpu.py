"""GPU: CUDA work-conserving simulator vs the reference's event streams and
the C oracle — bit-exact makespans and schedules (the
reference's own tests/test_backends.py pattern)."""
import numpy as np
import pytest

from helpers import cluster2, graph_from_golden, random_dag
from oracle import sim as osim
from paper_2505_23131_b200 import builders
from paper_2505_23131_b200.cluster import ClusterSpec
from paper_2505_23131_b200.features import static_features

pytestmark = pytest.mark.gpu
STRATS = ("fifo", "depth_first", "breadth_first")


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def test_exec_time_matches_reference_golden(sim_golden, torch_cuda):
    from paper_2505_23131_b200 import simulate as S
    for c in sim_golden:
        g = graph_from_golden(c["graph"])
        cl = ClusterSpec.from_dict(c["cluster"])
        if "deadlock" in c:
            with pytest.raises(S.DeadlockError, match="blocked frontier") as ei:
                S.exec_time(g, c["assign"], cl, c["strategy"], c["seed"])
            assert ei.value.time_ms == c["deadlock"]["time"]
            assert ei.value.blocked == c["deadlock"]["blocked"]
            continue
        mk, sched = S.exec_time(g, c["assign"], cl, c["strategy"], c["seed"])
        assert mk == c["makespan"], c["tag"]
        got = [[0 if e.task.kind == "exec" else 1, e.task.vertex,
                e.task.device if e.task.kind == "exec" else e.task.src,
                -1 if e.task.kind == "exec" else e.task.dst, e.time_ms,
                0 if e.type == "beg" else 1] for e in sched.events]
        assert got == c["events"], (c["tag"], c["strategy"])


def _batch_vs_oracle(torch, g, cl, B, seed, strategies=STRATS, wide=False, check=None):
    from paper_2505_23131_b200.simulate import SimProblem, decode_events
    feats = static_features(g, cl.comm_factor)
    prob = SimProblem(g, cl, feats)
    rng = np.random.default_rng(seed)
    a = rng.integers(0, cl.device_count, size=(B, len(g))).astype(np.int32)
    at = torch.from_numpy(a).cuda()
    for s in strategies:
        out = prob.simulate(at, s, trace=True, wide=wide)
        mk = out["makespan"].cpu().numpy()
        st = out["status"].cpu().numpy()
        ev = out["events"].cpu().numpy()
        tl = out["trace_len"].cpu().numpy()
        assert (st == 0).all()
        for b in (range(B) if check is None else check):
            omk, oev = osim.run_packed(*osim.pack(g, a[b], cl, feats, s, 0))
            assert mk[b] == omk, (s, b)
            assert decode_events(ev[b], int(tl[b])) == oev, (s, b)
        # makespan-only launch agrees with the traced one
        out2 = prob.simulate(at, s, trace=False, wide=wide)
        assert np.array_equal(out2["makespan"].cpu().numpy(), mk)


def test_random_dags_slots_devices_vs_oracle(torch_cuda):
    rng = np.random.default_rng(11)
    for dev, es, ts in ((1, 1, 1), (2, 1, 1), (3, 2, 1), (4, 1, 3), (8, 2, 2)):
        cl = ClusterSpec.uniform(dev, rate=100.0, bandwidth=64.0, exec_slots=es,
                                 transfer_slots=ts)
        for k in range(6):
            g = random_dag(rng, max_vertices=12)
            _batch_vs_oracle(torch_cuda, g, cl, 8, 100 * dev + k)


def test_bench_graphs_vs_oracle(torch_cuda):
    c4 = ClusterSpec.uniform(4, rate=1e6, bandwidth=1e5)
    c8 = ClusterSpec.uniform(8, rate=1e6, bandwidth=1e5)
    c8b = ClusterSpec.uniform(8, rate=1e9, bandwidth=1e7)
    _batch_vs_oracle(torch_cuda, builders.build_chainmm(64, 2), c4, 64, 1)
    _batch_vs_oracle(torch_cuda, builders.build_ffnn(8, 4, 16, 4, 2), c8, 64, 2)
    _batch_vs_oracle(torch_cuda, builders.build_llama_block(), c8b, 32, 3)
    _batch_vs_oracle(torch_cuda, builders.sparse_dag(1000, seed=0), c8b, 8, 4)


def test_heterogeneous_cluster_vs_oracle(torch_cuda):
    rng = np.random.default_rng(5)
    d = 4
    bw = rng.uniform(1e4, 1e5, size=(d, d))
    cl = ClusterSpec(d, tuple(rng.uniform(5e5, 2e6, size=d)), tuple(map(tuple, bw)),
                     (1, 2, 1, 2), tuple(tuple(int(x) for x in r)
                                         for r in rng.integers(1, 3, size=(d, d))))
    _batch_vs_oracle(torch_cuda, builders.build_chainmm(64, 2), cl, 64, 9)


def test_jitter_tables_bit_exact(torch_cuda):
    from paper_2505_23131_b200 import simulate as S
    from helpers import fixture6
    cl = cluster2(rate=100.0, bandwidth=64.0, jitter_sigma=0.2)
    for seed in range(4):
        mk, sched = S.exec_time(fixture6(), [0, 0, 1, 0, 1, 0], cl, "fifo", seed)
        omk, oev = osim.exec_time(fixture6(), [0, 0, 1, 0, 1, 0], cl, "fifo", seed)
        assert mk == omk


def test_exec_time_batch_api(torch_cuda):
    from paper_2505_23131_b200.simulate import exec_time_batch
    g = builders.build_ffnn(8, 4, 16, 4, 2)
    cl = ClusterSpec.uniform(8, rate=1e6, bandwidth=1e5)
    rng = np.random.default_rng(0)
    a = rng.integers(0, 8, size=(16, len(g)))
    mk, scheds = exec_time_batch(g, a, cl, schedules=True)
    for b in range(16):
        omk, _ = osim.exec_time(g, a[b], cl)
        assert mk[b] == omk == scheds[b].makespan_ms
    with pytest.raises(ValueError, match="outside the cluster"):
        exec_time_batch(g, np.full((1, len(g)), 9), cl)


# ---- wide (HBM-resident, hierarchical pending bitsets) simulator -----------
def test_wide_path_matches_reference_golden(sim_golden, torch_cuda):
    """Every reference event stream again, forcing the HBM-resident core."""
    from paper_2505_23131_b200.simulate import SimProblem, decode_events
    for c in sim_golden:
        if "deadlock" in c:
            continue
        g = graph_from_golden(c["graph"])
        cl = ClusterSpec.from_dict(c["cluster"])
        prob = SimProblem(g, cl)
        at = torch_cuda.tensor([c["assign"]], dtype=torch_cuda.int32, device="cuda")
        jit = prob.jitter_table(c["seed"])
        jt = torch_cuda.from_numpy(jit).cuda() if jit is not None else None
        out = prob.simulate(at, c["strategy"], jitter=jt, trace=True, wide=True)
        assert int(out["status"][0]) == 0
        assert float(out["makespan"][0]) == c["makespan"], c["tag"]
        ev = decode_events(out["events"][0].cpu().numpy(), int(out["trace_len"][0]))
        assert [list(e) for e in ev] == [[e[0], e[1], e[2], e[3], e[4], e[5]]
                                         for e in c["events"]], c["tag"]


def test_wide_path_random_and_bench_graphs(torch_cuda):
    rng = np.random.default_rng(21)
    for dev, es, ts in ((2, 1, 1), (4, 1, 3), (8, 2, 2)):
        cl = ClusterSpec.uniform(dev, rate=100.0, bandwidth=64.0, exec_slots=es,
                                 transfer_slots=ts)
        for k in range(3):
            _batch_vs_oracle(torch_cuda, random_dag(rng, max_vertices=12), cl, 8, 7 * dev + k,
                             wide=True)
    c8b = ClusterSpec.uniform(8, rate=1e9, bandwidth=1e7)
    _batch_vs_oracle(torch_cuda, builders.build_llama_block(), c8b, 16, 3, wide=True)
    _batch_vs_oracle(torch_cuda, builders.sparse_dag(1000, seed=0), c8b, 8, 4, wide=True)


def test_wide_path_large_dags_vs_oracle(torch_cuda):
    """Graphs beyond shared memory take the wide path on their own: 2.5k ops
    (traces bit-exact, 3 strategies) and 6k ops (fifo makespans)."""
    c8b = ClusterSpec.uniform(8, rate=1e9, bandwidth=1e7)
    _batch_vs_oracle(torch_cuda, builders.sparse_dag(2500, seed=1), c8b, 6, 5,
                     check=range(0, 6, 2))
    _batch_vs_oracle(torch_cuda, builders.sparse_dag(6000, seed=2), c8b, 3, 6,
                     strategies=("fifo",), check=[0])


def test_wide_workspace_contract(torch_cuda):
    import ctypes
    from paper_2505_23131_b200 import _native as N
    from paper_2505_23131_b200.simulate import SimProblem
    g = builders.sparse_dag(5000, seed=0)
    prob = SimProblem(g, ClusterSpec.uniform(8, rate=1e9, bandwidth=1e7))
    assert prob.workspace(4) is not None          # beyond shared memory: wide path
    assert SimProblem(builders.build_ffnn(8, 4, 16, 4, 2),
                      ClusterSpec.uniform(8, 1e6, 1e5)).workspace(4) is None
    at = torch_cuda.zeros((4, len(g)), dtype=torch_cuda.int32, device="cuda")
    mk = torch_cuda.empty(4, dtype=torch_cuda.float64, device="cuda")
    st = torch_cuda.empty(4, dtype=torch_cuda.int32, device="cuda")
    rc = N.lib().fp_sim_batch(prob.handle, N.ptr(at), ctypes.c_int32(4), ctypes.c_int32(0),
                              None, ctypes.c_int64(0), N.ptr(mk), N.ptr(st), None,
                              ctypes.c_int32(0), None, None, None, ctypes.c_int64(0),
                              ctypes.c_int32(0), None)
    assert rc == N.FP_ERR_INVALID and b"workspace" in N.lib().fp_last_error()


def test_run_packed_drop_in_large_graph(torch_cuda):
    """The Cython-ABI drop-in (fp_run_packed, _simcore.pyx:39-45) on a graph
    beyond shared memory (the call sizes and frees its own workspace):
    bit-identical event stream to the C oracle, and exec_time agrees."""
    from paper_2505_23131_b200 import simulate as S
    g = builders.sparse_dag(4000, seed=5)
    cl = ClusterSpec.uniform(8, rate=1e9, bandwidth=1e7)
    feats = static_features(g, cl.comm_factor)
    a = np.random.default_rng(2).integers(0, 8, size=len(g)).astype(np.int32)
    packed = osim.pack(g, a, cl, feats, "depth_first", 0)
    omk, oev = osim.run_packed(*packed)
    mk, ev = S.run_packed(*packed)
    assert mk == omk and ev == oev
    mk2, sched = S.exec_time(g, a, cl, "depth_first", 0, feats)
    assert mk2 == omk and len(sched.events) == len(oev)
