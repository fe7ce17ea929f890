"""GPU, two ranks on one device (gloo carries the CUDA gradient buffer): the
full multi-rank Stage-II step -- sharded episodes (episode_base = rank * B),
REINFORCE rows, deterministic reduction, backward, the single allreduce of
[grad | sum of returns], global baseline, SGD -- equals one process running
the union batch.  (NCCL refuses two ranks on one GPU; the pool gives one.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

pytestmark = pytest.mark.gpu
B, STEPS = 8, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    from paper_2505_23131_b200 import builders
    from paper_2505_23131_b200.cluster import ClusterSpec
    from paper_2505_23131_b200.params import init_policy_params
    from paper_2505_23131_b200.policy import PolicyConfig, PolicyContext
    from paper_2505_23131_b200.training import TrainConfig
    g, cl = builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, 1e6, 1e5)
    pc = PolicyConfig(hidden=16, k_rounds=2)
    cfg = TrainConfig(episodes=64, lr0=1e-2, lr1=1e-4, seed=0)
    return PolicyContext(g, cl, pc), init_policy_params(pc, seed=1), cfg


def _run(world, rank, batch, group=None):
    from paper_2505_23131_b200.training import BatchedTrainer
    ctx, params, cfg = _setup()
    tr = BatchedTrainer(ctx, params, cfg, batch_size=batch, world=world, rank=rank, group=group)
    for s in range(STEPS):
        tr.step(seed=100 + s)
    torch.cuda.synchronize()
    return tr.flat.cpu().numpy(), float(tr.upd.ret_sum.item()), tr.upd.count


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q.put((rank, _run(world, rank, B)))
    dist.destroy_process_group()


def test_two_rank_training_matches_union_batch():
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = _run(1, 0, 2 * B)
    f0, f1 = res[0][0], res[1][0]
    assert np.array_equal(f0, f1)                       # identical SGD on every rank
    assert res[0][2] == res[1][2] == single[2] == STEPS * 2 * B
    assert abs(res[0][1] - single[1]) <= 1e-12 * abs(single[1])  # global returns
    np.testing.assert_allclose(f0, single[0], rtol=1e-9, atol=1e-12)
    assert not np.allclose(f0, _setup()[0].flat_params(_setup()[1]).cpu().numpy())
