"""CPU, world_size 2 (gloo): the trainer's multi-rank update rule — one
allreduce of [grad | sum returns], global running-mean baseline, alpha — equals
the single-process computation over the union of the ranks' episodes."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from paper_2505_23131_b200.training import GlobalUpdate

B, NP = 4, 7


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data(rank, step):
    rng = np.random.default_rng(100 * step + rank)
    return rng.uniform(1, 10, size=B), rng.normal(size=NP)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    upd = GlobalUpdate(NP, B, world=world, device="cpu")
    alpha = torch.empty(B, dtype=torch.float64)
    res = []
    for step in range(3):
        mk, g = _data(rank, step)
        mk_t = torch.tensor(mk)
        upd.alpha(mk_t, alpha)
        upd.grad.copy_(torch.tensor(g))
        upd.finish(mk_t)
        res.append((alpha.numpy().copy(), upd.grad.numpy().copy(), float(upd.ret_sum.item()),
                    upd.count))
    q.put((rank, res))
    dist.destroy_process_group()


def test_two_rank_update_matches_single_process():
    world = 2
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process restatement over the union of episodes
    ret_sum, count = 0.0, 0
    for step in range(3):
        mks = [_data(r, step)[0] for r in range(world)]
        grads = [_data(r, step)[1] for r in range(world)]
        base = ret_sum / count if count else 0.0
        for r in range(world):
            a, g, rs, c = out[r][step]
            np.testing.assert_allclose(a, (mks[r] + base) / (B * world), rtol=1e-15)
            np.testing.assert_allclose(g, grads[0] + grads[1], rtol=1e-15)
        ret_sum += -sum(m.sum() for m in mks)
        count += B * world
        for r in range(world):
            assert abs(out[r][step][2] - ret_sum) < 1e-12 and out[r][step][3] == count
