"""Scaling sweep (BASELINE config 5): sparse random DAGs 1k-100k ops x episode
batches, one B200.  Per point: GNN encode + head tables (prepare), the fused
rollout + simulation launch, and the simulator alone on the same
assignments, each timed with CUDA events after warm-up.

    python tools/sweep.py [--sizes 1000,4000,10000,30000,100000] [--batch 1024]
                          [--reps 3] [--out gpurun_out/sweep.jsonl]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2505_23131_b200 import builders  # noqa: E402
from paper_2505_23131_b200.cluster import ClusterSpec  # noqa: E402
from paper_2505_23131_b200.params import init_policy_params  # noqa: E402
from paper_2505_23131_b200.policy import PolicyConfig, PolicyContext  # noqa: E402


def timed(fn, reps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        ms.append(ev[0].elapsed_time(ev[1]))
    return min(ms), sum(ms) / len(ms)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1000,4000,10000,30000,100000")
    ap.add_argument("--batch", default="1024")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--wide", action="store_true", help="force the HBM-resident path")
    ap.add_argument("--out", default="gpurun_out/sweep.jsonl")
    a = ap.parse_args()
    Path(a.out).parent.mkdir(exist_ok=True)
    cl = ClusterSpec.uniform(8, rate=1e9, bandwidth=1e7)
    pc = PolicyConfig()
    params = init_policy_params(pc, seed=0)
    for n in [int(x) for x in a.sizes.split(",")]:
        t0 = time.perf_counter()
        g = builders.sparse_dag(n, seed=0)
        ctx = PolicyContext(g, cl, pc)
        host_s = time.perf_counter() - t0
        flat = ctx.flat_params(params)
        for B in [int(x) for x in a.batch.split(",")]:
            out = ctx.alloc_batch(B)
            enc_ms, _ = timed(lambda: ctx.prepare(flat), a.reps)
            ws = ctx.workspace(B, wide=a.wide)
            ro_min, ro_avg = timed(lambda: ctx.rollout_batch(flat, B, 0.2, 7, out=out,
                                                             prepare=False, wide=a.wide),
                                   a.reps)
            st = out.status.cpu()
            assert bool((st == 0).all()), "episode failures"
            sim_min, _ = timed(lambda: ctx.sim.simulate(out.assign, "fifo", wide=a.wide), a.reps)
            rec = {"n": n, "edges": len(g.edges), "B": B, "wide": ws is not None,
                   "workspace_mb": 0 if ws is None else ws.numel() / 2 ** 20,
                   "encode_ms": enc_ms, "rollout_ms": ro_min, "rollout_avg_ms": ro_avg,
                   "episodes_per_s": B / (ro_min * 1e-3), "sim_only_ms": sim_min,
                   "sims_per_s": B / (sim_min * 1e-3), "host_setup_s": host_s,
                   "forest": ctx.forest}
            print(json.dumps(rec), flush=True)
            with open(a.out, "a") as f:
                f.write(json.dumps(rec) + "\n")
        del ctx
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
