"""GNN encode (aggregation + node MLPs + head tables) on large sparse DAGs, for
ncu launch lists and CUDA-event timing of fp_policy_prepare.

    python tools/encode_profile.py [--n 1000000] [--reps 5]
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

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1000000)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--shuffle", action="store_true", help="random vertex ids (no gather locality)")
ap.add_argument("--encoder", default="dmma", choices=("dmma", "tc", "fused"))
a = ap.parse_args()
t0 = time.perf_counter()
g = builders.sparse_dag(a.n, seed=0)
if a.shuffle:
    g = builders.relabel(g, seed=1)
cl = ClusterSpec.uniform(8, rate=1e9, bandwidth=1e7)
pc = PolicyConfig()
ctx = PolicyContext(g, cl, pc)
ctx.set_encoder(a.encoder)
flat = ctx.flat_params(init_policy_params(pc, seed=0))
setup = time.perf_counter() - t0
ctx.prepare(flat)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ms = []
for _ in range(a.reps):
    ev[0].record()
    ctx.prepare(flat)
    ev[1].record()
    torch.cuda.synchronize()
    ms.append(ev[0].elapsed_time(ev[1]))
print(json.dumps({"n": a.n, "edges": len(g.edges), "shuffle": a.shuffle, "encoder": a.encoder, "prepare_ms_min": min(ms),
                  "prepare_ms": ms, "host_setup_s": setup}))
