"""Simulator-only launches (fp_sim_batch) for ncu captures and CUDA-event
timing: B random assignments of a bench workload.

    python tools/sim_profile.py [--workload ffnn] [--batch 1024] [--reps 5]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import workload  # noqa: E402
from paper_2505_23131_b200.simulate import SimProblem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="ffnn")
ap.add_argument("--batch", type=int, default=1024)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
g, cl, desc = workload(a.workload)
prob = SimProblem(g, cl)
rng = np.random.default_rng(0)
assign = torch.from_numpy(rng.integers(0, cl.device_count, size=(a.batch, len(g)))
                          .astype(np.int32)).cuda()
out = prob.simulate(assign, "fifo")
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ms = []
for _ in range(a.reps):
    ev[0].record()
    out = prob.simulate(assign, "fifo")
    ev[1].record()
    torch.cuda.synchronize()
    ms.append(ev[0].elapsed_time(ev[1]))
assert bool((out["status"] == 0).all())
n, E = len(g), len(g.edges)
alg = a.batch * (4 * n + 12) + (n + 1) * 8 + E * 8 + 16 * n
print(json.dumps({"workload": desc, "B": a.batch, "ms": min(ms), "sims_per_s": a.batch / min(ms) * 1e3,
                  "alg_bytes": alg, "alg_GBps": alg / (min(ms) * 1e-3) / 1e9}))
