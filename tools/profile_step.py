"""Run a few hot-path steps for ncu capture (not a bench: numbers printed
under a profiler are never reported).

    python tools/profile_step.py [--workload ffnn] [--batch 1024] [--steps 2] [--nosim]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import EPSILON, workload  # noqa: E402
from paper_2505_23131_b200.params import init_policy_params  # noqa: E402
from paper_2505_23131_b200.policy import PolicyConfig, PolicyContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="ffnn")
ap.add_argument("--batch", type=int, default=1024)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--nosim", action="store_true")
ap.add_argument("--grad", action="store_true")
a = ap.parse_args()
g, cl, _ = workload(a.workload)
pc = PolicyConfig()
ctx = PolicyContext(g, cl, pc)
flat = ctx.flat_params(init_policy_params(pc, 0))
out = ctx.alloc_batch(a.batch, grad=a.grad, simulate=not a.nosim)
for i in range(a.steps):
    ctx.rollout_batch(flat, a.batch, EPSILON, 100 + i, out=out, simulate=not a.nosim)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
ctx.rollout_batch(flat, a.batch, EPSILON, 999, out=out, simulate=not a.nosim, prepare=False)
ev[1].record()
torch.cuda.synchronize()
print("rollout launch ms", ev[0].elapsed_time(ev[1]))
