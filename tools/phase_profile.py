"""Per-phase cycle breakdown of the rollout kernel (profiling build).

    python -m paper_2505_23131_b200._build --profile
    python tools/phase_profile.py [--workload ffnn] [--batch 1024]
"""
import argparse
import ctypes
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ["FLOWPLACE_B200_LIB"] = str(ROOT / "paper_2505_23131_b200" / "_flowplace_b200_prof.so")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import EPSILON, workload  # noqa: E402
from paper_2505_23131_b200 import _native as N  # noqa: E402
from paper_2505_23131_b200.params import init_policy_params  # noqa: E402
from paper_2505_23131_b200.policy import PolicyConfig, PolicyContext  # noqa: E402

NAMES = {0: "sel.compact", 1: "sel.softmax", 2: "sel.decide+publish", 3: "sel.lp/ent",
         4: "sel.cand-update", 5: "sel.tree-decide", 6: "sel.publish+lp", 7: "sel.tree-update", 10: "plc.wait-order", 11: "plc.features", 12: "plc.stats+xn",
         13: "plc.preact+reduce", 14: "plc.softmax", 15: "plc.decide", 16: "plc.lp/grad",
         17: "plc.commit", 21: "sim.start", 22: "sim.wait-placed", 23: "sim.tmin", 24: "sim.complete"}
MARKS = {40: "SEL chain done", 41: "PLC chain done", 42: "simulation done"}

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="ffnn")
ap.add_argument("--batch", type=int, default=1024)
ap.add_argument("--grad", action="store_true")
a = ap.parse_args()
g, cl, _ = workload(a.workload)
pc = PolicyConfig()
ctx = PolicyContext(g, cl, pc)
flat = ctx.flat_params(init_policy_params(pc, 0))
out = ctx.alloc_batch(a.batch, grad=a.grad)
lib = N.lib()
cyc = (ctypes.c_ulonglong * 64)()
cnt = (ctypes.c_ulonglong * 64)()
for i in range(3):
    ctx.rollout_batch(flat, a.batch, EPSILON, 100 + i, out=out)
torch.cuda.synchronize()
lib.fp_phase_read(cyc, cnt, 1)
lib.fp_phase_read_wide(cyc, cnt, 1)
lib.fp_phase_read_grad(cyc, cnt, 1)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
ctx.rollout_batch(flat, a.batch, EPSILON, 999, out=out, prepare=False)
ev[1].record()
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1])
lib.fp_phase_read(cyc, cnt, 1)
cyc2 = (ctypes.c_ulonglong * 64)()
cnt2 = (ctypes.c_ulonglong * 64)()
for rd in (lib.fp_phase_read_wide, lib.fp_phase_read_grad):
    rd(cyc2, cnt2, 1)
    for i in range(64):  # wide / grad kernels' counters live in their own TUs
        cyc[i] += cyc2[i]
        cnt[i] += cnt2[i]
print(f"{a.workload}: rollout+sim launch {ms:.3f} ms (instrumented)")
tot = {"sel": 0, "plc": 0, "sim": 0}
for i in sorted(NAMES):
    if cnt[i]:
        per = cyc[i] / cnt[i]
        tot[NAMES[i].split(".")[0]] += cyc[i] / a.batch
        print(f"  {NAMES[i]:22s} {per:8.1f} cyc/call  calls/episode {cnt[i] / a.batch:7.1f}"
              f"  total/episode {cyc[i] / a.batch:10.0f}")
print("  per-episode cycles:", {k: int(v) for k, v in tot.items()})
for i, name in MARKS.items():
    if cnt[i]:
        print(f"  milestone {name:18s} {cyc[i] / cnt[i]:10.0f} cycles after the block start")
