"""Phase cycles of the Stage-II replay kernel (profiling build).

    python -m paper_2505_23131_b200._build --profile
    python tools/replay_profile.py [--workload llama_layer] [--batch 1024]
"""
import argparse
import ctypes
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ["FLOWPLACE_B200_LIB"] = str(ROOT / "paper_2505_23131_b200" / "_flowplace_b200_prof.so")

import torch  # noqa: E402

from bench import workload  # noqa: E402
from paper_2505_23131_b200 import _native as N  # noqa: E402
from paper_2505_23131_b200.params import init_policy_params  # noqa: E402
from paper_2505_23131_b200.policy import PolicyConfig, PolicyContext  # noqa: E402
from paper_2505_23131_b200.training import BatchedTrainer, TrainConfig  # noqa: E402

NAMES = {25: "pass0 (records -> smem)", 26: "PLC adjoints", 27: "SEL pass 1 (qp, c1)",
         28: "SEL pass 2 (ds)", 29: "PLC prefix S_d", 30: "PLC chunk replay", 31: "CTA end"}
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="llama_layer")
ap.add_argument("--batch", type=int, default=1024)
a = ap.parse_args()
g, cl, _ = workload(a.workload)
pc = PolicyConfig()
ctx = PolicyContext(g, cl, pc)
tr = BatchedTrainer(ctx, init_policy_params(pc, 0), TrainConfig(episodes=10 ** 6), batch_size=a.batch)
lib = N.lib()
cyc = (ctypes.c_ulonglong * 64)()
cnt = (ctypes.c_ulonglong * 64)()
for i in range(3):
    tr.step(seed=100 + i)
torch.cuda.synchronize()
lib.fp_phase_read_grad(cyc, cnt, 1)
tr.step(seed=999)
torch.cuda.synchronize()
lib.fp_phase_read_grad(cyc, cnt, 1)
for i, name in NAMES.items():
    if cnt[i]:
        print(f"  {name:28s} {cyc[i] / cnt[i]:10.0f} cyc per warp (calls {cnt[i]})")
