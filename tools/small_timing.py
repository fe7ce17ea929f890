"""Phase cycles of the small-graph encoder (profiling build, -DFP_SMALL_TIMING)."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ["FLOWPLACE_B200_LIB"] = str(ROOT / "paper_2505_23131_b200" / "_flowplace_b200_prof.so")
import torch  # noqa: E402

from bench import workload  # noqa: E402
from paper_2505_23131_b200.params import init_policy_params  # noqa: E402
from paper_2505_23131_b200.policy import PolicyConfig, PolicyContext  # noqa: E402

g, cl, _ = workload(sys.argv[1] if len(sys.argv) > 1 else "ffnn")
pc = PolicyConfig()
ctx = PolicyContext(g, cl, pc)
flat = ctx.flat_params(init_policy_params(pc, 0))
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for i in range(4):
    flush.fill_(i)
    ctx.prepare(flat)
    torch.cuda.synchronize()
