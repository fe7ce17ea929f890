"""Small invocations of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): the compact rollout (sampled,
traced, teacher), the wide HBM-state rollout, per_step message passing, a
REINFORCE rollout + replay + backward + SGD, and the simulator alone.

    compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_23131_b200 import builders  # noqa: E402
from paper_2505_23131_b200.cluster import ClusterSpec  # noqa: E402
from paper_2505_23131_b200.params import init_policy_params  # noqa: E402
from paper_2505_23131_b200.policy import PolicyConfig, PolicyContext  # noqa: E402
from paper_2505_23131_b200.simulate import SimProblem  # noqa: E402
from paper_2505_23131_b200.training import BatchedTrainer, TrainConfig  # noqa: E402

g = builders.build_ffnn(4, 2, 8, 2, 2)
cl = ClusterSpec.uniform(4, rate=1e6, bandwidth=1e5)
pc = PolicyConfig(hidden=16)
params = init_policy_params(pc, seed=0)
ctx = PolicyContext(g, cl, pc)
B = 4
ctx.rollout_batch(params, B, 0.2, 1)                                   # compact, lean
ctx.rollout_batch(params, B, 0.2, 2, trace_steps=True, sim_trace=True)  # compact, outputs
ctx.rollout_batch(params, B, 0.0, 3, mode="teacher", tie_random=True)
ctx.rollout_batch(params, B, 0.2, 4, wide=True)                        # wide (HBM state)
tr = BatchedTrainer(ctx, params, TrainConfig(episodes=64), batch_size=B)
tr.step(seed=5)                                                        # REINFORCE + replay
tr.check()
prob = SimProblem(g, cl)
a = np.random.default_rng(0).integers(0, 4, size=(B, len(g))).astype(np.int32)
prob.simulate(torch.from_numpy(a).cuda(), "fifo")
ps = PolicyContext(g, cl, PolicyConfig(hidden=16, mp_mode="per_step"))
ps.rollout_batch(params, 2, 0.2, 6)                                    # per_step
torch.cuda.synchronize()
print("sanitize workload done")
# round-2 additions: per_step staged aggregation under the bf16 encoder too,
# and a > 64-op graph so the PDL-chained multi-kernel encode + rollout and the
# PDL backward / replay / SGD chain run
ps.set_encoder("tc")
ps.rollout_batch(params, 2, 0.2, 7)                                    # per_step, tc + staged
gl = builders.build_llama_block()
cll = ClusterSpec.uniform(8, rate=1e9, bandwidth=1e7)
pcl = PolicyConfig()
pl = init_policy_params(pcl, seed=0)
cx = PolicyContext(gl, cll, pcl)
cx.rollout_batch(pl, 2, 0.2, 8)                                        # PDL encode chain + rollout
trl = BatchedTrainer(cx, pl, TrainConfig(episodes=64), batch_size=2)
trl.step(seed=9)                                                       # PDL backward chain
trl.check()
torch.cuda.synchronize()
print("sanitize workload done")
