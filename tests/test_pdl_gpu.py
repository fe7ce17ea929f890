"""GPU: programmatic dependent launch changes scheduling only.  The same
Llama-block sampled rollout (PDL-chained multi-kernel encode + rollout) and
the same Stage-II update (PDL-chained replay, backward and SGD) with PDL on
and off (FP_PDL=0) must give bit-identical actions, log-probs, makespans and
updated parameters."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2505_23131_b200 import builders
from paper_2505_23131_b200.cluster import ClusterSpec
from paper_2505_23131_b200.params import init_policy_params
from paper_2505_23131_b200.policy import PolicyConfig, PolicyContext
from paper_2505_23131_b200.training import BatchedTrainer, TrainConfig
g, cl = builders.build_llama_block(), ClusterSpec.uniform(8, 1e9, 1e7)
pc = PolicyConfig()
ctx = PolicyContext(g, cl, pc)
params = init_policy_params(pc, seed=4)
rb = ctx.rollout_batch(params, 64, 0.2, 13, trace_steps=True)
tr = BatchedTrainer(ctx, params, TrainConfig(episodes=10 ** 6), batch_size=32)
for s in range(2):
    tr.step(seed=100 + s)
tr.check()
np.savez(sys.argv[2], vd=rb.step_vd.cpu().numpy(), lp=rb.step_lp.cpu().numpy(),
         mk=rb.makespan.cpu().numpy(), st=rb.status.cpu().numpy(),
         flat=tr.flat.cpu().numpy())
"""


def _run(tmp_path, pdl):
    out = tmp_path / f"pdl_{int(pdl)}.npz"
    env = dict(os.environ)
    if not pdl:
        env["FP_PDL"] = "0"
    subprocess.run([sys.executable, "-c", _SCRIPT, str(ROOT), str(out)], env=env, check=True,
                   timeout=600)
    return np.load(out)


def test_pdl_on_off_bit_identical(tmp_path):
    a, b = _run(tmp_path, True), _run(tmp_path, False)
    assert (a["st"] == 0).all() and (b["st"] == 0).all()
    for k in ("vd", "lp", "mk", "flat"):
        assert np.array_equal(a[k], b[k]), k
