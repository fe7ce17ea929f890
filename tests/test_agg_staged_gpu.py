"""GPU: the staged per_step aggregation (gnn_agg_staged_kernel: episode P / Q
slices moved into shared memory by 1-D TMA bulk copies) against the row-gather
kernel it replaces (FP_AGG_STAGED=0) -- the same per-row message order and
arithmetic, so a sampled per_step batch must come out bit-identical (actions,
log-probs, entropies, makespans).  Plus the aggregation timer bench.py uses
(fp_agg_timer_*): one event-timed launch per encode round per decision."""
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
which, out = sys.argv[2], sys.argv[3]
if which == "ffnn":
    g, cl = builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, 1e6, 1e5)
    pc = PolicyConfig(mp_mode="per_step")
else:
    g, cl = builders.build_llama_block(), ClusterSpec.uniform(8, 1e9, 1e7)
    pc = PolicyConfig(mp_mode="per_step")
ctx = PolicyContext(g, cl, pc)
rb = ctx.rollout_batch(init_policy_params(pc, seed=3), 24, 0.2, 11, trace_steps=True)
np.savez(out, vd=rb.step_vd.cpu().numpy(), lp=rb.step_lp.cpu().numpy(),
         ent=rb.step_ent.cpu().numpy(), mk=rb.makespan.cpu().numpy(),
         st=rb.status.cpu().numpy())
"""


def _run(tmp_path, which, staged):
    out = tmp_path / f"{which}_{int(staged)}.npz"
    env = dict(os.environ)
    if not staged:
        env["FP_AGG_STAGED"] = "0"
    subprocess.run([sys.executable, "-c", _SCRIPT, str(ROOT), which, str(out)], env=env,
                   check=True, timeout=600)
    return np.load(out)


@pytest.mark.parametrize("which", ["ffnn", "llama_block"])
def test_staged_aggregation_bit_identical_to_gather(tmp_path, which):
    a, b = _run(tmp_path, which, True), _run(tmp_path, which, False)
    assert (a["st"] == 0).all() and (b["st"] == 0).all()
    for k in ("vd", "lp", "ent", "mk"):
        assert np.array_equal(a[k], b[k]), k


def test_agg_timer_counts_every_aggregation_launch():
    import torch

    from paper_2505_23131_b200 import _native as N
    from paper_2505_23131_b200 import builders
    from paper_2505_23131_b200.cluster import ClusterSpec
    from paper_2505_23131_b200.params import init_policy_params
    from paper_2505_23131_b200.policy import PolicyConfig, PolicyContext

    g, cl = builders.build_ffnn(8, 4, 16, 4, 2), ClusterSpec.uniform(8, 1e6, 1e5)
    pc = PolicyConfig(mp_mode="per_step")
    ctx = PolicyContext(g, cl, pc)
    flat = ctx.flat_params(init_policy_params(pc, seed=0))
    N.agg_timer(True)
    try:
        rb = ctx.rollout_batch(flat, 16, 0.2, 5)
        torch.cuda.synchronize()
        ms, launches = N.agg_timer_read()
    finally:
        N.agg_timer(False)
    assert (rb.status.cpu().numpy() == 0).all()
    assert launches == len(g) * pc.k_rounds  # one launch per round per decision (both encoders)
    assert ms > 0.0
    assert N.agg_timer_read() == (0.0, 0)  # read resets
