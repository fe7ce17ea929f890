"""Config-5 golden vectors at 10k ops from the ORACLE (oracle/policy.py +
oracle/wc_sim.c, themselves pinned against the reference's goldens at small
sizes: tests/test_oracle*.py).  A 10k-op oracle rollout takes ~2 min of numpy,
too slow for the GPU box's test run, so its outputs are committed:

    python tests/golden/make_dag10k_golden.py

Writes tests/golden/dag10k.npz: sparse_dag(10000, seed=0), 8 devices
(rate 1e9, bandwidth 1e7), policy hidden 32 / K 2 init seed 0, epsilon 0.2,
Philox seed 31; for episodes EPISODES of that stream: every step's (vertex,
device), the log-probs / entropies of every 7th step, and the makespan.
"""

from __future__ import annotations

import multiprocessing as mp
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
EPISODES = (0, 777)
SEED, EPS, N = 31, 0.2, 10_000


def _one(ep):
    sys.path.insert(0, str(ROOT))
    from oracle import policy as OP
    from oracle import sim as osim
    from paper_2505_23131_b200 import builders
    from paper_2505_23131_b200.cluster import ClusterSpec
    from paper_2505_23131_b200.params import init_policy_params
    from paper_2505_23131_b200.policy import PolicyConfig
    g, cl = builders.sparse_dag(N, seed=0), ClusterSpec.uniform(8, 1e9, 1e7)
    pc = PolicyConfig()
    octx = OP.Ctx(g, cl, pc.hidden, pc.k_rounds, pc.leaky_slope, pc.shared_encoder)
    ro = OP.rollout(OP.leaves(init_policy_params(pc, seed=0), need=False), octx, EPS,
                    mode="uniform", seed=SEED, episode=ep)
    mk, _ = osim.exec_time(g, ro["assign"], cl)
    vd = np.array([(s["vertex"], s["device"]) for s in ro["steps"]], dtype=np.uint16)
    lp = np.array([(s["sel_logprob"], s["plc_logprob"], s["sel_entropy"], s["plc_entropy"])
                   for s in ro["steps"][::7]])
    return vd, lp, mk


def main():
    with mp.get_context("spawn").Pool(len(EPISODES)) as pool:
        res = pool.map(_one, EPISODES)
    np.savez_compressed(HERE / "dag10k.npz", episodes=np.array(EPISODES),
                        vd=np.stack([r[0] for r in res]), lp_ent=np.stack([r[1] for r in res]),
                        makespan=np.array([r[2] for r in res]), seed=SEED, epsilon=EPS)
    print("dag10k.npz:", [r[2] for r in res])


if __name__ == "__main__":
    main()
