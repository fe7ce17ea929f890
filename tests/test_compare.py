"""compare (reference cli.py:316-366 evaluate loop + metrics.py) against the
reference's own outputs (tests/golden/compare_cases.json, made by
tests/golden/make_compare_golden.py)."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2505_23131_b200 import builders
from paper_2505_23131_b200.cluster import ClusterSpec
from paper_2505_23131_b200.compare import average_ranks, pearson, spearman
from paper_2505_23131_b200.heuristics import random_assign, single_device_assign

GOLD = json.loads((Path(__file__).parent / "golden" / "compare_cases.json").read_text())
BUILD = {"ffnn64": lambda: builders.build_ffnn(8, 4, 16, 4, 2),
         "chainmm": lambda: builders.build_chainmm(64, 2)}


def _case(c):
    g = BUILD[c["builder"]]()
    cl = ClusterSpec.uniform(c["devices"], rate=1e6, bandwidth=1e5)
    return g, cl, [(r["engine"], r["assignment"]) for r in c["rows"]]


def test_metrics_known_answers():
    for m in GOLD["metrics"]:
        assert pearson(m["x"], m["y"]) == m["pearson"]
        assert spearman(m["x"], m["y"]) == m["spearman"]
    assert average_ranks([3.0, 1.0, 3.0, 2.0]).tolist() == [3.5, 1.0, 3.5, 2.0]
    with pytest.raises(ValueError, match="at least two"):
        pearson([1.0], [2.0])
    with pytest.raises(ValueError, match="constant"):
        pearson([1.0, 1.0], [2.0, 3.0])
    with pytest.raises(ValueError, match="equal-length"):
        pearson([1.0, 2.0], [2.0, 3.0, 4.0])


def test_compare_assignments_are_the_reference_ones():
    for c in GOLD["cases"]:
        g, cl, pairs = _case(c)
        want = {name: a for name, a in pairs}
        assert list(single_device_assign(g)) == want["single"]
        assert list(random_assign(g, cl.device_count, seed=c["seed"])) == want["random"]
        for k in range(3):
            assert list(random_assign(g, cl.device_count, seed=c["seed"] + 1000 + k)) == \
                want[f"probe_{k}"]


@pytest.mark.gpu
def test_compare_rows_bit_exact_with_reference():
    from paper_2505_23131_b200.compare import compare_assignments
    for c in GOLD["cases"]:
        g, cl, pairs = _case(c)
        got = compare_assignments(g, cl, pairs, c["trials"], c["jitter_sigma"], c["seed"],
                                  c["strategy"])
        for r, w in zip(got["rows"], c["rows"]):
            assert r["engine"] == w["engine"]
            assert r["clean_ms"] == w["clean_ms"], (c["tag"], r["engine"])
            assert r["noisy_mean_ms"] == w["noisy_mean_ms"], (c["tag"], r["engine"])
            assert r["noisy_std_ms"] == w["noisy_std_ms"], (c["tag"], r["engine"])
        assert got["pearson"] == c["pearson"] and got["spearman"] == c["spearman"]


@pytest.mark.gpu
def test_compare_engines_end_to_end():
    from paper_2505_23131_b200.compare import compare
    from paper_2505_23131_b200.params import init_policy_params
    from paper_2505_23131_b200.policy import PolicyConfig
    from paper_2505_23131_b200.simulate import exec_time

    g = builders.build_ffnn(8, 4, 16, 4, 2)
    cl = ClusterSpec.uniform(8, rate=1e6, bandwidth=1e5)
    pc = PolicyConfig(hidden=16, k_rounds=1)
    doc = compare(g, cl, engines=("critical_path", "random", "single", "doppler"), trials=5,
                  probe_assignments=2, jitter_sigma=0.1, seed=2,
                  params=init_policy_params(pc, seed=1), pconfig=pc)
    names = [r["engine"] for r in doc["rows"]]
    assert names == ["critical_path", "random", "single", "doppler", "probe_0", "probe_1"]
    # the single-device row re-derived through the per-call drop-in API
    single = doc["rows"][2]
    assert single["clean_ms"] == exec_time(g, single_device_assign(g), cl)[0]
    jc = ClusterSpec.from_dict({**cl.to_dict(), "jitter_sigma": 0.1})
    noisy = [exec_time(g, single_device_assign(g), jc, seed=2 + t)[0] for t in range(5)]
    assert single["noisy_mean_ms"] == float(np.mean(noisy))
    assert -1.0 <= doc["pearson"] <= 1.0 and -1.0 <= doc["spearman"] <= 1.0
    with pytest.raises(ValueError, match="unknown engine"):
        compare(g, cl, engines=("nope",))


@pytest.mark.gpu
def test_compare_clean_run_uses_the_clusters_own_jitter():
    """cli.py:339: the clean column is exec_time on the cluster as given (its
    own jitter_sigma, seed 0); the noisy ones use --jitter-sigma."""
    from paper_2505_23131_b200.compare import compare_assignments
    from paper_2505_23131_b200.simulate import exec_time
    g = builders.build_ffnn(8, 4, 16, 4, 2)
    cl = ClusterSpec.from_dict({**ClusterSpec.uniform(8, rate=1e6, bandwidth=1e5).to_dict(),
                                "jitter_sigma": 0.05})
    pairs = [(f"r{k}", list(random_assign(g, 8, seed=k))) for k in range(3)]
    doc = compare_assignments(g, cl, pairs, trials=2, jitter_sigma=0.3, seed=9)
    for (name, a), row in zip(pairs, doc["rows"]):
        assert row["clean_ms"] == exec_time(g, a, cl, seed=0)[0]
        jc = ClusterSpec.from_dict({**cl.to_dict(), "jitter_sigma": 0.3})
        assert row["noisy_mean_ms"] == float(np.mean([exec_time(g, a, jc, seed=9 + t)[0]
                                                      for t in range(2)]))
