"""CPU: the C oracle simulator against event streams dumped from the reference
(tests/golden/sim_cases.json, made by tests/golden/make_golden.py)."""
import numpy as np
import pytest

from helpers import graph_from_golden
from oracle import sim as osim
from paper_2505_23131_b200.cluster import ClusterSpec


def test_oracle_matches_every_reference_event_stream(sim_golden):
    assert len(sim_golden) >= 150
    for c in sim_golden:
        g = graph_from_golden(c["graph"])
        cl = ClusterSpec.from_dict(c["cluster"])
        if "deadlock" in c:
            with pytest.raises(osim.OracleDeadlock) as ei:
                osim.exec_time(g, c["assign"], cl, c["strategy"], c["seed"])
            assert ei.value.time_ms == c["deadlock"]["time"]
            assert ei.value.blocked == c["deadlock"]["blocked"]
            continue
        mk, ev = osim.exec_time(g, c["assign"], cl, c["strategy"], c["seed"])
        assert mk == c["makespan"], c["tag"]
        assert [list(e) for e in ev] == c["events"], c["tag"]


def test_oracle_mix64_and_jitter_known_answers():
    # tests/test_cluster.py:42-45 of the reference
    from paper_2505_23131_b200.cluster import jitter_factor, mix64
    assert mix64(0) == 16294208416658607535
    assert mix64(123456789) == 2466975172287755897
    lib = osim.lib()
    for seed in range(5):
        for kind in (0, 1):
            a = lib.oracle_jitter_factor(seed, kind, 3, 1, 0 if kind == 0 else 2, 0.2)
            assert a == jitter_factor(seed, kind, 3, 1, 0 if kind == 0 else 2, 0.2)


def test_oracle_arithmetic_pins():
    # tests/test_simulator.py:26-57 of the reference
    from helpers import chain_graph, cluster2
    mk, _ = osim.exec_time(chain_graph((1000, 2000)), [0, 0, 0], cluster2(rate=100.0))
    assert mk == 30.0
    mk, ev = osim.exec_time(chain_graph((1000, 2000), bytes_=100), [0, 0, 1],
                            cluster2(rate=100.0, bandwidth=800.0))
    assert mk == 30.5 and any(e[0] == 1 for e in ev)
