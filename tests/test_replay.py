"""CPU: the event-driven replay checker (reference simulate.py:346-420
invariants) accepts every reference event stream and flags corrupted ones;
utilization_report (simulate.py:314-343) on a hand-checkable schedule."""
import copy

import pytest

from helpers import cluster2, graph_from_golden
from paper_2505_23131_b200.cluster import ClusterSpec
from paper_2505_23131_b200.replay import replay_violations, utilization_report


def _cases(sim_golden):
    for c in sim_golden:
        if "deadlock" in c or c["cluster"].get("jitter_sigma", 0.0) > 0:
            continue
        yield (graph_from_golden(c["graph"]), ClusterSpec.from_dict(c["cluster"]), c)


def test_reference_streams_replay_clean(sim_golden):
    k = 0
    for g, cl, c in _cases(sim_golden):
        ev = [tuple(e) for e in c["events"]]
        assert replay_violations(g, c["assign"], cl, ev, c["makespan"]) == [], c["tag"]
        k += 1
    assert k > 50


def test_corrupted_streams_are_flagged(sim_golden):
    g, cl, c = next((x for x in _cases(sim_golden) if len(x[2]["events"]) >= 8))
    ev = [tuple(e) for e in c["events"]]
    # drop an end: incomplete + dangling/overflow downstream
    bad = ev[:-1]
    assert replay_violations(g, c["assign"], cl, bad, c["makespan"])
    # delay the first start: idle advance with a startable task
    first = list(ev[0])
    bad = [tuple(first[:4] + [first[4] + 1.0, 0])] + ev[1:]
    out = replay_violations(g, c["assign"], cl, sorted(bad, key=lambda e: e[4]), c["makespan"])
    assert any(m.startswith(("work-conservation", "time-order", "invalid-start")) for m in out)
    # wrong makespan
    assert any(m.startswith("makespan-mismatch")
               for m in replay_violations(g, c["assign"], cl, ev, c["makespan"] + 1.0))


def test_utilization_report_hand_case():
    from helpers import chain_graph
    g = chain_graph((1000, 1000, 1000))
    cl = cluster2(rate=100.0, bandwidth=64.0)
    # all on device 0: three 10 ms execs back to back
    ev = []
    for i, v in enumerate((1, 2, 3)):
        ev += [(0, v, 0, -1, 10.0 * i, 0), (0, v, 0, -1, 10.0 * (i + 1), 1)]
    rep = utilization_report(ev, cl, 30.0)
    assert rep["devices"][0]["busy_ms"] == 30.0 and rep["devices"][0]["busy_fraction"] == 1.0
    assert rep["devices"][1]["busy_ms"] == 0.0 and rep["links"] == []
    assert replay_violations(g, [0, 0, 0, 0], cl, ev, 30.0) == []


@pytest.mark.gpu
def test_100k_op_episode_replays_clean():
    """Size-independent parity at the sweep's largest graph: a 100k-op
    sampled episode from the wide (HBM-resident) kernel, its full event
    stream (~10^6 events) replayed against the work-conserving rules."""
    from paper_2505_23131_b200 import builders
    from paper_2505_23131_b200.params import init_policy_params
    from paper_2505_23131_b200.policy import PolicyConfig, PolicyContext
    from paper_2505_23131_b200.simulate import decode_events
    g = builders.sparse_dag(100000, seed=0)
    cl = ClusterSpec.uniform(8, rate=1e9, bandwidth=1e7)
    pc = PolicyConfig()
    ctx = PolicyContext(g, cl, pc)
    rb = ctx.rollout_batch(init_policy_params(pc, 0), 2, 0.2, 11, sim_trace=True)
    assert rb.status.cpu().numpy().tolist() == [0, 0]
    a = rb.assign.cpu().numpy()
    mk = rb.makespan.cpu().numpy()
    tr = rb.trace.cpu().numpy()
    tl = rb.trace_len.cpu().numpy()
    for b in range(2):
        ev = decode_events(tr[b], int(tl[b]))
        assert len(ev) > 2 * len(g)
        assert replay_violations(g, a[b], cl, ev, float(mk[b])) == []
