"""CPU: host-side mirror of the reference API (builders, features, JSON) and
the C-ABI library surface (loads, exports every symbol include/*.h declares)."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2505_23131_b200 import builders, graph as G
from paper_2505_23131_b200.features import static_features

ROOT = Path(__file__).resolve().parent.parent


def test_builder_golden_counts():
    # reference tests/test_builders.py:74-117
    g = builders.build_chainmm(8, 2)
    assert (len(g), len(g.edges), len(g.meta_ops)) == (60, 80, 4)
    g = builders.build_ffnn(8, 4, 16, 4, 2)
    assert (len(g), len(g.edges), len(g.meta_ops)) == (64, 92, 9)
    assert len(builders.build_chainmm(8, 1)) == 9
    assert len(builders.build_ffnn(8, 4, 16, 4, 1)) == 14


def test_llama_builders_golden_counts():
    b = builders.build_llama_block()
    assert (len(b), len(b.edges), len(b.meta_ops), len(b.entry_vertices())) == (208, 324, 27, 36)
    layer = builders.build_llama_layer()
    assert (len(layer), len(layer.edges), len(layer.meta_ops)) == (248, 392, 35)
    for g in (b, layer):
        assert G.validate(g) == []
        assert G.graph_from_dict(G.graph_to_dict(g)).edges == g.edges


def test_builders_match_reference_graphs(sim_golden):
    want = {c["tag"].split("#")[0]: c["graph"] for c in sim_golden
            if c["tag"].startswith(("chainmm60", "ffnn64"))}
    assert G.graph_to_dict(builders.build_chainmm(64, 2)) == want["chainmm60"]
    assert G.graph_to_dict(builders.build_ffnn(8, 4, 16, 4, 2)) == want["ffnn64"]


def test_sparse_dag_is_valid_and_sparse():
    g = builders.sparse_dag(2000, seed=0)
    assert G.validate(g) == []
    assert len(g.edges) < 2.1 * len(g)
    assert len(g.entry_vertices()) == 100


def test_graph_json_errors():
    with pytest.raises(G.GraphFormatError, match="missing field: edges"):
        G.graph_from_dict({"vertices": [], "meta_ops": []})
    with pytest.raises(G.GraphValidationError, match="empty-graph"):
        G.graph_from_dict({"vertices": [], "edges": [], "meta_ops": []})


def test_library_exports_every_declared_symbol():
    from paper_2505_23131_b200 import _build, _native
    header = (ROOT / "include" / "flowplace_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|const char \*|void)\s*\*?\s*(fp_\w+)\s*\(", header,
                              re.M))
    assert {"fp_run_packed", "fp_sim_batch", "fp_problem_create"} <= declared
    if not _build.LIB.exists():
        _build.build()
    lib = ctypes.CDLL(str(_build.LIB))
    for sym in sorted(declared):
        assert hasattr(lib, sym), sym
    assert set(_native.EXPORTED) <= declared


def test_feature_forests_reproduce_path_lists():
    """The next-pointer forests the large-graph encoder consumes give the
    reference's explicit b/t paths (features.py:88-95) and their lengths."""
    for g in (builders.build_llama_block(), builders.sparse_dag(1500, seed=2)):
        f = static_features(g, 4.0)
        for which, paths, nxt in (("b", f.b_paths, f.b_next), ("t", f.t_paths, f.t_next)):
            for v in range(0, len(g), 7):
                walk = [v]
                while nxt[walk[-1]] >= 0:
                    walk.append(int(nxt[walk[-1]]))
                assert tuple(walk) == paths[v]
            assert f.path_lengths(which).tolist() == [len(p) for p in paths]


def test_native_static_features_bit_exact():
    """fp_static_features (native host sweep used from NATIVE_MIN_N ops on)
    reproduces the Python mirror of features.py:51-96 bit for bit, next
    forests included, and refuses a cycle."""
    from paper_2505_23131_b200 import _native as N
    graphs = (builders.build_llama_block(), builders.build_ffnn(8, 4, 16, 4, 2),
              builders.sparse_dag(5000, seed=4), builders.relabel(builders.sparse_dag(3000, seed=5), 9))
    for g in graphs:
        for cf in (4.0, 3.7):
            a = static_features(g, cf, native=False)
            b = static_features(g, cf, native=True)
            assert a.matrix.tobytes() == b.matrix.tobytes()
            assert a.b_next.tolist() == b.b_next.tolist()
            assert a.t_next.tolist() == b.t_next.tolist()
    # 0 -> 1 -> 2 -> 1 (cycle)
    ip = np.array([0, 0, 2, 3], np.int32)
    pi = np.array([0, 2, 1], np.int32)
    si_p = np.array([0, 1, 2, 3], np.int32)
    si = np.array([1, 2, 1], np.int32)
    z = np.ones(3)
    out = np.zeros((3, 5)); nx = np.zeros(3, np.int32); tx = np.zeros(3, np.int32)
    with pytest.raises(N.NativeError, match="not a DAG"):
        N.check(N.lib().fp_static_features(ctypes.c_int32(3), N.ptr(ip), N.ptr(pi), N.ptr(si_p),
                                           N.ptr(si), N.ptr(z), N.ptr(z), ctypes.c_double(4.0),
                                           N.ptr(out), N.ptr(nx), N.ptr(tx)))


def test_relabel_keeps_the_dag():
    g = builders.sparse_dag(500, seed=1)
    r = builders.relabel(g, seed=3)
    assert G.validate(r) == []
    assert len(r) == len(g) and len(r.edges) == len(g.edges)
    # same multiset of (flops, bytes) and same degree sequence
    assert sorted((v.flops, v.output_bytes) for v in r.vertices) == \
        sorted((v.flops, v.output_bytes) for v in g.vertices)
    assert sorted(len(r.preds(v)) for v in range(len(r))) == \
        sorted(len(g.preds(v)) for v in range(len(g)))
    # longest paths are relabelling-invariant
    assert np.isclose(static_features(r, 4.0).t_level.max(), static_features(g, 4.0).t_level.max())


def test_policy_config_modes():
    from paper_2505_23131_b200.policy import PolicyConfig
    assert PolicyConfig(mp_mode="per_step").mp_mode == "per_step"
    with pytest.raises(ValueError):
        PolicyConfig(mp_mode="sometimes")


def test_layout_flags_are_distinct_bits():
    from paper_2505_23131_b200 import _native as N
    header = (ROOT / "include" / "flowplace_b200.h").read_text()
    flags = {k: int(v) for k, v in re.findall(r"#define (FP_FLAG_\w+) (\d+)", header)}
    assert flags == {"FP_FLAG_WIDE": N.FLAG_WIDE, "FP_FLAG_TIE_RANDOM": N.FLAG_TIE_RANDOM,
                     "FP_FLAG_PER_STEP": N.FLAG_PER_STEP}
    vals = list(flags.values())
    assert all(v & (v - 1) == 0 for v in vals) and len(set(vals)) == len(vals)
