"""Run INSIDE a flowplace tree patched by integration/install_cuda_backend.py
(tests/test_refshim_gpu.py launches it in a subprocess with that tree first on
sys.path): the reference's own backend-parity pattern
(tests/test_backends.py:33-67 of the reference) with the cuda core in place
of the Cython one -- exec_time under FLOWPLACE_SIM_BACKEND=python vs cuda (and
cython) on every golden simulator case: makespans and Schedules equal,
DeadlockError with the same arguments."""
import json
import os
import sys

import flowplace.simulate as simulate
from flowplace import graph as G
from flowplace._simpy import DeadlockError
from flowplace.cluster import ClusterSpec


def run(backend, g, a, cl, strategy, seed):
    os.environ["FLOWPLACE_SIM_BACKEND"] = backend
    assert simulate.backend_name() == backend
    try:
        return simulate.exec_time(g, a, cl, strategy, seed)
    except DeadlockError as exc:
        return ("deadlock", exc.time_ms, exc.blocked)


def main(path):
    cases = json.loads(open(path).read())["cases"]
    n_dead = 0
    for c in cases:
        gd = c["graph"]  # built unvalidated: one golden case is a deliberate cycle
        g = G.DataflowGraph(tuple(G.Vertex(v["id"], G.OpKind(v["op_kind"]), v["flops"],
                                           v["output_bytes"], v["label"])
                                  for v in gd["vertices"]),
                            tuple(tuple(e) for e in gd["edges"]))
        cl = ClusterSpec.from_dict(c["cluster"])
        args = (g, c["assign"], cl, c["strategy"], c["seed"])
        py = run("python", *args)
        cu = run("cuda", *args)
        cy = run("cython", *args)
        assert py == cu, c["tag"]
        assert cy == cu, c["tag"]
        n_dead += py[0] == "deadlock"
    print(json.dumps({"cases": len(cases), "deadlock_cases": n_dead,
                      "cudacore": simulate.__file__}))


if __name__ == "__main__":
    main(sys.argv[1])
