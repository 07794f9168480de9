"""On-disk format goldens (§8f row 4: proj/src/topology.cpp:283-324,
proj/src/admm.cpp:223-236, proj/include/topoopt/textio.hpp:10-14,
proj/tools/topoopt.cpp:244-296): the reference's own serializations of
topologies, gossip matrices, traces and the optimize command's
solution.json / allocation.json, byte for byte (the oracle build's nlohmann
prints as stock 3.11.3, oracle/Makefile).
Run in the development container: ``python tests/golden/make_formats.py``."""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from oracle import topoopt_oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    cases = []
    c1 = json.load(open(os.path.join(OUT, "config1.json")))
    s = ref.solve(16, 32, warm_edges=np.array(c1["warm"]), **c1["cfg"])
    cases.append({"label": "config1", "n": 16, "edges": s.edges.tolist(), "weights": s.weights.tolist(),
                  "topology_json": ref.topology_to_json(16, s.edges, s.weights),
                  "w_csv": ref.matrix_to_csv(s.w), "trace_csv": s.trace_csv,
                  # the CLI's own objects (proj/tools/topoopt.cpp:244-246, 285-296)
                  "solution": {"acf": s.acf, "lambda_tilde": s.lambda_tilde, "converged": bool(s.converged),
                               "connected": bool(s.connected), "repaired": bool(s.repaired),
                               "iterations": int(s.iterations), "residual": s.residual,
                               "note": s.note},
                  "solution_json": ref.solution_json("homogeneous", s.acf, s.lambda_tilde, s.converged,
                                                     s.connected, s.repaired, s.iterations, s.residual,
                                                     len(s.edges), s.note)})
    c2 = json.load(open(os.path.join(OUT, "config2.json")))
    cases[0]["allocation"] = {"b_unit": c2["b_unit"], "e": c2["degrees"]}
    cases[0]["allocation_json"] = ref.allocation_json(c2["b_unit"], c2["degrees"])
    for kind, n in [("ring", 8), ("exponential", 16), ("grid2d", 9)]:
        e, w = ref.generate_benchmark(kind, n)
        cases.append({"label": f"{kind}_{n}", "n": n, "edges": e.tolist(), "weights": w.tolist(),
                      "topology_json": ref.topology_to_json(n, e, w),
                      "w_csv": ref.matrix_to_csv(O.gossip_matrix(n, e, w))})
    # awkward magnitudes: 1e-05, exact binary fractions, long mantissas
    e = np.array([[0, 1], [0, 2], [1, 3], [2, 3], [0, 3]])
    w = np.array([1e-05, 0.5, 0.1, 0.30000000000000004, 2.0 ** -20])
    cases.append({"label": "magnitudes", "n": 4, "edges": e.tolist(), "weights": w.tolist(),
                  "topology_json": ref.topology_to_json(4, e, w),
                  "w_csv": ref.matrix_to_csv(O.gossip_matrix(4, e, w))})
    with open(os.path.join(OUT, "formats.json"), "w") as f:
        json.dump(cases, f)


if __name__ == "__main__":
    main()
