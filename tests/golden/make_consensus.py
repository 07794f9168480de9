"""Consensus-simulation golden (§8f row 2: proj/src/consensus.cpp:29-67,
generate_benchmark at proj/src/topology.cpp:227-281) from the compiled
reference (oracle/_ref): error traces of x <- W x for optimized and baseline
gossip matrices. Run in the development container:
``make -C oracle && python tests/golden/make_consensus.py``."""
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


def case(label, n, edges, weights, dim, iters, seed):
    w = O.gossip_matrix(n, np.asarray(edges), np.asarray(weights))
    err = ref.simulate(w, dim, iters, seed)
    return {"label": label, "n": n, "edges": np.asarray(edges).tolist(), "weights": np.asarray(weights).tolist(),
            "dim": dim, "iters": iters, "seed": seed, "errors": err.tolist(),
            "acf": ref.spectral_report(w)["acf"]}


def main():
    cases = []
    c1 = json.load(open(os.path.join(OUT, "config1.json")))["solution"]
    cases.append(case("config1_optimized", 16, c1["edges"], c1["weights"], 8, 60, 3))
    for kind, n, dim, iters, seed in [("ring", 16, 4, 40, 0), ("exponential", 64, 16, 30, 7),
                                      ("torus2d", 64, 8, 25, 11), ("grid2d", 16, 3, 20, 5)]:
        e, w = ref.generate_benchmark(kind, n)
        cases.append(case(f"{kind}_{n}", n, e, w, dim, iters, seed))
    c3 = json.load(open(os.path.join(OUT, "config3.json")))["solution"]
    cases.append(case("config3_optimized", 256, c3["edges"], c3["weights"], 128, 60, 0))
    for kind in ("ring", "exponential"):
        e, w = ref.generate_benchmark(kind, 256)
        cases.append(case(f"{kind}_256", 256, e, w, 128, 60, 0))
    with open(os.path.join(OUT, "consensus.json"), "w") as f:
        json.dump(cases, f)


if __name__ == "__main__":
    main()
