"""Capacity-bound system goldens (§8f row 3: intra_server_constraints /
bcube_constraints at proj/src/bandwidth.cpp:172-261, project_binary_z_capped
at proj/src/admm_het.cpp:125-154, anneal_capacity_topology at
proj/src/anneal.cpp:275-391, solve_het on capacity rows) from the compiled
reference. Run in the development container:
``make -C oracle && python tests/golden/make_capacity.py``."""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
TIGHT = dict(rho=10.0, epsilon=1e-8, max_iter=3000)  # proj/tests/test_admm_het.cpp:19-25
T8 = ["tiered8", 4.88, 4.88, 9.76]


def sol_dict(s):
    return {"edges": s.edges.tolist(), "weights": s.weights.tolist(), "acf": s.acf,
            "lambda_tilde": s.lambda_tilde, "residual": s.residual, "converged": s.converged,
            "connected": s.connected, "iterations": s.iterations, "note": s.note, "trace": s.trace.tolist()}


def main():
    out = {"systems": {}, "capped": [], "anneal": [], "solves": []}
    for name, spec in [("tiered8", T8), ("bcube_4_2", ["bcube", 4, 2]), ("bcube_2_2", ["bcube", 2, 2]),
                       ("bcube_3_2", ["bcube", 3, 2]), ("bcube_3_1", ["bcube", 3, 1])]:
        out["systems"][name] = {"spec": spec, **ref.capacity_system(tuple(spec))}
    rng = np.random.default_rng(5)
    for spec, r in [(T8, 12), (["bcube", 4, 2], 24), (["bcube", 2, 2], 5), (["bcube", 3, 1], 3),
                    (["bcube", 3, 2], 10)]:
        m = out["systems"][{"tiered8": "tiered8"}.get(spec[0], f"bcube_{spec[1]}_{spec[2]}")]["m"]
        for trial in range(3):
            v = rng.standard_normal(m)
            if trial == 2:
                v = np.round(v, 1)  # ties to the lower index
            out["capped"].append({"spec": spec, "r": r, "v": v.tolist(),
                                  "z": ref.project_binary_z_capped(tuple(spec), v, r).tolist()})
    for spec, r, steps, seed in [(T8, 12, 200, 0), (T8, 10, 200, 0), (["bcube", 4, 2], 24, 50, 1),
                                 (["bcube", 3, 2], 12, 30, 2), (["bcube", 4, 3], 100, 200, 3),
                                 (["bcube", 3, 3], 40, 200, 4)]:
        out["anneal"].append({"spec": spec, "r": r, "steps": steps, "seed": seed,
                              "edges": ref.anneal_capacity(tuple(spec), r, steps=steps, seed=seed).tolist()})
    # solves (proj/tests/test_admm_het.cpp:171-229, acceptance.cpp:238-268)
    for spec, r, warm, drop in [(T8, 12, None, False), (["bcube", 4, 2], 24, None, False),
                                (["bcube", 2, 2], 5, [[0, 1], [0, 2], [1, 3], [2, 3]], False),
                                (T8, 10, "anneal", False), (T8, 10, "anneal", True)]:
        if warm == "anneal":
            warm = ref.anneal_capacity(tuple(spec), r).tolist()
        if warm is None:
            warm = ref.anneal_capacity(tuple(spec), r, drop_last=drop).tolist()
        s = ref.solve_het_capacity(tuple(spec), r, warm_edges=np.array(warm), drop_last=drop, **TIGHT)
        out["solves"].append({"spec": spec, "r": r, "drop_last": drop, "warm": warm, "cfg": TIGHT,
                              "solution": sol_dict(s)})
    with open(os.path.join(OUT, "capacity.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
