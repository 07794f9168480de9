"""Config 5 goldens (the batched n=256 sweep's heterogeneous
scenarios) from the compiled reference (oracle/_ref): node-level solves at
r=1024 with the sweep's warm start (the reference's own annealer at
AnnealConfig{steps=1, moves_per_temp=1} on the Alg. 1 allocation), rho=10,
epsilon=1e-8. Scenario (ii) two-tier 3:1 (128 nodes at 9.76, 128 at 3.25) and
(iv) four-tier (9.76, 6.5, 4.88, 3.25) x 64 nodes. Tens of minutes of CPU per
scenario; run in the development container:
``python tests/golden/make_config5.py ii`` (or ``iv``). The trace is stored
every 10th iteration (plus the last)."""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
N, R = 256, 1024
CFG = dict(rho=10.0, epsilon=1e-8, max_iter=40000)
SCENARIOS = {
    "ii": [9.76] * 128 + [3.25] * 128,
    "iv": [9.76] * 64 + [6.5] * 64 + [4.88] * 64 + [3.25] * 64,
}


def main(which):
    b = SCENARIOS[which]
    bu, e = ref.allocate(b, R)
    warm = ref.anneal_degree(e, steps=1, moves_per_temp=1, seed=0)
    t = time.time()
    s = ref.solve_het_node(e, warm_edges=warm, **CFG)
    dt = time.time() - t
    tr = s.trace.tolist()
    keep = sorted(set(range(0, len(tr), 10)) | {len(tr) - 1})
    sol = {"edges": s.edges.tolist(), "weights": s.weights.tolist(), "acf": s.acf,
           "lambda_tilde": s.lambda_tilde, "residual": s.residual, "converged": s.converged,
           "iterations": s.iterations, "connected": s.connected, "repaired": s.repaired,
           "note": s.note, "trace_rows": keep, "trace": [tr[i] for i in keep]}
    out = {"scenario": which, "n": N, "r": R, "bandwidths": b, "b_unit": bu, "degrees": e.tolist(),
           "cfg": CFG, "warm": warm.tolist(), "reference_seconds": {"solve": dt}, "solution": sol}
    with open(os.path.join(OUT, f"config5_{which}.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "ii")
