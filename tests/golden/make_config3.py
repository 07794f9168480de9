"""Config 3 golden (n=256, homogeneous, r=1024, default warm
start) from the compiled reference (oracle/_ref). About an hour of CPU: the
default 200-step anneal (~100 s) plus ~4200 ADMM iterations at ~0.8 s each.
Run in the development container: ``python tests/golden/make_config3.py``.
The trace is stored every 10th iteration (plus the last) to keep the fixture
small."""
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


def main(raw=None):
    if raw is None:
        t = time.time()
        warm = ref.default_warm_start(N, R, 0)
        ta = time.time() - t
        t = time.time()
        s = ref.solve(N, R, warm_edges=warm, **CFG)
        raw = {"warm": warm.tolist(), "anneal_s": ta, "solve_s": time.time() - t, "acf": s.acf,
               "lambda_tilde": s.lambda_tilde, "iterations": s.iterations, "converged": s.converged,
               "edges": s.edges.tolist(), "weights": s.weights.tolist(), "residual": s.residual,
               "connected": s.connected, "trace": s.trace.tolist()}
    tr = raw["trace"]
    keep = sorted(set(range(0, len(tr), 10)) | {len(tr) - 1})
    sol = {k: raw[k] for k in ("edges", "weights", "acf", "lambda_tilde", "residual", "converged",
                               "iterations")}
    sol["connected"] = raw.get("connected", raw["acf"] < 1.0 - 1e-8)
    sol["trace_rows"] = keep
    sol["trace"] = [tr[i] for i in keep]
    out = {"n": N, "r": R, "cfg": CFG, "warm": raw["warm"], "reference_seconds":
           {"default_warm_start": raw["anneal_s"], "solve": raw["solve_s"]}, "solution": sol}
    with open(os.path.join(OUT, "config3.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    # optional: reuse a raw dump of the same run (json with the fields above)
    main(json.load(open(sys.argv[1])) if len(sys.argv) > 1 else None)
