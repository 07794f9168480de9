"""Config 5 goldens (the batched n=256 sweep's node-level
heterogeneous scenarios) from the compiled reference (oracle/_ref): the first
K iterations of the reference's solve_het loop (proj/src/admm_het.cpp:266-301;
ref_shim.cpp::ref_admm_het_trace, BiCGSTAB restarted in chunks of 10 until it
meets its 1e-10 tolerance) at r=1024 from the sweep's warm start (the
reference's own annealer at AnnealConfig{steps=1, moves_per_temp=1} on the
Alg. 1 allocation), rho=10: per-iteration residual, lambda and acf.
Scenario (ii) two-tier 3:1 (128 nodes at 9.76, 128 at 3.25) and (iv)
four-tier (9.76, 6.5, 4.88, 3.25) x 64 nodes. About a minute of CPU:
``python tests/golden/make_config5.py``."""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
N, R, K = 256, 1024, 40
SCENARIOS = {
    "ii": [9.76] * 128 + [3.25] * 128,
    "iv": [9.76] * 64 + [6.5] * 64 + [4.88] * 64 + [3.25] * 64,
}


def main():
    out = {"n": N, "r": R, "iterations": K, "rho": 10.0, "alpha": 2.0, "scenarios": {}}
    for which, b in SCENARIOS.items():
        bu, e = ref.allocate(b, R)
        warm = ref.anneal_degree(e, steps=1, moves_per_temp=1, seed=0)
        t = time.time()
        tr = ref.admm_het_trace(e, warm, K)
        out["scenarios"][which] = {"bandwidths": b, "b_unit": bu, "degrees": e.tolist(), "warm": warm.tolist(),
                                   "trace": tr.tolist(), "reference_seconds": time.time() - t}
        print(which, f"{time.time() - t:.1f} s", tr[-1].tolist(), flush=True)
    with open(os.path.join(OUT, "config5_lockstep.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
