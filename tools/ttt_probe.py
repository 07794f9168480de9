"""Time-to-topology probe: full solves to epsilon (SURVEY §8d config 4 and
larger n), wall time through tp_solve with host buffers."""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2512_07536_b200 import topoopt as T  # noqa: E402

for arg in sys.argv[1:]:
    n, r, max_iter = (int(v) for v in arg.split(":"))
    bu, e = T.allocate_edge_capacity([1.0] * n, r)
    t0 = time.time()
    warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
    t_warm = time.time() - t0
    t0 = time.time()
    s = T.solve(n, r, warm_start=warm, rho=10.0, epsilon=1e-8, max_iter=max_iter)
    wall = time.time() - t0
    print(json.dumps({"n": n, "r": r, "warm_s": t_warm, "solve_s": wall, "iterations": s.iterations,
                      "converged": s.converged, "connected": s.connected, "acf": s.acf_value,
                      "edges": len(s.edges), "iter_per_s": s.iterations / wall, "note": s.note}),
          flush=True)
