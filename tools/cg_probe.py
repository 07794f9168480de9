"""CG x-step probe: n=1024 solve with linear_solver=1 for a few iterations
(used under ncu: -k regex:xstep_cg)."""
import sys

sys.path.insert(0, ".")
from oracle import topoopt_oracle as O  # noqa: E402  (warm-start allocation only)
from paper_2512_07536_b200 import topoopt as T  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
r = 4 * n
bu, e = O.allocate_edge_capacity([1.0] * n, r)
warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
s = T.solve(n, r, warm_start=warm, rho=10.0, epsilon=1e-8, max_iter=4, linear_solver=1)
print("iterations", s.iterations)
