"""Workload for compute-sanitizer runs (tools/sanitize.sh): smoke() plus one
n=256 solve (grid top-r path needs n >= 362: one n=400 solve, a few
iterations) and the Ozaki GEMM / sym_eig / capped projection entry points."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import __graft_entry__  # noqa: E402
from oracle import topoopt_oracle as O  # noqa: E402
from paper_2512_07536_b200 import topoopt as T  # noqa: E402

__graft_entry__.smoke()
for n, r, its in ((256, 1024, 6), (400, 1600, 4)):
    bu, e = O.allocate_edge_capacity([1.0] * n, r)
    warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
    s = T.solve(n, r, warm_start=warm, rho=10.0, epsilon=1e-8, max_iter=its)
    print(f"n={n}: {s.iterations} iterations, acf {s.acf_value:.6f}", flush=True)
s = T.solve(16, 32, rho=10.0, epsilon=1e-8, max_iter=20, linear_solver=1)
print("cg solve", s.iterations, flush=True)
d = T.solve_het([3] * 8 + [1] * 8, rho=10.0, epsilon=1e-8, max_iter=20)
print("het solve", d.iterations, flush=True)
print("done", flush=True)
