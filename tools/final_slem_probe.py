"""One-off SLEM report cost at n=1024 (feasible start + final topology) vs tolerance."""
import os, sys, time
sys.path.insert(0, ".")
from paper_2512_07536_b200 import topoopt as T
n, r = 1024, 4096
bu, e = T.allocate_edge_capacity([1.0] * n, r)
warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
T.solve(n, r, warm_start=warm, max_iter=2, rho=10.0, epsilon=1e-8)
for k in range(3):
    t = time.time(); s = T.solve(n, r, warm_start=warm, max_iter=30, rho=10.0, epsilon=1e-8); dt = time.time() - t
print(os.environ.get("TPB_FINAL_TOL", "1e-10"), f"e2e30 {dt*1e3:.1f} ms acf {s.acf_value:.15f} l2 {s.lambda2:.15f} ln {s.lambda_n:.15f} lam {s.lambda_tilde:.15f}")
