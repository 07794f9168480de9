import sys, time
sys.path.insert(0, ".")
from paper_2512_07536_b200 import topoopt as T
n, r = 1024, 4096
bu, e = T.allocate_edge_capacity([1.0] * n, r)
warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
T.solve(n, r, warm_start=warm, max_iter=5, rho=10.0, epsilon=1e-8)
t = time.time(); s = T.solve(n, r, warm_start=warm, max_iter=30, rho=10.0, epsilon=1e-8); print("e2e 30 its", time.time() - t)
