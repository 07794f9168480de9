import sys, torch
sys.path.insert(0, ".")
from paper_2512_07536_b200 import topoopt as T
n, r = 1024, 4096
bu, e = T.allocate_edge_capacity([1.0] * n, r)
warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
bs = T.BatchSolver(n, r=[r], max_iter=100, rho=10.0, epsilon=1e-8)
bs.set_warm(0, warm); bs.start()
bs.iterate(12); bs.sync()
bs.close()
