"""e2e variance probe: tp_solve (K=30) repeated, before/after other solver use."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2512_07536_b200 import topoopt as T
n, r = 1024, 4096
bu, e = T.allocate_edge_capacity([1.0] * n, r)
warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
def e2e(tag):
    ts = []
    for _ in range(4):
        torch.cuda.synchronize()
        t = time.time(); T.solve(n, r, warm_start=warm, max_iter=30, rho=10.0, epsilon=1e-8); ts.append(time.time() - t)
    print(tag, " ".join(f"{x*1e3:.1f}" for x in ts), "ms", flush=True)
e2e("fresh")
bs = T.BatchSolver(n, r=[r], max_iter=60, linear_solver=1, rho=10.0, epsilon=1e-8)
bs.set_warm(0, warm); bs.start(); bs.iterate(20); bs.sync(); bs.close()
e2e("after CG solver")
bs = T.BatchSolver(n, r=[r], max_iter=60, rho=10.0, epsilon=1e-8)
bs.set_warm(0, warm); bs.start(); bs.iterate(20); bs.sync()
for ph in range(7): bs.bench_phase(ph, 3)
torch.cuda.synchronize(); bs.close()
e2e("after phases")
