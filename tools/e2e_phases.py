"""Where the end-to-end time of a short n=1024 solve goes (GPU box): the
handle API's phases timed on the host with device syncs in between."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from oracle import topoopt_oracle as O  # noqa: E402
from paper_2512_07536_b200 import topoopt as T  # noqa: E402

n, r, K = 1024, 4096, 30
bu, e = O.allocate_edge_capacity([1.0] * n, r)
warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
for rep in range(3):
    t = [time.perf_counter()]
    bs = T.BatchSolver(n, r=[r], rho=10.0, epsilon=1e-8, max_iter=K)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    bs.set_warm(0, warm)
    bs.start()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    bs.iterate(K)
    bs.sync()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    bs.finish()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    s = bs.result(0)
    t.append(time.perf_counter())
    bs.close()
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    print(f"rep {rep}: create {d[0]:.1f} ms | start (feasible + SLEM + capture) {d[1]:.1f} | {K} iterations {d[2]:.1f} "
          f"| finish (extraction + final SLEM) {d[3]:.1f} | result {d[4]:.1f}", flush=True)
for rep in range(3):
    t0 = time.perf_counter()
    s = T.solve(n, r, warm_start=warm, max_iter=K, rho=10.0, epsilon=1e-8)
    print(f"tp_solve {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
