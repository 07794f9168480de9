"""Per-phase device time of one lockstep iteration of the config-5 batches
(GPU box): the homogeneous batch (64 budgets) and the node-level het batch
(192 jobs), via BatchSolver.bench_phase (0 projection, 1 x-step, 2 top-r /
binary z, 3 trace SLEM, 4 prep) and the whole iteration."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_07536_b200 import topoopt as T  # noqa: E402
from paper_2512_07536_b200.sweep import sweep_jobs  # noqa: E402

n = 256
jobs = sweep_jobs(n, 64)
hom = [j for j in jobs if j.scenario == "homogeneous"]
het = [j for j in jobs if j.scenario != "homogeneous"]
bu, e, st = T.allocate_batch(np.array([j.bandwidths for j in het]), [j.r for j in het])
deg = [d for d, s in zip(e, st) if s == 0]
for name, mk in (("hom", lambda: T.BatchSolver(n, r=[j.r for j in hom], rho=10.0, epsilon=1e-30, max_iter=200)),
                 ("het", lambda: T.BatchSolver(n, degrees=np.array(deg), rho=10.0, epsilon=1e-30, max_iter=200))):
    bs = mk()
    for b in range(bs.batch):
        if name == "hom":
            _, ee = T.allocate_edge_capacity([1.0] * n, hom[b].r)
            w = T.anneal_degree_topology(ee, steps=1, moves_per_temp=1, seed=0)
        else:
            w = T.anneal_degree_topology(deg[b], steps=1, moves_per_temp=1, seed=0)
        bs.set_warm(b, w)
    bs.start()
    s = torch.cuda.ExternalStream(bs.stream)
    bs.iterate(8)
    bs.sync()

    def timed(fn, reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn(reps)
        b.record(s)
        b.synchronize()
        return a.elapsed_time(b) / reps

    it = timed(bs.iterate, 16)
    ph = {p: timed(lambda k, p=p: bs.bench_phase(p, k), 4) for p in (0, 1, 2, 3, 4)}
    print(f"{name} B={bs.batch}: iteration {it:.2f} ms | projection {ph[0]:.2f} x-step {ph[1]:.2f} "
          f"select {ph[2]:.2f} SLEM {ph[3]:.2f} prep {ph[4]:.2f} ms", flush=True)
    bs.close()
