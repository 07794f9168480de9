"""Per-iteration device time of small node-level het batches at n=256 (the
tail of the config-5 sweep, when few solves are still running) against the
phases (GPU box): is the iteration bound by the projection or by the trace
SLEM running beside it?"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_07536_b200 import topoopt as T  # noqa: E402
from paper_2512_07536_b200.sweep import scenario_bandwidths  # noqa: E402

n = 256
bw = scenario_bandwidths("two_tier", n)
for B, stride in ((1, 1), (1, 16), (2, 1), (4, 1), (4, 16), (16, 1), (64, 1)):
    rs = [1024 + 32 * k for k in range(B)]
    bu, e, st = T.allocate_batch(np.array([bw] * B), rs)
    deg = np.array(e)
    bs = T.BatchSolver(n, degrees=deg, rho=10.0, epsilon=1e-30, max_iter=400, trace_stride=stride)
    for b in range(B):
        bs.set_warm(b, T.anneal_degree_topology(deg[b], steps=1, moves_per_temp=1, seed=0))
    bs.start()
    s = torch.cuda.ExternalStream(bs.stream)
    bs.iterate(16)
    bs.sync()

    def timed(fn, reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn(reps)
        b.record(s)
        b.synchronize()
        return a.elapsed_time(b) / reps

    it = timed(bs.iterate, 32)
    ph = {p: timed(lambda k, p=p: bs.bench_phase(p, k), 4) for p in (0, 1, 2, 3, 4)}
    print(f"het two_tier B={B} trace_stride={stride}: iteration {it:.3f} ms | projection {ph[0]:.3f} x-step {ph[1]:.3f} "
          f"select {ph[2]:.3f} trace SLEM {ph[3]:.3f} prep {ph[4]:.3f} ms", flush=True)
    bs.close()
