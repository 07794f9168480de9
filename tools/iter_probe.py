"""Per-iteration time of the n=1024 config-4 solve under variations (GPU box):
trace SLEM every iteration vs every 1000th, to locate the critical path of
the 3-stream iteration graph."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from oracle import topoopt_oracle as O  # noqa: E402  (warm-start allocation only)
from paper_2512_07536_b200 import topoopt as T  # noqa: E402

n, r = 1024, 4096
bu, e = O.allocate_edge_capacity([1.0] * n, r)
warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
for stride in (1, 1000):
    bs = T.BatchSolver(n, r=[r], rho=10.0, epsilon=1e-30, max_iter=400, trace_stride=stride)
    bs.set_warm(0, warm)
    bs.start()
    st = torch.cuda.ExternalStream(bs.stream)
    bs.iterate(16)
    bs.sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        a.record(st)
        bs.iterate(160)
        b.record(st)
    b.synchronize()
    print(f"trace_stride={stride:5d}: {a.elapsed_time(b) / 160:.3f} ms/iter", flush=True)
    bs.close()
