import sys, os
sys.path.insert(0, "/root/repo")
import torch
from paper_2512_07536_b200 import topoopt as T
n, r = 1024, 4096
bu, e = T.allocate_edge_capacity([1.0] * n, r)
warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
for ts in (1, 8, 1, 8):
    bs = T.BatchSolver(n, r=[r], max_iter=400, rho=10.0, epsilon=1e-8, trace_stride=ts)
    bs.set_warm(0, warm); bs.start()
    st = torch.cuda.ExternalStream(bs.stream)
    bs.iterate(8); bs.sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); bs.iterate(32); b.record(st); b.synchronize()
    print("trace_stride", ts, "ms/iter", a.elapsed_time(b) / 32, flush=True)
    bs.close()
