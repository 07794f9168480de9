"""Per-phase times of one lockstep iteration for a batch of B n=256 solves
(the config-5 sweep shape): event-timed bench_phase replays."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2512_07536_b200 import topoopt as T

n = 256
B = int(sys.argv[1]) if len(sys.argv) > 1 else 192
het = len(sys.argv) > 2 and sys.argv[2] == "het"
rs = [256 + 32 * (k % 64) for k in range(B)]
if het:
    degs = []
    for r in rs:
        bu, e = T.allocate_edge_capacity([9.76] * 128 + [3.25] * 128, r)
        degs.append(e)
    bs = T.BatchSolver(n, degrees=np.array(degs), max_iter=200, rho=10.0, epsilon=1e-8)
    warms = [T.anneal_degree_topology(d, steps=1, moves_per_temp=1) for d in degs]
else:
    bs = T.BatchSolver(n, r=rs, max_iter=200, rho=10.0, epsilon=1e-8)
    warms = []
    for r in rs:
        bu, e = T.allocate_edge_capacity([1.0] * n, r)
        warms.append(T.anneal_degree_topology(e, steps=1, moves_per_temp=1))
for b, w in enumerate(warms):
    bs.set_warm(b, w)
bs.start()
st = torch.cuda.ExternalStream(bs.stream)
bs.iterate(5); bs.sync()
a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st); bs.iterate(20); b_.record(st); b_.synchronize()
print(f"B={B} {'het' if het else 'hom'}: {a.elapsed_time(b_)/20:.3f} ms/iter")
for ph, name in [(0, "cone"), (1, "xstep"), (2, "topr"), (3, "slem"), (4, "prep")]:
    bs.bench_phase(ph, 1); torch.cuda.synchronize()
    a.record(st); per = bs.bench_phase(ph, 3); b_.record(st); b_.synchronize()
    print(f"  {name:6s} {a.elapsed_time(b_)/3:.3f} ms ({per} launches)")
bs.close()
