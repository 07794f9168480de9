"""Per-phase times of one lockstep batch (event-timed replays on the solver
stream) next to the whole iteration: where an iteration's time goes.
    python tools/phase_probe.py [n] [batch]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_07536_b200 import topoopt as T
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
r = 4 * n
bu, e = T.allocate_edge_capacity([1.0] * n, r)
warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
bs = T.BatchSolver(n, r=[r] * B, max_iter=400, rho=10.0, epsilon=1e-8)
bs.set_warm(0, warm)
for b in range(1, B):
    bs.set_warm(b, warm)
bs.start()
st = torch.cuda.ExternalStream(bs.stream)
def timed(f, reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f(1); torch.cuda.synchronize()
    a.record(st); f(reps); b.record(st); b.synchronize()
    return a.elapsed_time(b) / reps
it = timed(lambda k: (bs.iterate(k), None), 32)
names = ["cone", "xstep", "topr", "slem", "prep", "xstep_a", "xstep_b"]
out = {"n": n, "B": B, "iteration_ms": it}
for ph, nm in enumerate(names):
    out[nm + "_ms"] = timed(lambda k, ph=ph: bs.bench_phase(ph, k), 8)
print(out)
