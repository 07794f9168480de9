"""Per-phase device time of the config-2 solve (n=64 node-level het) at
trace strides 1 and 32 (GPU box), via BatchSolver.bench_phase."""
import json, os, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2512_07536_b200 import topoopt as T
c2 = json.load(open("tests/golden/config2.json"))
for stride in (1, 32):
    bs = T.BatchSolver(64, degrees=np.array([c2["degrees"]]), rho=10.0, epsilon=1e-30, max_iter=2000, trace_stride=stride)
    bs.set_warm(0, np.array(c2["warm"]))
    bs.start()
    s = torch.cuda.ExternalStream(bs.stream)
    bs.iterate(64); bs.sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s); bs.iterate(640); b.record(s); b.synchronize()
    it = a.elapsed_time(b) / 640
    ph = {}
    for p in (0, 1, 2, 3, 4):
        a.record(s); bs.bench_phase(p, 20); b.record(s); b.synchronize(); ph[p] = a.elapsed_time(b) / 20
    print(f"config2 stride={stride}: iteration {it*1000:.1f} us | proj {ph[0]*1000:.1f} xstep {ph[1]*1000:.1f} select {ph[2]*1000:.1f} slem {ph[3]*1000:.1f} prep {ph[4]*1000:.1f}", flush=True)
    bs.close()
