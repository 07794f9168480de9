"""Device-timed ADMM iterations at n=1024 under cone/trace variants:
    TPB_CONE=dmma|ozaki x trace_stride 1|1000 (run on a GPU box)."""
import os
import subprocess
import sys

CODE = r'''
import sys, time, torch
sys.path.insert(0, ".")
from paper_2512_07536_b200 import topoopt as T
n, r, ts = 1024, 4096, int(sys.argv[1])
bu, e = T.allocate_edge_capacity([1.0] * n, r)
warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
bs = T.BatchSolver(n, r=[r], max_iter=100, rho=10.0, epsilon=1e-8, trace_stride=ts)
bs.set_warm(0, warm); bs.start()
st = torch.cuda.ExternalStream(bs.stream)
bs.iterate(8); bs.sync()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st); bs.iterate(40); b.record(st); b.synchronize()
print(f"cone={__import__('os').environ.get('TPB_CONE','ozaki'):6s} trace_stride={ts:5d}: {a.elapsed_time(b)/40:7.3f} ms/iter")
bs.close()
'''

for cone, ts, tol in [("ozaki", 1, "1e-6"), ("ozaki", 1000, "1e-6")]:
    env = dict(os.environ, TPB_CONE=cone, TPB_SLEM_TOL=tol, TPB_SLEM_STATS="1")
    print("tol", tol, flush=True)
    subprocess.run([sys.executable, "-c", CODE, str(ts)], env=env, check=False)
