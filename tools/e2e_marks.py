"""tp_solve phase timings at n=1024 (instrumentation build with
-DTPB_PHASE_TIMING: phase_mark lines on stderr; GPU box)."""
import sys

sys.path.insert(0, ".")
from oracle import topoopt_oracle as O  # noqa: E402
from paper_2512_07536_b200 import topoopt as T  # noqa: E402

n, r = 1024, 4096
bu, e = O.allocate_edge_capacity([1.0] * n, r)
warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
for k in range(3):
    print(f"--- call {k}", file=sys.stderr, flush=True)
    T.solve(n, r, warm_start=warm, max_iter=30, rho=10.0, epsilon=1e-8)
