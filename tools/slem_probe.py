"""One-off SLEM report of an n=1024, 4096-edge topology (tp_spectral_edges,
tol 1e-10): the kernel an ncu capture of slem_trace_kernel looks at (GPU box)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from oracle import topoopt_oracle as O  # noqa: E402
from paper_2512_07536_b200 import topoopt as T  # noqa: E402

n, r = 1024, 4096
bu, e = O.allocate_edge_capacity([1.0] * n, r)
warm = np.asarray(T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)).reshape(-1, 2)
w = np.full(len(warm), 1.0 / 9.0)
for k in range(3):
    t = time.perf_counter()
    rep = T.spectral_edges(n, warm, w)
    print(f"{1e3 * (time.perf_counter() - t):.2f} ms", rep, flush=True)
