import ctypes as C, os, sys, time
import numpy as np
sys.path.insert(0, ".")
os.environ["TPB_TIMING"] = "1"
from paper_2512_07536_b200 import topoopt as T, _lib
L = _lib.load()
n, r = 1024, 4096
bu, e = T.allocate_edge_capacity([1.0] * n, r)
w = T.anneal_degree_topology(e, steps=1, moves_per_temp=1)
for K in (30, 30, 30):
    cfg = T.SolverConfig(max_iter=K, rho=10.0, epsilon=1e-8).to_c()
    res = T.tp_result()
    edges = np.zeros((r, 2), np.int32); weights = np.zeros(r); trace = np.zeros((K, 3)); note = C.create_string_buffer(512)
    we = np.ascontiguousarray(w, np.int32)
    t = time.time()
    rc = L.tp_solve(n, r, C.byref(cfg), T._ip(we), len(we), C.byref(res), T._ip(edges), T._dp(weights), T._dp(trace), note, 512)
    t1 = time.time()
    W = T.gossip_matrix(n, edges[:res.n_edges], weights[:res.n_edges])
    t2 = time.time()
    print(f"K={K} tp_solve {t1-t:.3f}s  gossip_matrix {t2-t1:.3f}s rc={rc}", flush=True)
