"""Phase breakdown of the grid top-r kernel at n=1024 (bench workload) from
globaltimer stamps (instrumentation build: make -C paper_2512_07536_b200
STAMPS=1; GPU box):
  TPB_LIB=paper_2512_07536_b200/libtopoopt_b200_stamps.so python tools/topr_stamps.py"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_07536_b200 import _lib  # noqa: E402
from paper_2512_07536_b200 import topoopt as T  # noqa: E402

n, r = 1024, 4096
lib = _lib.load()
buf = torch.zeros(16 * 148, dtype=torch.int64, device="cuda")
e = T.allocate_edge_capacity([1.0] * n, r)[1]
warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
bs = T.BatchSolver(n, r=[r], rho=10.0, epsilon=1e-8, max_iter=400)
bs.set_warm(0, warm)
bs.start()
bs.iterate(20)
bs.sync()
assert lib.tp_topr_set_stamps(C.c_void_p(buf.data_ptr())) == 0
for it in range(4):
    buf.fill_(-1)
    bs.bench_phase(2, 1)
    torch.cuda.synchronize()
    st = buf.view(-1, 16).cpu().numpy().astype(np.float64)
    st[st < 0] = np.nan
    t0 = np.nanmin(st[:, 0])
    rel = (st - t0) / 1e3
    rounds = int(np.sum(~np.isnan(rel[0, 2:14:2])))
    print(f"run {it}: rounds {rounds}, end {np.nanmax(rel[:, 13]):.2f} us")
    names = [("start spread", 0, 0), ("load", 0, 1)]
    prev = 1
    for k in range(rounds):
        names += [(f"round {k} hist+atomics", prev, 2 + 2 * k), (f"round {k} grid sync", 2 + 2 * k, 3 + 2 * k)]
        prev = 3 + 2 * k
    names += [("select + count pass", prev, 14), ("final grid sync", 14, 15), ("prefix + list pass", 15, 13)]
    for name, a, b in names:
        d = rel[:, b] - rel[:, a] if a != b else rel[:, a]
        print(f"  {name:28s} mean {np.nanmean(d):7.2f}  min {np.nanmin(d):7.2f}  max {np.nanmax(d):7.2f} us")
bs.close()
