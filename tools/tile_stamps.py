"""Phase breakdown of the tile kernels (prep, x-step passes A and B) at
n=1024 (bench workload) from globaltimer stamps (instrumentation build:
make -C paper_2512_07536_b200 STAMPS=1; GPU box):
  TPB_LIB=paper_2512_07536_b200/libtopoopt_b200_stamps.so python tools/tile_stamps.py"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_07536_b200 import _lib  # noqa: E402
from paper_2512_07536_b200 import topoopt as T  # noqa: E402

n, r = 1024, 4096
lib = _lib.load()
ntile = (n // 32) * (n // 32 + 1) // 2
buf = torch.zeros(16 * ntile, dtype=torch.int64, device="cuda")
e = T.allocate_edge_capacity([1.0] * n, r)[1]
warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
bs = T.BatchSolver(n, r=[r], rho=10.0, epsilon=1e-8, max_iter=400)
bs.set_warm(0, warm)
bs.start()
bs.iterate(20)
bs.sync()
assert lib.tp_tile_set_stamps(C.c_void_p(buf.data_ptr())) == 0


def show(title, spans):
    st = buf.view(-1, 16).cpu().numpy().astype(np.float64)
    st[st <= 0] = np.nan
    print(title)
    for name, a, b, mode in spans:
        if mode == "lastgap0":  # spread of the CTA start times
            print(f"  {name:34s} {(np.nanmax(st[:, a]) - np.nanmin(st[:, a])) / 1e3:7.2f} us")
            continue
        if mode == "cta":  # per-CTA span
            dlt = (st[:, b] - st[:, a]) / 1e3
            print(f"  {name:34s} mean {np.nanmean(dlt):7.2f}  min {np.nanmin(dlt):7.2f}  max {np.nanmax(dlt):7.2f} us")
        elif mode == "grid":  # kernel-level: earliest a -> latest b
            print(f"  {name:34s} {(np.nanmax(st[:, b]) - np.nanmin(st[:, a])) / 1e3:7.2f} us")
        else:  # serial tail: latest a -> latest b
            print(f"  {name:34s} {(np.nanmax(st[:, b]) - np.nanmax(st[:, a])) / 1e3:7.2f} us")


for it in range(3):
    buf.fill_(0)
    bs.bench_phase(4, 1)
    torch.cuda.synchronize()
    show(f"prep, run {it}", [("S (loads, symmetrise, stores)", 0, 1, "cta"), ("T", 1, 2, "cta"), ("g part", 2, 3, "cta"),
                             ("y/lambda + Frobenius partials", 3, 4, "cta"), ("block arrival", 4, 5, "cta"),
                             ("first start -> last start", 0, 0, "lastgap0"), ("first start -> last arrival", 0, 5, "grid"),
                             ("last arrival -> last finisher done", 5, 6, "tail"),
                             ("last finisher -> scale written", 6, 7, "tail"), ("first start -> end", 0, 7, "grid")])
    buf.fill_(0)
    bs.bench_phase(1, 1)
    torch.cuda.synchronize()
    show(f"x-step, run {it}", [("pass A per CTA", 8, 9, "cta"), ("pass A start -> last end", 8, 9, "grid"),
                               ("A last end -> B last start", 9, 10, "tail"),
                               ("B prologue (node space) per CTA", 10, 11, "cta"), ("B body per CTA", 11, 12, "cta"),
                               ("B arrival per CTA", 12, 13, "cta"), ("B start spread", 10, 10, "lastgap0"), ("B start -> last arrival", 10, 13, "grid"),
                               ("B last arrival -> end", 13, 14, "tail"), ("A start -> B end", 8, 14, "grid")])
bs.close()
