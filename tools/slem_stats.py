"""Lanczos step counts of the trace and one-off SLEM reports (instrumentation
build: make -C paper_2512_07536_b200 STAMPS=1; GPU box):
  TPB_LIB=paper_2512_07536_b200/libtopoopt_b200_stamps.so python tools/slem_stats.py"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from oracle import topoopt_oracle as O  # noqa: E402
from paper_2512_07536_b200 import _lib  # noqa: E402
from paper_2512_07536_b200 import topoopt as T  # noqa: E402
from paper_2512_07536_b200.sweep import sweep_jobs  # noqa: E402

lib = _lib.load()
st = (C.c_ulonglong * 16)()


def report(tag):
    lib.tp_slem_stats(st, 1)
    c0, s0, c1, s1, k0, k1, t0, t1 = list(st)[:8]
    g0, e0, v0, g1, e1, v1, n0, n1 = list(st)[8:16]
    if c0 or c1:
        print(f"  checks per report: trace {n0 / max(c0, 1):.2f}, one-off {n1 / max(c1, 1):.2f}")
        print(f"  check parts (warp 0, rank 0; us per report): trace gershgorin {g0 / max(c0, 1) / 1.9e3:.1f} "
              f"multisection {e0 / max(c0, 1) / 1.9e3:.1f} inverse iteration {v0 / max(c0, 1) / 1.9e3:.1f} | one-off "
              f"{g1 / max(c1, 1) / 1.9e3:.1f} {e1 / max(c1, 1) / 1.9e3:.1f} {v1 / max(c1, 1) / 1.9e3:.1f}", flush=True)
    print(f"{tag}: trace {c0} reports, {s0 / max(c0, 1):.1f} steps, {t0 / max(c0, 1) / 1.9e3:.1f} us "
          f"(checks {k0 / max(c0, 1) / 1.9e3:.1f} us) each | one-off {c1} reports, {s1 / max(c1, 1):.1f} steps, "
          f"{t1 / max(c1, 1) / 1.9e3:.1f} us (checks {k1 / max(c1, 1) / 1.9e3:.1f} us) each", flush=True)


lib.tp_slem_stats(st, 1)
n, r = 1024, 4096
bu, e = O.allocate_edge_capacity([1.0] * n, r)
warm = T.anneal_degree_topology(e, steps=1, moves_per_temp=1, seed=0)
s = T.solve(n, r, warm_start=warm, rho=10.0, epsilon=1e-8, max_iter=60)
report("n=1024 hom, 60 iterations")
bs1 = T.BatchSolver(n, r=[r], rho=10.0, epsilon=1e-8, max_iter=60)
bs1.set_warm(0, warm)
bs1.start()
bs1.sync()
report("n=1024 feasible-start report alone")
bs1.iterate(60)
bs1.sync()
report("n=1024 60 trace reports")
bs1.finish()
report("n=1024 final report alone (warm-started from the trace's Ritz vectors)")
bs1.close()
jobs = sweep_jobs(256, 64)
het = [j for j in jobs if j.scenario == "two_tier"][:16]
bu, e, stt = T.allocate_batch(np.array([j.bandwidths for j in het]), [j.r for j in het])
deg = [d for d, q in zip(e, stt) if q == 0]
bs = T.BatchSolver(256, degrees=np.array(deg), rho=10.0, epsilon=1e-8, max_iter=60)
for b in range(bs.batch):
    bs.set_warm(b, T.anneal_degree_topology(deg[b], steps=1, moves_per_temp=1, seed=0))
bs.start()
bs.iterate(60)
bs.sync()
report(f"n=256 het two_tier x{bs.batch}, 60 iterations")
bs.close()
