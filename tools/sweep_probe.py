"""Probe the config-5 sweep at reduced budgets (iteration counts, timing)."""
import sys, time
sys.path.insert(0, ".")
from paper_2512_07536_b200.sweep import sweep_jobs, run_jobs
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 2
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 40000
jobs = sweep_jobs(n=256, n_budgets=nb, dr=32 * (64 // nb))
t = time.time()
res, dev = run_jobs(jobs, 256, rho=10.0, epsilon=1e-8, max_iter=maxit)
print(f"{len(jobs)} jobs in {time.time()-t:.1f}s (device {dev:.1f}s)")
for r in res:
    print(f"  {r.scenario:12s} r={r.r:5d} {r.status:10s} it={r.iterations:6d} conv={r.converged} acf={r.acf:.6f} edges={r.n_edges} b_unit={r.b_unit:.4f}")
