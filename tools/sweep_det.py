"""Per-job dump of one config-5 sweep run (scenario, r, iterations, final
ACF, edges) for run-to-run determinism checks across fresh processes:
``python tools/sweep_det.py out.json`` (GPU box)."""
import json, sys
sys.path.insert(0, ".")
from paper_2512_07536_b200 import sweep as S
jobs = S.sweep_jobs(256, 64)
res, dev_s = S.run_jobs(jobs, 256, rho=10.0, epsilon=1e-8, max_iter=40000)
json.dump({r.index: [r.scenario, r.r, r.iterations, r.acf, r.n_edges] for r in res}, open(sys.argv[1], "w"))
print(sum(r.iterations for r in res), flush=True)
