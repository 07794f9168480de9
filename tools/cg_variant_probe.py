"""Register-resident vs global-memory CG x-step (TPB_CG_GLOBAL) against the
closed form, repeated calls (fresh and recycled pool memory)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2512_07536_b200 import topoopt as T
order = sys.argv[1].split(",") if len(sys.argv) > 1 else ["reg", "reg", "glob", "glob"]
for n in (65, 256, 512, 1024):
    r = 4 * n
    m = n*(n-1)//2; nx = m + 1 + 2*n*n + n
    rng = np.random.default_rng(7 + n)
    y = rng.standard_normal(nx); d = rng.standard_normal(nx) * 0.3
    x_c, _ = T.update_X(n, r, y, d, rho=2.5)
    for mode in order:
        if mode == "glob": os.environ["TPB_CG_GLOBAL"] = "1"
        else: os.environ.pop("TPB_CG_GLOBAL", None)
        x, kkt, its, rel = T.update_X_cg(n, r, y, d, rho=2.5, linear_tol=1e-10)
        print(n, mode, its, rel, "max|x-x_closed| =", np.abs(x - x_c).max(), "g-part", np.abs(x[:m]-x_c[:m]).max(), flush=True)
