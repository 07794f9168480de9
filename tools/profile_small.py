"""Short solves for the per-kernel launch list (run under ncu)."""
import sys
sys.path.insert(0, ".")
from paper_2512_07536_b200 import topoopt as T
which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if which == "cfg1":
    T.solve(16, 32, rho=10.0, epsilon=1e-8, max_iter=64)
else:
    bu, e = T.allocate_edge_capacity([9.76] * 32 + [3.25] * 32, 192)
    T.solve_het(e, rho=10.0, epsilon=1e-8, max_iter=64)
