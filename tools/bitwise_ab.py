"""Dump solve outputs for a bitwise A/B between two builds of the library
(TPB_LIB=path/to/lib.so): ``python tools/bitwise_ab.py out.npz``; compare two
dumps with ``--cmp a.npz b.npz``. Cases: homogeneous n = 16 .. 1024, node-level
heterogeneous and a capacity-bound system."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print("bitwise-equal" if not bad else f"DIFFER: {bad}")
    sys.exit(0)
from paper_2512_07536_b200 import topoopt as tp  # noqa: E402

out = {}
cases = [("hom", 16, 32), ("hom", 64, 192), ("hom", 256, 1024), ("hom", 100, 300), ("hom", 1024, 4096),
         ("het", 64, 0), ("het", 96, 0), ("cap", 8, 12)]
for kind, n, r in cases:
    if kind == "hom":
        s = tp.solve(n, r, max_iter=3000 if n < 1024 else 300)
    elif kind == "het":
        s = tp.solve_het(np.array([9] * (n // 2) + [3] * (n - n // 2)), max_iter=3000)
    else:
        s = tp.solve_het_capacity(tp.tiered8_tree_system(), r, rho=10.0, epsilon=1e-8, max_iter=3000)
    k = f"{kind}_{n}_{r}"
    out[k + "_w"] = s.weights
    out[k + "_e"] = s.edges
    out[k + "_t"] = s.trace[: s.iterations]
    print(k, s.iterations, repr(s.acf_value), flush=True)
np.savez(sys.argv[1], **out)
