"""Dump solve outputs for a bitwise A/B between two builds (TPB_LIB=...):
python tools/bitwise_ab.py out.npz; compare two dumps with --cmp a.npz b.npz."""
import sys
import numpy as np

if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print("bitwise-equal" if not bad else f"DIFFER: {bad}")
    sys.exit(0)
from paper_2512_07536_b200 import topoopt as tp

out = {}
for n, r, het in [(16, 32, False), (64, 192, False), (256, 1024, False), (64, 0, True)]:
    if het:
        s = tp.solve_het(np.array([9] * 32 + [3] * 32), max_iter=3000)
    else:
        s = tp.solve(n, r, max_iter=3000)
    k = f"{n}_{r}_{int(het)}"
    out[k + "_w"] = s.weights
    out[k + "_e"] = s.edges
    out[k + "_t"] = s.trace[: s.iterations]
    print(k, s.iterations, repr(s.acf_value))
np.savez(sys.argv[1], **out)
