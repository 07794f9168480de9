"""Wall time of the small golden solves through the C ABI (GPU box): config 1
(n=16 hom, r=32) and config 2 (n=64 node-level het), three calls each (the
first also builds the solve plan)."""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2512_07536_b200 import topoopt as T  # noqa: E402

G = os.path.join("tests", "golden")
c1 = json.load(open(os.path.join(G, "config1.json")))
c2 = json.load(open(os.path.join(G, "config2.json")))
for rep in range(3):
    t = time.perf_counter()
    s = T.solve(16, 32, warm_start=c1["warm"], **c1["cfg"])
    t1 = time.perf_counter() - t
    t = time.perf_counter()
    kw = dict(c2["cfg"])
    s2 = T.solve_het(np.array(c2["degrees"]), warm_start=np.array(c2["warm"]), **kw)
    t2 = time.perf_counter() - t
    print(f"config1 {s.iterations} its {t1 * 1e3:.1f} ms ({t1 / s.iterations * 1e6:.1f} us/it) | "
          f"config2 {s2.iterations} its {t2 * 1e3:.1f} ms ({t2 / s2.iterations * 1e6:.1f} us/it)", flush=True)
