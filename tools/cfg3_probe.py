"""Config 3 on the GPU: warm-start and solve wall times vs the reference golden."""
import json, sys, time
sys.path.insert(0, ".")
from paper_2512_07536_b200 import topoopt as T
g = json.load(open("tests/golden/config3.json"))
t = time.time(); w = T.default_warm_start(256, 1024, 0); ta = time.time() - t
t = time.time(); s = T.solve(256, 1024, warm_start=g["warm"], **g["cfg"]); ts = time.time() - t
print(f"warm start {ta:.2f} s (reference {g['reference_seconds']['default_warm_start']:.1f} s); "
      f"solve {ts:.2f} s (reference {g['reference_seconds']['solve']:.0f} s); iterations {s.iterations} "
      f"(reference {g['solution']['iterations']}); acf {s.acf_value:.15f} vs {g['solution']['acf']:.15f}")
