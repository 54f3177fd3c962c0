"""Wall time of the user-level C5 synthesis vs its device phases (where the host time goes)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2005_06191_b200 import gridmdp as g  # noqa: E402
from paper_2005_06191_b200 import workloads as W  # noqa: E402

m = g.parse_config(W.WORKLOADS["C5"](), "C5")
for i in range(4):
    t0 = time.perf_counter()
    r = g.synthesize(m, m.spec, g.SynthesisOptions(mode="ofa"))
    t1 = time.perf_counter()
    b, s = g.last_times(m)
    v = float(r.values[:, 0].sum())
    t2 = time.perf_counter()
    print(f"run {i}: wall {1e3 * (t1 - t0):8.1f} ms  device build {b:6.2f} sweep {s:8.2f} ms  touch {1e3 * (t2 - t1):6.1f} ms  sum {v:.6e}",
          flush=True)
