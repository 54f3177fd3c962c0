"""Repeated syntheses of one workload (timing stability / knob checks): device build
and sweep time of each. Usage: c3b_repeat.py [workload] [runs] [time_steps]."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2005_06191_b200 import gridmdp as g  # noqa: E402
from paper_2005_06191_b200 import workloads as W  # noqa: E402
from paper_2005_06191_b200 import _capi  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3b"
ov = {"time_steps": int(sys.argv[3])} if len(sys.argv) > 3 else {}
text = W.WORKLOADS[name]() if name in W.WORKLOADS else Path(name).read_text()  # a workload or a config path
m = g.parse_config(text, Path(name).stem, **ov)
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    t = time.perf_counter()
    g.synthesize(m)
    wall = time.perf_counter() - t
    b, s = g.last_times(m)
    var = _capi.lib.gm_last_kernel_variant(_capi.KF_EXPECT_OFA).decode()
    print(f"{name} {i:3d} wall {wall * 1e3:8.2f} ms  build {b:7.3f} ms  sweep {s:8.3f} ms  ofa {var}", flush=True)
