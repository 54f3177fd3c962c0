"""Stage (i) for the north-star BMW 320i model (C5) on one B200: its stored MDP is
220.5 GB, so one GPU builds a row-range shard (SURVEY.md §8 d): the states
[0, n_x/2) = 1.97 M rows x 7,000 (110 GB). Times the in-place rebuild of that shard
(k_build_ws, CUDA events of the engine's kernel timer) and prints one JSON line:
probabilities/s and the fraction of HBM (8 B per probability + 8 B per row origin)."""
import ctypes as C
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2005_06191_b200 import _capi  # noqa: E402
from paper_2005_06191_b200 import gridmdp as g  # noqa: E402
from paper_2005_06191_b200 import workloads as W  # noqa: E402

peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
hbm = float(peaks.get("hbm_gbs", 6545.0))
m = g.parse_config(W.WORKLOADS["C5"](), "C5")
s = m.sizes()
nuw = int(s.n_inputs) * int(s.n_disturbances)
x1 = m.n_states // 2
rows, R = x1 * nuw, int(s.row_width)
lib = _capi.lib
h = C.c_void_p()
t = time.perf_counter()
_capi.call("gm_build_shard", m.handle, C.c_int64(0), C.c_int64(x1), C.byref(h))
first = time.perf_counter() - t
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
out = []
for _ in range(reps):
    lib.gm_reset_kernel_stats()
    lib.gm_enable_kernel_timing(1)
    t = time.perf_counter()
    _capi.call("gm_build_shard", m.handle, C.c_int64(0), C.c_int64(x1), C.byref(h))
    wall = time.perf_counter() - t
    lib.gm_enable_kernel_timing(0)
    out.append((lib.gm_kernel_ms_total(_capi.KF_BUILD), wall * 1e3))
variant = lib.gm_last_kernel_variant(_capi.KF_BUILD).decode()
lib.gm_matrix_free(h)
ms = sorted(k for k, _ in out)[len(out) // 2]
probs = rows * R
gbs = (probs * 8 + rows * 8) / (ms * 1e-3) / 1e9
print(json.dumps({"workload": "C5 stored-matrix build, states [0, n_x/2)", "rows": rows, "R": R,
                  "bytes": probs * 8 + rows * 8, "first_call_s": first, "build_ms": [round(k, 3) for k, _ in out],
                  "wall_ms": [round(w, 3) for _, w in out], "median_ms": ms, "probs_per_s": probs / (ms * 1e-3),
                  "achieved_gbs": gbs, "hbm_peak_gbs": hbm, "frac": gbs / hbm, "kernel_variant": variant}))
