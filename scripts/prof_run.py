"""Short single-GPU run of one workload for ncu captures (launch lists and
`--set full` reports). Not a benchmark: numbers printed under a profiler are
never reported.

  python scripts/prof_run.py --workload C2b --horizon 2
  python scripts/prof_run.py --workload C5 --horizon 2 --mode ofa
"""
import argparse
import re
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C2b")
    ap.add_argument("--horizon", type=int, default=2)
    ap.add_argument("--mode", default=None)
    ap.add_argument("--repeat", type=int, default=1)
    a = ap.parse_args()

    import torch

    from paper_2005_06191_b200 import gridmdp as g
    from paper_2005_06191_b200 import sharded as S
    from paper_2005_06191_b200 import workloads as W

    text = W.WORKLOADS[a.workload]()
    text = re.sub(r"spec.time_steps = \d+;", f"spec.time_steps = {a.horizon};", text)
    if a.mode:
        text = re.sub(r"exec.mode = \w+;", f"exec.mode = {a.mode};", text)
    m = g.parse_config(text, a.workload)
    s = m.sizes()
    be = S.DeviceBackend(m, torch.cuda.current_stream())
    for _ in range(a.repeat):
        t = time.perf_counter()
        S.synthesize_sharded(be, int(s.n_states), int(s.horizon), m.spec.is_reach(), m.options.mode == "matrix",
                             torch.device("cuda", 0))
        torch.cuda.synchronize()
        print(f"{a.workload}: rows={s.rows} R={s.row_width} T={s.horizon} mode={m.options.mode} "
              f"wall={time.perf_counter() - t:.3f}s")
    be.release()


if __name__ == "__main__":
    main()
