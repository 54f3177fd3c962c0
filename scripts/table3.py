"""Table-3 scaling harness (SURVEY.md §8 f row 4): synthesis time against the
state dimension on the reference's benchmark family (benchmark_chain_config,
config.cpp:374-394: n in 1..12, 2^n states, R = 2^n, T = 6, matrix mode), the
engine on one B200 next to the reference's own CPU synthesize (oracle/_ref,
all host threads). Not a bench line: a table for profiles/.

  python scripts/table3.py [--max-n 12] [--out profiles/r01/table3.md]
"""
import argparse
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
REF_BIN = REPO / "oracle" / "_ref" / "gridmdp_ref"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-n", type=int, default=12)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()

    import torch  # noqa: F401  (CUDA context up front)

    from paper_2005_06191_b200 import gridmdp as g

    rows = ["| n | states | R | rows | engine synthesize (s) | reference CPU synthesize (s) | threads | speed-up |",
            "|---|---|---|---|---|---|---|---|"]
    for n in range(1, a.max_n + 1):
        text = g.benchmark_chain_config(n)
        m = g.parse_config(text)
        s = m.sizes()
        for _ in range(2):  # warm-up (device buffers, first launches, clocks)
            g.synthesize(m)
        times = []
        for _ in range(7):
            t = time.perf_counter()
            g.synthesize(m)
            times.append(time.perf_counter() - t)
        gpu_s = sorted(times)[len(times) // 2]  # median: ms-scale calls see host jitter
        cpu_s, th = None, os.cpu_count()
        if REF_BIN.exists():
            with tempfile.TemporaryDirectory() as d:
                cfg = Path(d) / "c.cfg"
                cfg.write_text(text)
                out = subprocess.run([str(REF_BIN), "synthesize", "-c", str(cfg), "-o", str(Path(d) / "r.bin"),
                                      "--threads", "0"], capture_output=True, text=True, check=True).stdout
                cpu_s = float(out.split("time_synthesize_s:")[1].split()[0])
        sp = f"{cpu_s / gpu_s:.1f}x" if cpu_s else "-"
        rows.append(f"| {n} | {s.n_states} | {s.row_width} | {s.rows} | {gpu_s:.5f} | "
                    f"{cpu_s if cpu_s is not None else '-'} | {th} | {sp} |")
        print(rows[-1], flush=True)
    text = "\n".join(rows) + "\n"
    if a.out:
        Path(a.out).write_text("# Table-3 family (benchmark_chain_config), one B200 vs the reference on the host CPU\n\n"
                               "Wall-clock per `gridmdp.synthesize` call (median of 7 after two warm-up calls), matrix mode,\n"
                               "host tables included; the reference's `time_synthesize_s` with all host threads.\n\n"
                               + text)


if __name__ == "__main__":
    main()
