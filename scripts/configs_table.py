"""Per-configuration measurements (SURVEY.md §8 d "other 1-GPU targets"): every
§8.0 workload synthesised on one B200 next to the reference's own CPU path
(oracle/_ref, all host threads), plus the FP64 DFMA peak (scripts/fp64_peak.cu)
for the FP64-utilisation column. Not a bench line: a table for profiles/.

GPU: one full synthesis (build + T steps in matrix mode, T OFA steps otherwise)
after a warm-up run of the same model (T = 1 for the traffic cases), device-timed with CUDA events on the engine's
stream. CPU: the reference's `synthesize` (time_synthesize_s) where the whole
horizon takes seconds, else one reference `bellman_step` over all rows x T
(steps cost the same, synthesis.cpp:165-195). `--threads 1` runs give per-core
numbers for C1 and C3n.

  python scripts/configs_table.py [--only C1,C5] [--out profiles/r01/configs.md]
"""
import argparse
import json
import os
import re
import subprocess
import sys
import tempfile
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
REF_BIN = REPO / "oracle" / "_ref" / "gridmdp_ref"
ORDER = ["C1", "C2a", "C2b", "C3n", "C3u", "C3e", "C3b", "C4p", "C4", "C5"]
FULL_CPU = {"C1", "C2a", "C3n", "C3u", "C3e", "C3b"}  # whole-horizon reference runs (seconds each)
SINGLE_THREAD = {"C1", "C3n"}


def with_horizon(text, T):
    return re.sub(r"spec.time_steps = \d+;", f"spec.time_steps = {T};", text)


def with_mode(text, mode):
    return re.sub(r"exec.mode = \w+;", f"exec.mode = {mode};", text)


def mem_available():
    for line in open("/proc/meminfo"):
        if line.startswith("MemAvailable:"):
            return int(line.split()[1]) * 1024
    return 0


def ref_synthesize(text, threads):
    with tempfile.TemporaryDirectory() as d:
        cfg = Path(d) / "c.cfg"
        cfg.write_text(text)
        out = subprocess.run([str(REF_BIN), "synthesize", "-c", str(cfg), "-o", str(Path(d) / "r.bin"), "--threads",
                              str(threads)], capture_output=True, text=True, check=True).stdout
        return float(out.split("time_synthesize_s:")[1].split()[0])


def live_fraction(text):
    """Share of rows the sweep reads: all but the absorbed states' rows (reach specs),
    from the CPU oracle's absorbing flags."""
    from oracle import oracle_py as O
    om = O.load(text)
    if not om.reach:
        return 1.0
    return float((om.absorbing() == 0).mean())


def fp64_peak():
    exe = REPO / "scripts" / "_fp64_peak"
    if not exe.exists():
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", str(exe),
                        str(REPO / "scripts" / "fp64_peak.cu")], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    return float(out.split("fp64_dfma_tflops:")[1].split()[0])


def gpu_run(name, text, stream, dev):
    """One synthesis through the engine's C++ entry (gm_synthesize: build, then the T
    steps enqueued back to back), device time from the model's own CUDA events
    (gm_model_last_times), after a warm-up run; a third run with per-launch timing
    gives the kernel-family split."""
    from paper_2005_06191_b200 import _capi
    from paper_2005_06191_b200 import gridmdp as g

    lib = _capi.lib
    m = g.parse_config(text, name)
    s = m.sizes()
    big = int(s.rows) * int(s.row_width) * int(s.horizon) > 2e12
    if big:  # the 7-step traffic OFA cases warm at T = 1
        g.synthesize(g.parse_config(with_horizon(text, 1), name))
    else:
        g.synthesize(m)
    g.synthesize(m)
    build_ms, sweep_ms = g.last_times(m)
    fam = {}
    if not big:
        lib.gm_reset_kernel_stats()
        lib.gm_enable_kernel_timing(1)
        g.synthesize(m)
        lib.gm_enable_kernel_timing(0)
        fam = {n: lib.gm_kernel_ms_total(i) for i, n in enumerate(_capi.KF_NAMES) if lib.gm_kernel_ms_total(i)}
    g.release_cached_memory()
    return s, build_ms / 1e3, sweep_ms / 1e3, fam


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-from", default=None,
                    help="reuse the CPU columns of an earlier configs.md (its JSON records) instead of re-running them")
    a = ap.parse_args()
    prior = {}
    if a.cpu_from:
        for ln in Path(a.cpu_from).read_text().splitlines():
            if ln.startswith("{"):
                r = json.loads(ln)
                prior[r["workload"]] = {k: v for k, v in r.items() if k.startswith("cpu_")}
    import torch

    from paper_2005_06191_b200 import workloads as W
    sys.path.insert(0, str(REPO))
    import bench

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    hbm, peak_kind = bench.peaks()
    f64 = fp64_peak()
    print(f"hbm {hbm} GB/s ({peak_kind}); fp64 dfma {f64:.2f} TFLOP/s", flush=True)
    names = [n for n in ORDER if not a.only or n in a.only.split(",")]
    rows, recs = [], []
    for name in names:
        text = W.WORKLOADS[name]()
        s, build_s, sweep_s, fam = gpu_run(name, text, stream, dev)
        rows_n, R, T, nx = int(s.rows), int(s.row_width), int(s.horizon), int(s.n_states)
        mode = "matrix" if "exec.mode = matrix;" in text else "ofa"
        terms = rows_n * R * T
        tps = terms / sweep_s
        live = live_fraction(text)  # rows of absorbed states are never read (synthesis.cpp:86-89)
        rec = {"workload": name, "mode": mode, "states": nx, "rows": rows_n, "R": R, "T": T,
               "gpu_build_s": build_s, "gpu_sweep_s": sweep_s, "gpu_total_s": build_s + sweep_s,
               "terms_per_s": tps, "live_fraction": live, "hbm_equiv_frac": tps * live * 8 / 1e9 / hbm,
               "fp64_util": 2 * tps * live / (f64 * 1e12), "kernel_ms": fam}
        if mode == "matrix" and build_s > 0:
            rec["build_probs_per_s"] = rows_n * R / build_s
        if name in prior and "cpu_s" in prior[name]:
            rec.update(prior[name])
            rec["speedup"] = rec["cpu_s"] / rec["gpu_total_s"]
        elif not a.no_cpu and REF_BIN.exists():
            th = os.cpu_count() or 1
            if name in FULL_CPU:
                cmode = mode
                if mode == "matrix" and rows_n * R * 8 * 2 > mem_available():
                    cmode = "ofa"  # the reference's matrix would not fit host RAM twice over
                rec["cpu_mode"] = cmode
                rec["cpu_s"] = ref_synthesize(with_mode(text, cmode), 0)
                rec["cpu_kind"] = f"reference synthesize ({cmode}), {th} threads"
                if name in SINGLE_THREAD:
                    rec["cpu_s_1thread"] = ref_synthesize(with_mode(text, cmode), 1)
            else:
                step_s, th = bench.cpu_sweep_step(text, nx)
                rec["cpu_s"] = step_s * T
                rec["cpu_step_s"] = step_s
                rec["cpu_kind"] = f"reference OFA bellman_step x {T}, {th} threads"
            rec["speedup"] = rec["cpu_s"] / rec["gpu_total_s"]
        recs.append(rec)
        print(json.dumps(rec), flush=True)
    hdr = ("| cfg | mode | states | rows | R | T | GPU build (s) | GPU sweep (s) | G terms/s | HBM-equiv | FP64 util "
           "| reference CPU (s) | how | speed-up | CPU 1 thread (s) |")
    rows.append(hdr)
    rows.append("|" + "---|" * 15)
    for r in recs:
        rows.append(f"| {r['workload']} | {r['mode']} | {r['states']:,} | {r['rows']:,} | {r['R']:,} | {r['T']} | "
                    f"{r['gpu_build_s']:.4f} | {r['gpu_sweep_s']:.4f} | {r['terms_per_s'] / 1e9:.0f} | "
                    f"{r['hbm_equiv_frac'] * 100:.0f} % | {r['fp64_util'] * 100:.1f} % | "
                    f"{r.get('cpu_s', float('nan')):.2f} | {r.get('cpu_kind', '-')} | "
                    f"{r.get('speedup', float('nan')):.0f}x | {r.get('cpu_s_1thread', '-')} |")
    table = "\n".join(rows) + "\n"
    print(table)
    if a.out:
        Path(a.out).write_text(
            "# SURVEY §8.0 workloads on one B200 vs the reference on the host CPU\n\n"
            f"`python scripts/configs_table.py --out {a.out}`. HBM = {hbm} GB/s ({peak_kind}); FP64 DFMA peak "
            f"{f64:.2f} TFLOP/s measured by scripts/fp64_peak.cu on the same box. GPU: one full synthesis (gm_synthesize) after a "
            "warm-up run of the same model (T = 1 for C4/C4p), CUDA events on the engine's stream (build = stage i of matrix mode; sweep = the T "
            "Bellman steps; OFA has no build). G terms/s = rows·R·T / sweep; HBM-equiv = 8 B per term of the "
            "rows the sweep reads (absorbed states' rows excluded) against HBM (the bytes matrix mode streams); "
            "FP64 util = 2 flops per such term against the DFMA peak. "
            "CPU: the reference compiled from its sources (oracle/_ref), all host threads"
            + (f" (CPU columns from {a.cpu_from}, an earlier run on the same pool)" if a.cpu_from else "")
            + ".\n\n" + table
            + "\n```\n" + "\n".join(json.dumps(r) for r in recs) + "\n```\n")


if __name__ == "__main__":
    main()
