"""Benchmark of the B200 AMYTISS engine (driver contract: one JSON line).

Metric (BASELINE.json): "MDP probs/sec + Bellman sweep time (s) vs CPU ref".
Workload (N=1 and per GPU): C2b = 3-D vehicle reach-avoid with eta/4, stored
MDP, T=32 (BASELINE configs[1]; 741,393 states, 18,534,825 rows, R=729, a
108 GB matrix on one B200). One step = one full synthesis in matrix mode:
stage (i) builds the sharded matrix + target-hit vector in HBM, stage (ii)
runs the 32 backward Bellman steps (all-gather of V between ranks).

  value      MDP probabilities built per second, whole job (rows*R / build time,
             device time with CUDA events on the engine's stream, max over ranks)
  sweep_s    Bellman sweep seconds per synthesis (device time, max over ranks)
  e2e        the same metric through the public C ABI from host data: config text
             parsed on the host, model uploaded, shard built (gm_build_shard_host),
             origins + target-hit vector streamed into pinned host memory
             (wall clock, max over ranks); e2e_synthesize = one full
             gridmdp.synthesize (value/policy tables on the host)
  cpu_baseline        the reference's row kernel on a bounded sample (probs/s)
  cpu_baseline_sweep  one reference bellman_step over the whole workload (OFA,
                      host threads) x T: the CPU sweep time the GPU's sweep_s
                      is compared with

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/gridmdp_ref: RowKernel::compute + fill_row, the body of
build_matrix) on a bounded sample of the same rows with all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

REF_BIN = REPO / "oracle" / "_ref" / "gridmdp_ref"
METRIC = "MDP probs/sec + Bellman sweep time (s) vs CPU ref, 1/2/4/8 B200"


def peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_l1tex(workload: str):
    """L1/TEX utilisation of the OFA consumer kernel from the newest committed ncu capture
    (profiles/*/ncu_l1tex.json, scripts/ncu_summary.py --l1tex), else None."""
    for f in sorted(REPO.glob("profiles/*/ncu_l1tex.json"), reverse=True):
        for k, e in json.loads(f.read_text()).items():
            if e.get("workload") == workload:
                return dict(e, kernel=k, source=str(f.relative_to(REPO)))
    return None


def ncu_traffic(kernel: str, workload: str):
    """DRAM bytes per launch of `kernel` from the newest committed ncu --set full capture
    (profiles/*/ncu_traffic.json, written by scripts/ncu_summary.py --traffic), else None."""
    for f in sorted(REPO.glob("profiles/*/ncu_traffic.json"), reverse=True):
        e = json.loads(f.read_text()).get(kernel)
        if e and e.get("workload") == workload:
            return e["dram_bytes_per_launch"]
    return None


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None
        self.f = None

    def __enter__(self):
        try:
            self.f = tempfile.TemporaryFile(mode="w+")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        if not self.f:
            return None
        self.f.seek(0)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def store_ceiling_ms(be, stream, reps=3):
    """The in-step store ceiling of stage (i): a plain zero fill (torch's vectorised fill
    kernel) of the same matrix buffer, straight after the timed synthesis steps (same
    power / clock regime), device time on the engine's stream. Diagnostic only."""
    import ctypes as C

    import torch

    from paper_2005_06191_b200 import _capi

    rb, re_, R, dp = C.c_int64(), C.c_int64(), C.c_int64(), C.c_void_p()
    _capi.call("gm_matrix_info", be._tm, C.byref(rb), C.byref(re_), C.byref(R), C.byref(dp), None)
    n = (re_.value - rb.value) * int(_capi.lib.gm_matrix_pitch(be._tm))

    class _Buf:  # zero-copy view of the engine's device buffer
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (dp.value, False), "version": 3}

    t = torch.as_tensor(_Buf(), device="cuda")

    def timed(fill):
        out = []
        with torch.cuda.stream(stream):
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fill()
                b.record(stream)
                b.synchronize()
                out.append(a.elapsed_time(b))
        return statistics.median(out)

    # HBM write power depends on the data (zeros toggle few bits): the ceiling is a
    # write of varied doubles (gm_store_probe: hashed mantissas, 16-byte evict-first
    # stores); torch's zero fill is reported beside it
    ms = timed(lambda: _capi.call("gm_store_probe", C.c_void_p(dp.value), C.c_int64(n), C.c_uint64(7),
                                  C.c_void_p(stream.cuda_stream)))
    zero_ms = timed(t.zero_)
    return {"ms": ms, "bytes": n * 8, "gbs": n * 8 / (ms / 1e3) / 1e9, "zero_fill_ms": zero_ms,
            "note": "varied-data write of the matrix buffer after the timed steps (same regime): the build's "
                    "store ceiling; zero_fill_ms: the same bytes as zeros"}


def load_workloads():
    """paper_2005_06191_b200/workloads.py by file path: importing the package would
    load the engine library, which the reference arm must not map."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("_gm_workloads", REPO / "paper_2005_06191_b200" / "workloads.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def ref_sizes(cfg_text: str) -> dict:
    """Sizes of a workload from the reference itself (`gridmdp_ref estimate`:
    print_sizes, tools/gridmdp_main.cpp:43-54) plus the horizon of its spec."""
    import re

    if not REF_BIN.exists():
        raise FileNotFoundError(f"{REF_BIN} missing (make -C oracle ref)")
    with tempfile.NamedTemporaryFile("w", suffix=".cfg", delete=False) as f:
        f.write(cfg_text)
        path = f.name
    try:
        out = subprocess.run([str(REF_BIN), "estimate", "-c", path], capture_output=True, text=True,
                             check=True).stdout
    finally:
        os.unlink(path)
    d = {}
    for line in out.splitlines():
        k, v = line.split(":", 1)
        d[k.strip()] = [int(x) for x in v.split()] if k.strip() == "window" else int(v)
    d["horizon"] = int(re.search(r"spec\.time_steps\s*=\s*(\d+)\s*;", cfg_text).group(1))
    return d


MODEL_NAMES = {"C2b": "vehicle3-eta/4 reach-avoid (stored MDP)", "C2a": "vehicle3 reach-avoid (stored MDP)",
               "C1": "robot 2-d reach-avoid (stored MDP)"}


def bench_config(workload: str, sz: dict, world: int) -> dict:
    """The `config` object of the JSON line; byte-identical in both arms."""
    return {"workload": workload, "model": MODEL_NAMES.get(workload, workload), "states": sz["states"],
            "rows": sz["rows"], "row_width": sz["row_width"], "horizon": sz["horizon"],
            "matrix_bytes": sz["rows"] * sz["row_width"] * 8, "parallelism": f"state-shard x{world}",
            "l2": "inputs larger than L2 (108 GB matrix streamed per step)" if workload == "C2b"
            else "inputs smaller than L2 are re-read every step"}


def cpu_sample(cfg_text: str, rows_total: int, target_s: float, threads: int = 0, cal_rows: int = 20000):
    """Times the reference's row kernel (RowKernel::compute + fill_row) on a bounded
    contiguous sample of rows; returns (probs/s, rows, R, threads, seconds)."""
    if not REF_BIN.exists():
        raise FileNotFoundError(f"{REF_BIN} missing (make -C oracle ref)")
    with tempfile.NamedTemporaryFile("w", suffix=".cfg", delete=False) as f:
        f.write(cfg_text)
        path = f.name

    def run(b, e):
        out = subprocess.run([str(REF_BIN), "time-rows", "-c", path, "--threads", str(threads), "--rows", str(b),
                              str(e)], capture_output=True, text=True, check=True).stdout.split()
        d = dict(zip(out[0::2], out[1::2]))
        return int(d["rows"]), int(d["R"]), int(d["threads"]), float(d["seconds"])

    try:
        # calibrate on a small block, then time up to the whole workload (all rows)
        # or about target_s seconds of host work, whichever is smaller
        n, R, th, s = run(0, min(rows_total, cal_rows))
        want = int(min(rows_total, max(cal_rows, cal_rows * target_s / max(s, 1e-6))))
        n, R, th, s = run(0, want)
        return n * R / s, n, R, th, s
    finally:
        os.unlink(path)


def cpu_sweep_step(cfg_text: str, n_x: int, threads: int = 0):
    """One reference bellman_step (synthesis.cpp:147-161) over the whole workload in OFA
    mode (matrix-free: C2b's 108 GB matrix does not fit host RAM) with V_{k+1} ~ U(0,1)
    from mt19937_64(20240), all host threads. Returns (seconds, threads)."""
    import numpy as np
    if not REF_BIN.exists():
        raise FileNotFoundError(f"{REF_BIN} missing (make -C oracle ref)")
    d = tempfile.mkdtemp()
    try:
        cfg = os.path.join(d, "w.cfg")
        open(cfg, "w").write(cfg_text)
        vn = os.path.join(d, "vnext.f64")
        np.random.Generator(np.random.MT19937(20240)).random(n_x).astype(np.float64).tofile(vn)
        th = threads or (os.cpu_count() or 1)
        out = subprocess.run([str(REF_BIN), "step", "-c", cfg, "--mode", "ofa", "--threads", str(threads),
                              "--vnext", vn, "-o", os.path.join(d, "out")], capture_output=True, text=True,
                             check=True).stdout
        secs = float(out.split("time_step_s:")[1].split()[0])
        return secs, th
    finally:
        subprocess.run(["rm", "-rf", d])


def reference_arm(args, cfg_text, sz):
    """The reference's own CPU implementation of stage (i) (oracle/_ref: the
    unmodified reference sources), all host threads, on bounded samples of the
    workload's rows. Imports nothing from the engine package."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    vals = []
    last = None
    for i in range(args.warmup + args.steps):
        v, n, R, th, s = cpu_sample(cfg_text, sz["rows"], args.cpu_seconds / 2)
        if i >= args.warmup:
            vals.append(v)
        last = (n, R, th, s)
    n, R, th, s = last
    value = statistics.median(vals)
    sample = f"{n} contiguous rows (of {sz['rows']}) x R={R} via RowKernel::compute+fill_row, {s:.2f} s"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "probs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": n * R / value * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (config-defined grids; no external data)",
        "config": bench_config(args.workload, sz, world),
        "cpu_baseline": {"value": value, "unit": "probs/s", "cores": th, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "probs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_legs(args, cfg_text, sz) -> dict:
    """The GPU arm's CPU baselines, run before any CUDA work in this process (the
    reference in its own processes, the host otherwise idle): the reference arm's
    row-kernel sample (one warm-up sample, then the timed one) and one reference
    Bellman step over the whole workload."""
    out = {}
    try:
        cpu_sample(cfg_text, sz["rows"], args.cpu_seconds / 2)
        v, n, Rr, th, s = cpu_sample(cfg_text, sz["rows"], args.cpu_seconds / 2)
        out["cpu_baseline"] = {"value": v, "unit": "probs/s", "cores": th, "kind": "reference",
                               "sample": f"{n} contiguous rows (of {sz['rows']}) x R={Rr} via "
                                         f"RowKernel::compute+fill_row, {s:.2f} s (before any CUDA work)"}
    except Exception as e:  # noqa: BLE001
        out["cpu_baseline"] = {"value": None, "error": str(e)}
    try:  # the sweep half of the metric: one reference Bellman step on the same workload
        secs, th = cpu_sweep_step(cfg_text, sz["states"])
        T = sz["horizon"]
        out["cpu_baseline_sweep"] = {
            "value": secs * T, "unit": "s", "cores": th, "kind": "reference", "step_s": secs,
            "sample": f"one OFA bellman_step over all {sz['rows']} rows (x{T} steps = a sweep); the stored-matrix "
                      f"mode needs the {sz['rows'] * sz['row_width'] * 8 / 1e9:.0f} GB matrix in host RAM"}
    except Exception as e:  # noqa: BLE001
        out["cpu_baseline_sweep"] = {"value": None, "error": str(e)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="C2b")
    ap.add_argument("--extra", default="C5", help="comma list of extra OFA workloads timed once (sweep only)")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--exchange", default="auto", choices=["auto", "halo", "allgather"],
                    help="V exchange between ranks (N > 1)")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()

    W = load_workloads()
    cfg_text = W.WORKLOADS[args.workload]()
    if args.impl == "reference":
        reference_arm(args, cfg_text, ref_sizes(cfg_text))
        return
    cpu = {}
    if int(os.environ.get("RANK", "0")) == 0 and int(os.environ.get("WORLD_SIZE", "1")) == 1 and not args.no_cpu:
        try:
            cpu = cpu_legs(args, cfg_text, ref_sizes(cfg_text))
        except Exception as e:  # noqa: BLE001
            cpu = {"cpu_baseline": {"value": None, "error": str(e)}}

    import torch
    import torch.distributed as dist

    from paper_2005_06191_b200 import _capi
    from paper_2005_06191_b200 import gridmdp as g
    from paper_2005_06191_b200 import sharded as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    _capi.call("gm_set_device", local)
    # under torchrun (any N, including 1) the NCCL path is the one exercised
    if world > 1 or ("MASTER_ADDR" in os.environ and "RANK" in os.environ):
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    m = g.parse_config(cfg_text, args.workload)
    sz = m.sizes()
    n_x, T, R = int(sz.n_states), int(sz.horizon), int(sz.row_width)
    nuw = int(sz.n_inputs) * int(sz.n_disturbances)
    reach = m.spec.is_reach()
    matrix = m.options.mode == "matrix"
    plan = S.ShardPlan(n_x, world, rank)
    my_rows = (plan.x1 - plan.x0) * nuw
    stream = torch.cuda.current_stream()
    be = S.DeviceBackend(m, stream)
    # V exchange for N > 1, planned once per model: the shards' cutoff-bounded halos
    # (point-to-point) when they are at most half the all-gather, else the all-gather
    xplan = S.exchange_plan(be, plan, None, args.exchange) if world > 1 else None
    exchange = xplan if xplan is not None else "allgather"

    def one_step():
        ev = {}

        def mark(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            ev[name] = e

        S.synthesize_sharded(be, n_x, T, reach, matrix, dev, None, mark, exchange=exchange)
        return ev

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
    lib = _capi.lib
    lib.gm_reset_kernel_stats()
    lib.gm_enable_kernel_timing(1)
    launches0 = lib.gm_launch_count()
    build_ms, sweep_ms = [], []
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        evs = [one_step() for _ in range(args.steps)]
        t1.record(stream)
        torch.cuda.synchronize()
    launches = lib.gm_launch_count() - launches0
    lib.gm_enable_kernel_timing(0)
    store_ceiling = store_ceiling_ms(be, stream) if matrix else None
    be.release()  # free the shard's matrix before the end-to-end run allocates its own
    torch.cuda.empty_cache()
    for ev in evs:
        build_ms.append(ev["build_start"].elapsed_time(ev["build_end"]))
        sweep_ms.append(ev["build_end"].elapsed_time(ev["sweep_end"]))
    total_ms = t0.elapsed_time(t1)
    fam_ms = {n: lib.gm_kernel_ms_total(i) for i, n in enumerate(_capi.KF_NAMES)}
    fam_n = {n: lib.gm_kernel_launches(i) for i, n in enumerate(_capi.KF_NAMES)}

    t = torch.tensor([total_ms, sum(build_ms), sum(sweep_ms)], dtype=torch.float64, device=dev)
    if dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, bsum, ssum = t.tolist()
    rows_all = int(sz.rows)
    probs_per_step = rows_all * R
    value = probs_per_step * args.steps / (bsum / 1e3) if matrix and bsum > 0 else None
    terms_per_step = rows_all * R * T
    sweep_s = ssum / args.steps / 1e3

    hbm, peak_kind = peaks()
    dom = "expect_matrix" if matrix else "expect_ofa"
    dom_ms = fam_ms[dom] / max(fam_n[dom], 1)
    # algorithmic bytes: per non-absorbed row its stored T row + origin (+ T0x); absorbed
    # rows are never read (synthesis.cpp:86-89), as in the reference
    live_rows = my_rows
    if reach:
        ab = g.absorbing_states(m, m.spec)[plan.x0:plan.x1]
        live_rows = int((ab == 0).sum()) * nuw
    dom_bytes = live_rows * (R * 8 + 8 + (8 if reach else 0))
    tpr = 1  # threads per row (tpr_for_width, gm_host.cpp): a power of two ~R/16 in [1, 128]
    while tpr * 2 <= R // 16 and tpr < 128:
        tpr *= 2
    kname = ("k_expect_matrix_et2" if tpr == 32 else "k_expect_matrix_et") if matrix else "k_expect_ofa"
    roofline = {"kernel": kname, "family": dom, "bound": "hbm", "achieved": dom_bytes / (dom_ms / 1e3) / 1e9, "peak": hbm,
                "peak_kind": peak_kind, "unit": "GB/s", "traffic": ncu_traffic(dom, args.workload),
                "algorithmic_bytes_per_launch": dom_bytes, "avg_launch_ms": dom_ms, "launches": fam_n[dom]}
    roofline["frac"] = roofline["achieved"] / hbm
    if not matrix:
        roofline["note"] = "OFA: HBM-equivalent bytes (8 per recomputed term), SURVEY.md §8d"
    exp_ms = fam_ms["build"] / max(fam_n["build"], 1)
    build_bytes = my_rows * (R * 8 + 8 + (8 if reach else 0))  # rows written + origins (+ T0x)
    roofline_build = {"kernel": "k_build_ws", "bound": "hbm",
                      "achieved": build_bytes / (exp_ms / 1e3) / 1e9 if exp_ms > 0 else None, "peak": hbm,
                      "unit": "GB/s", "algorithmic_bytes_per_launch": build_bytes, "avg_launch_ms": exp_ms,
                      "traffic": ncu_traffic("k_build_ws", args.workload)}
    if roofline_build["achieved"]:
        roofline_build["frac"] = roofline_build["achieved"] / hbm
        if store_ceiling:  # build time against a plain fill of the same bytes in the same regime
            roofline_build["frac_of_store_ceiling"] = store_ceiling["ms"] / exp_ms

    line = {
        "metric": METRIC, "value": value, "unit": "probs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",  # C2b's states sharded over the ranks
        "data": "synthetic (config-defined grids; no external data)",
        "config": bench_config(args.workload, {"states": n_x, "rows": rows_all, "row_width": R, "horizon": T}, world),
        "v_exchange": ("none" if world == 1 else
                       f"halo p2p ({xplan.halo_states} of {xplan.allgather_states} all-gather states)"
                       if xplan is not None else "all-gather per step"),
        "build_ms_per_step": bsum / args.steps, "sweep_s": sweep_s,
        "sweep_terms_per_s": terms_per_step / sweep_s if sweep_s > 0 else None,
        "kernel_ms_per_step": {k: v / args.steps for k, v in fam_ms.items() if v},
        "gpu_launches": int(launches),
        "roofline": roofline, "roofline_build": roofline_build, "store_ceiling": store_ceiling,
        "clocks": clk.summary(),
    }

    # e2e: the same metric (MDP probs/s of stage (i)) through the public C ABI from
    # host data: each step parses the configuration text on the host, uploads the
    # model (bytecode, line table, absorbing flags), builds this rank's shard with
    # gm_build_shard_host, which streams the shard's origins + target-hit vector into
    # pinned host memory slice by slice; wall clock, max over ranks.
    if not args.no_e2e:
        import ctypes as C

        nrow = my_rows
        h_org = torch.empty(max(nrow, 1), dtype=torch.int64, pin_memory=True)
        h_t0x = torch.empty(max(nrow, 1), dtype=torch.float64, pin_memory=True)

        def e2e_step():
            m3 = g.parse_config(cfg_text, args.workload)
            h = C.c_void_p()
            # build in slices; each slice's origins / T0x reach the pinned host buffers
            # while the next slice builds
            _capi.call("gm_build_shard_host", m3.handle, C.c_int64(plan.x0), C.c_int64(plan.x1), C.byref(h),
                       C.c_void_p(h_org.data_ptr()), C.c_void_p(h_t0x.data_ptr()) if reach else None)
            _capi.lib.gm_matrix_free(h)
            return m3

        for _ in range(args.warmup):
            e2e_step()
        e2e = []
        m3 = None
        for _ in range(args.steps):
            m3 = None  # the previous step's model is torn down outside the timed region
            torch.cuda.synchronize()
            if dist.is_initialized():
                dist.barrier()
            a = time.perf_counter()
            m3 = e2e_step()
            torch.cuda.synchronize()
            dt = torch.tensor([time.perf_counter() - a], dtype=torch.float64, device=dev)
            if dist.is_initialized():
                dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            e2e.append(float(dt.item()))
        prog_bytes = int(_capi.lib.gm_model_program_size(m3.handle)) * 8
        n_lines = R // int(sz.extents[int(sz.n_dim) - 1])
        h2d = prog_bytes + 4 * n_lines  # dynamics bytecode + literals, slab line table (config text stays host)
        d2h = nrow * 8 * (2 if reach else 1)
        line["e2e"] = {"value": probs_per_step / statistics.median(e2e), "unit": "probs/s",
                       "seconds_per_step": statistics.median(e2e), "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h,
                       "note": "config text -> gm_build_shard_host (origins/T0x to pinned host, overlapped) , wall clock"}
        # the full user-facing synthesis (rank 0, one GPU): host text -> value/policy tables on host
        if world == 1:
            t = time.perf_counter()
            res = g.synthesize(g.parse_config(cfg_text, args.workload))
            line["e2e_synthesize"] = {
                "seconds": time.perf_counter() - t,
                "d2h_bytes": int(res.values.nbytes + res.policy.nbytes + res.worst_dist.nbytes + res.absorbing.nbytes)}

    # extra OFA workloads (north-star BMW C5): sweep time only, one run after one warm
    # run; under torchrun the states are sharded over the N ranks like the main
    # workload (same V exchange policy) and the time is the max over ranks
    if args.extra:
        extra = {}
        for wname in [w for w in args.extra.split(",") if w]:
            mt = g.parse_config(W.WORKLOADS[wname](), wname)
            st = mt.sizes()
            nxt = int(st.n_states)
            bet = S.DeviceBackend(mt, stream)
            xp = S.exchange_plan(bet, S.ShardPlan(nxt, world, rank), None, args.exchange) if world > 1 else None
            ex = xp if xp is not None else "allgather"
            S.synthesize_sharded(bet, nxt, int(st.horizon), mt.spec.is_reach(), False, dev, exchange=ex)
            torch.cuda.synchronize()
            if dist.is_initialized():
                dist.barrier()
            lib.gm_reset_kernel_stats()
            lib.gm_enable_kernel_timing(1)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            S.synthesize_sharded(bet, nxt, int(st.horizon), mt.spec.is_reach(), False, dev, exchange=ex)
            b.record(stream)
            torch.cuda.synchronize()
            lib.gm_enable_kernel_timing(0)
            tms = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
            if dist.is_initialized():
                dist.all_reduce(tms, op=dist.ReduceOp.MAX)
            ms = float(tms.item())
            terms = int(st.rows) * int(st.row_width) * int(st.horizon)
            ofa_ms = lib.gm_kernel_ms_total(_capi.KF_EXPECT_OFA)
            extra[wname] = {"sweep_s": ms / 1e3, "terms_per_s": terms / (ms / 1e3), "n_gpus": world,
                            "hbm_equiv_frac": terms * 8 / (ms / 1e3) / 1e9 / (hbm * world),
                            "kernel_ms": {n: lib.gm_kernel_ms_total(i) for i, n in enumerate(_capi.KF_NAMES)
                                          if lib.gm_kernel_ms_total(i)},  # rank 0
                            "expect_ofa_terms_per_s": (terms / world) / (ofa_ms / 1e3) if ofa_ms else None,
                            "v_exchange": ("none" if world == 1 else
                                           f"halo p2p ({xp.halo_states} of {xp.allgather_states} states)"
                                           if xp is not None else "all-gather per step"),
                            "rows": int(st.rows), "row_width": int(st.row_width), "horizon": int(st.horizon),
                            # OFA reads (almost) nothing from DRAM: its ceiling is the L1/TEX pipe that
                            # serves the V gathers and the shared-memory tables (ncu, committed profile)
                            "roofline_l1tex": ncu_l1tex(wname),
                            "kernel_variant": _capi.lib.gm_last_kernel_variant(_capi.KF_EXPECT_OFA).decode()}
            bet.release()
            if world == 1:  # the user-level call: gridmdp.synthesize, value / policy tables on the host
                del g.synthesize(mt, mt.spec, g.SynthesisOptions(mode="ofa")).values  # warm (first-call setup)
                t0 = time.perf_counter()
                res = g.synthesize(mt, mt.spec, g.SynthesisOptions(mode="ofa"))
                extra[wname]["e2e_synthesize"] = {
                    "seconds": time.perf_counter() - t0,
                    "d2h_bytes": int(res.values.nbytes + res.policy.nbytes + res.worst_dist.nbytes),
                    "note": "wall clock of one call after a warm call (first-call setup: ~0.75 s, "
                            "scripts/c5_e2e_probe.py)"}
                del res
                g.release_cached_memory()
        line["extra"] = extra

    line.update(cpu)
    if line.get("cpu_baseline_sweep", {}).get("value") and sweep_s:
        line["cpu_baseline_sweep"]["gpu_speedup_sweep"] = line["cpu_baseline_sweep"]["value"] / sweep_s
        if "e2e_synthesize" in line:  # the whole user-level synthesis against the reference's (OFA: T steps)
            line["e2e_synthesize"]["reference_synthesize_s"] = line["cpu_baseline_sweep"]["value"]
            line["e2e_synthesize"]["speedup_vs_reference"] = (line["cpu_baseline_sweep"]["value"] /
                                                              line["e2e_synthesize"]["seconds"])
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
