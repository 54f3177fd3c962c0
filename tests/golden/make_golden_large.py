"""Full-size / full-horizon golden fixtures from the REFERENCE itself (oracle/_ref).

Companion of make_golden.py for the BASELINE.json configurations,
where the small hand cases say nothing about long horizons and wide rows:

  C5   bmw7.cfg, reach-avoid, T = 32, OFA     (the north star; ~12 min on 8 cores)
  C1   robot_reachavoid.cfg --time-steps 8   (BASELINE configs[0], the CPU-oracle run)
  C2a  vehicle3.cfg at its own T = 32
  bmw7_mid  bmw7 dynamics on a 4x4 position grid, T = 8 (nonzero values with an
            absorbing target, fast enough for every GPU test run)
  C2b  one bellman_step (OFA ≡ matrix in the reference, test_cli.cpp:104-124) of
       vehicle3 at eta/4 with a hashed v_next, recorded on every 16th state

Results are `gridmdp-results 1` containers exactly as the reference's
write_results produced them (io.cpp:142-179), gzipped. Only this container has
/root/reference; the GPU box reads the committed files.
Usage: python tests/golden/make_golden_large.py [name ...]
"""
from __future__ import annotations

import gzip
import importlib.util
import json
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
REF_BIN = REPO / "oracle" / "_ref" / "gridmdp_ref"
REF_CFG = Path("/root/reference/proj/configs")
OUT = HERE / "large"

sys.path.insert(0, str(HERE))
from make_golden import canonical  # noqa: E402


def _workloads():
    # by path: the package __init__ would load the engine library
    spec = importlib.util.spec_from_file_location("_wl", REPO / "paper_2005_06191_b200" / "workloads.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def hashed_v(n: int) -> np.ndarray:
    """Deterministic v_next in [0,1): splitmix64 of the state index, top 53 bits.
    Restated by tests/golden_io.hashed_v (no fixture needed for the input)."""
    z = np.arange(n, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def bmw7_mid() -> str:
    wl = _workloads()
    text = wl.bmw7(T=8, mode="ofa")
    text = text.replace("states.lb = {-10.0, -10.0,", "states.lb = {-3.0, -3.0,")
    text = text.replace("states.ub = {10.0, 10.0,", "states.ub = {3.0, 3.0,")
    text = text.replace("states.eta = {4.0, 4.0,", "states.eta = {2.0, 2.0,")
    return text


SYNTH = {
    # name: (config text producer, extra flags)
    "C1": (lambda: canonical(REF_CFG / "robot_reachavoid.cfg"), ["--time-steps", "8"]),
    "C2a": (lambda: canonical(REF_CFG / "vehicle3.cfg"), []),
    "bmw7_mid": (bmw7_mid, []),
    "C5": (lambda: canonical(REF_CFG / "bmw7.cfg"), []),
}
STEP_STRIDE = 16


def ref(*args) -> str:
    p = subprocess.run([str(REF_BIN), *map(str, args)], capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"{args}: rc={p.returncode}\n{p.stderr}")
    return p.stdout


def main(names) -> None:
    if not REF_BIN.exists():
        sys.exit("build oracle/_ref first: make -C oracle ref")
    OUT.mkdir(exist_ok=True)
    mpath = OUT / "manifest.json"
    manifest = json.loads(mpath.read_text()) if mpath.exists() else {}
    for name in names:
        t0 = time.time()
        if name in SYNTH:
            producer, extra = SYNTH[name]
            cfg = OUT / f"{name}.cfg"
            cfg.write_text(producer())
            res = OUT / f"_{name}.results.bin"
            log = ref("synthesize", "-c", cfg, "-o", res, "--mode", "ofa", "--threads", "0", *extra)
            (OUT / f"{name}.results.bin.gz").write_bytes(gzip.compress(res.read_bytes(), 9, mtime=0))
            res.unlink()
            manifest[name] = {"kind": "synthesize", "config": cfg.name, "overrides": extra,
                              "results": f"{name}.results.bin.gz", "sizes": _sizes(cfg, extra),
                              "ref_log": log.strip().splitlines()}
        elif name == "C2b_step":
            cfg = OUT / "C2b.cfg"
            cfg.write_text(_workloads().WORKLOADS["C2b"]().replace("exec.mode = matrix;", "exec.mode = ofa;"))
            sizes = _sizes(cfg, [])
            n_x = sizes["states"]
            vf = OUT / "_C2b.vnext.f64"
            hashed_v(n_x).astype("<f8").tofile(vf)
            pre = OUT / "_C2b.step"
            log = ref("step", "-c", cfg, "--vnext", vf, "-o", pre, "--mode", "ofa", "--threads", "0")
            v = np.fromfile(f"{pre}.v", "<f8")
            pol = np.fromfile(f"{pre}.pol", "<u4")
            wst = np.fromfile(f"{pre}.wst", "<u4")
            idx = np.arange(0, n_x, STEP_STRIDE)
            blob = {"v": v[idx], "pol": pol[idx], "wst": wst[idx]}
            for k, a in blob.items():
                (OUT / f"C2b_step.{k}.gz").write_bytes(gzip.compress(a.tobytes(), 9, mtime=0))
            for f in (vf, Path(f"{pre}.v"), Path(f"{pre}.pol"), Path(f"{pre}.wst")):
                f.unlink()
            manifest[name] = {"kind": "step", "config": cfg.name, "stride": STEP_STRIDE, "v_next": "hashed_v",
                              "sizes": sizes, "nonzero": int(np.count_nonzero(v)),
                              "ref_log": log.strip().splitlines()}
        else:
            raise SystemExit(f"unknown golden {name}")
        manifest[name]["generate_s"] = round(time.time() - t0, 1)
        mpath.write_text(json.dumps(manifest, indent=1, sort_keys=True))
        print(name, manifest[name]["generate_s"], "s", flush=True)


def _sizes(cfg: Path, extra) -> dict:
    d = {}
    for line in ref("estimate", "-c", cfg, *extra).splitlines():
        k, v = line.split(":", 1)
        d[k] = [int(x) for x in v.split()] if k == "window" else int(v)
    return d


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2a", "C1", "bmw7_mid", "C2b_step", "C5"])
