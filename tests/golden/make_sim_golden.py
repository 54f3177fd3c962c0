"""Simulation fixtures from the REFERENCE (sim.cpp via oracle/_ref/gridmdp_ref
`simulate`, the same code path as `gridmdp simulate`, tools/gridmdp_main.cpp:119-140).

For each case: the committed golden results container, an x0 (the representative
whose full-horizon value is closest to 0.5, so the empirical rate is far from 0
and 1), `runs` rollouts per disturbance mode; records the reference's
empirical rate, satisfied count and mean steps into tests/golden/sim.json, plus
one small trajectory CSV (format check). The GPU simulator draws from a
different generator (Philox, not mt19937_64), so tests compare rates
statistically. Only this container has oracle/_ref built from /root/reference.
Usage: python tests/golden/make_sim_golden.py
"""
from __future__ import annotations

import gzip
import json
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import golden_io as G  # noqa: E402

REF_BIN = HERE.parents[1] / "oracle" / "_ref" / "gridmdp_ref"
RUNS = 20000
SEED = 20240
CASES = ["fixture2d_ra", "fixture2d_safety", "ref_vehicle3_T8", "ref_robot_reachavoid_T2", "room5_exp",
         "room5_beta", "mult1d", "chain09", "reach_uniform", "custom_tri1d", "custom_tri2d"]


def ref_case(cfgp: Path, tmp: Path):
    """(reference config, flags): custom-density cases run through ref_driver --custom-* on the
    same config with a placeholder noise (as tests/golden/make_golden.py)."""
    import re
    text = cfgp.read_text()
    if "noise.type = custom;" not in text:
        return cfgp, []
    kv, keep = {}, []
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        k = line.split("=", 1)[0].strip() if "=" in line else ""
        if k in ("noise.type", "noise.pdf", "noise.support.lb", "noise.support.ub"):
            kv[k] = line.split("=", 1)[1].strip().rstrip(";").strip()
        else:
            keep.append(raw)
    n = int(re.search(r"states.dim = (\d+);", text).group(1))
    keep += ["noise.type = normal;", "noise.sigma = {" + ", ".join(["1.0"] * n) + "};"]
    rp = tmp / f"{cfgp.stem}.ref.cfg"
    rp.write_text("\n".join(keep) + "\n")
    return rp, ["--custom-pdf", kv["noise.pdf"], "--custom-lb", kv["noise.support.lb"], "--custom-ub",
                kv["noise.support.ub"]]


def grid_point(kv: dict, prefix: str, flat: int) -> list:
    lb = [float(x) for x in kv[prefix + ".lb"].strip("{}").split(",")]
    ub = [float(x) for x in kv[prefix + ".ub"].strip("{}").split(",")]
    eta = [float(x) for x in kv[prefix + ".eta"].strip("{}").split(",")]
    count = [int(np.floor((u - l) / e + 1e-9)) + 1 for l, u, e in zip(lb, ub, eta)]
    idx = []
    for c in reversed(count):
        idx.append(flat % c)
        flat //= c
    idx = idx[::-1]
    return [l + j * e for l, j, e in zip(lb, idx, eta)]


def main() -> None:
    man = G.manifest()
    out = {"runs": RUNS, "seed": SEED, "cases": {}}
    with tempfile.TemporaryDirectory() as d:
        for case in CASES:
            e = man["cases"][case]
            res = G.read_results(G.load(e["results"]))
            v0 = res["values"][:, 0]
            free = np.ones_like(v0, dtype=bool) if res["absorbing"].size == 0 else res["absorbing"] == 0
            cand = np.where(free)[0]
            ix = int(cand[np.argmin(np.abs(v0[cand] - 0.5))])
            x0 = grid_point(res["manifest"], "states", ix)
            rpath = Path(d) / f"{case}.results.bin"
            rpath.write_bytes(G.load(e["results"]))
            entry = {"x0": x0, "x0_index": ix, "value_at_x0": float(v0[ix]), "modes": {}}
            for dm in ("random", "worst-case"):
                cfg_ref, custom = ref_case(G.case_cfg(case), Path(d))
                args = [str(REF_BIN), "simulate", "-c", str(cfg_ref), *custom, "--results", str(rpath),
                        "--x0", "{" + ", ".join(repr(v) for v in x0) + "}", "--runs", str(RUNS), "--seed",
                        str(SEED), "--dist-mode", dm, "--threads", "0", *e.get("overrides", [])]
                txt = subprocess.run(args, capture_output=True, text=True, check=True).stdout
                kv = dict(line.split(": ", 1) for line in txt.strip().splitlines())
                entry["modes"][dm] = {"rate": float(kv["empirical_rate"]), "satisfied": int(kv["satisfied"]),
                                      "mean_steps": int(kv["steps_total"]) / RUNS}
            out["cases"][case] = entry
            print(case, x0, entry["value_at_x0"], entry["modes"])
        # one trajectory CSV (format check): 3 runs of fixture2d_ra
        e = man["cases"]["fixture2d_ra"]
        x0 = out["cases"]["fixture2d_ra"]["x0"]
        rpath = Path(d) / "fixture2d_ra.results.bin"
        csv = Path(d) / "traj.csv"
        subprocess.run([str(REF_BIN), "simulate", "-c", str(G.case_cfg("fixture2d_ra")), "--results", str(rpath),
                        "--x0", "{" + ", ".join(repr(v) for v in x0) + "}", "--runs", "3", "--seed", "7",
                        "--traj", str(csv)], check=True, capture_output=True)
        (G.OUT / "fixture2d_ra.traj.csv.gz").write_bytes(gzip.compress(csv.read_bytes(), mtime=0))
        out["traj_csv"] = {"case": "fixture2d_ra", "runs": 3, "seed": 7, "file": "fixture2d_ra.traj.csv"}
    (HERE / "sim.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
