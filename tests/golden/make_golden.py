"""Regenerates the golden fixtures under tests/golden/ from the REFERENCE itself.

Runs oracle/_ref/gridmdp_ref (the unmodified reference sources compiled by
oracle/Makefile against the Eigen storage shim) on:
  * the hand-made cases in tests/golden/cases/*.cfg (restating the reference's
    own test fixtures, file:line in each header), and
  * canonical re-serialisations of selected bundled configs from
    /root/reference/proj/configs (written to tests/golden/cases/ref_*.cfg),
and records the reference's outputs: `gridmdp-results 1` containers (matrix and
OFA), raw `gridmdp-matrix 1` dumps (small cases), target-hit vectors, one
bellman_step with a seeded random v_next, and the estimate-mem sizes.

Only this container has /root/reference; the GPU box uses the committed files.
Usage: python tests/golden/make_golden.py
"""
from __future__ import annotations

import gzip
import json
import re
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
REF_BIN = REPO / "oracle" / "_ref" / "gridmdp_ref"
REF_CFG = Path("/root/reference/proj/configs")
CASES = HERE / "cases"
OUT = HERE / "out"

# bundled configs restated as canonical cases: name -> (cfg, extra overrides, modes)
BUNDLED = {
    "vehicle3_desk": ("vehicle3_desk.cfg", [], ["matrix", "ofa"]),
    "bmw7_desk": ("bmw7_desk.cfg", [], ["matrix", "ofa"]),
    "traffic3_desk": ("traffic3_desk.cfg", [], ["matrix", "ofa"]),
    "traffic5_desk": ("traffic5_desk.cfg", [], ["ofa"]),
    "room3": ("room3.cfg", [], ["matrix", "ofa"]),
    "room5": ("room5.cfg", [], ["matrix", "ofa"]),
    "vehicle3_T8": ("vehicle3.cfg", ["--time-steps", "8"], ["matrix", "ofa"]),
    "robot_safety_T2": ("robot_safety.cfg", ["--time-steps", "2"], ["ofa"]),
    "robot_reachavoid_T2": ("robot_reachavoid.cfg", ["--time-steps", "2"], ["ofa"]),
}
# hand cases: modes; small enough for matrix dumps
HAND_MODES = {
    "room5_beta": ["ofa"],
}
DUMP_LIMIT = 2_000_000  # bytes of stored matrix committed per case
STEP_CASES = ["fixture2d_ra", "fixture2d_safety", "vehicle3_desk", "bmw7_desk", "room5_exp", "exp_dist",
              "reach_uniform", "room3"]


def canonical(cfg_path: Path) -> str:
    """Re-serialises a reference config as sorted `key = value;` lines (no comments)."""
    stmts = {}
    for raw in cfg_path.read_text().splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        assert line.endswith(";"), line
        k, v = line[:-1].split("=", 1)
        stmts[k.strip()] = v.strip()
    return "".join(f"{k} = {stmts[k]};\n" for k in sorted(stmts))


def ref(*args, check=True) -> subprocess.CompletedProcess:
    p = subprocess.run([str(REF_BIN), *map(str, args)], capture_output=True, text=True)
    if check and p.returncode != 0:
        raise RuntimeError(f"{args}: rc={p.returncode}\n{p.stderr}")
    return p


def parse_sizes(text: str) -> dict:
    d = {}
    for line in text.splitlines():
        k, v = line.split(":", 1)
        v = v.strip()
        d[k] = [int(x) for x in v.split()] if k == "window" else int(v)
    return d


def main() -> None:
    if not REF_BIN.exists():
        sys.exit("build oracle/_ref first: make -C oracle ref")
    OUT.mkdir(exist_ok=True)
    for name, (cfg, _, _) in BUNDLED.items():
        (CASES / f"ref_{name}.cfg").write_text(
            f"# canonical restatement of /root/reference/proj/configs/{cfg}\n" + canonical(REF_CFG / cfg))

    manifest = {"cases": {}, "estimate": {}}
    # estimate-mem sizes of every bundled config (the fast acceptance check)
    for cfg in sorted(REF_CFG.glob("*.cfg")):
        text = canonical(cfg)
        tmp = OUT / f"_est_{cfg.stem}.cfg"
        tmp.write_text(text)
        manifest["estimate"][cfg.stem] = {"config": text, "sizes": parse_sizes(ref("estimate", "-c", tmp).stdout)}
        tmp.unlink()

    # front-end error behaviour: rc and message of the reference for bad inputs
    tiny = (CASES / "tiny.cfg").read_text()
    bad_inputs = {
        "no_semicolon": "states.dim = 1\n",
        "no_equals": "states.dim 1;\n",
        "empty_key": " = 1;\n",
        "duplicate": "states.dim = 1;\nstates.dim = 2;\n",
        "missing_lb": "states.dim = 1;\n",
        "bad_vector": tiny.replace("states.lb = {-1.0};", "states.lb = -1.0;"),
        "bad_number": tiny.replace("states.eta = {0.25};", "states.eta = {0.2x5};"),
        "unknown_key": tiny + "exec.gpus = 8;\n",
        "unknown_noise": tiny.replace("noise.type = normal;", "noise.type = cauchy;"),
        "bad_mode": tiny + "noise.mode = both;\n",
        "vec_size": tiny.replace("noise.sigma = {0.3};", "noise.sigma = {0.3, 0.3};"),
        "neg_eta": tiny.replace("states.eta = {0.25};", "states.eta = {-0.25};"),
        "lb_gt_ub": tiny.replace("states.lb = {-1.0};", "states.lb = {2.0};"),
        "sigma_zero": tiny.replace("noise.sigma = {0.3};", "noise.sigma = {0.0};"),
        "gamma_range": tiny.replace("noise.cutting_probability = 0.001;", "noise.cutting_probability = 2;"),
        "parse_ident": tiny.replace("0.7*x0 + 0.4*u0", "0.7*x0 + y0"),
        "parse_range": tiny.replace("0.7*x0 + 0.4*u0", "x1"),
        "parse_func": tiny.replace("0.7*x0 + 0.4*u0", "foo(x0)"),
        "parse_paren": tiny.replace("0.7*x0 + 0.4*u0", "(x0 + 1"),
        "parse_trailing": tiny.replace("0.7*x0 + 0.4*u0", "x0 1"),
        "parse_number": tiny.replace("0.7*x0 + 0.4*u0", "1.2.3*x0"),
        "parse_char": tiny.replace("0.7*x0 + 0.4*u0", "x0 $ 1"),
        "parse_arity": tiny.replace("0.7*x0 + 0.4*u0", "min(x0)"),
        "spec_kind": tiny.replace("spec.type = safety;", "spec.type = liveness;"),
        "spec_box": tiny.replace("spec.type = safety;", "spec.type = reachability;") +
        "target.lb = {0.5};\ntarget.ub = {3.0};\n",
        "spec_safety_box": tiny + "target.lb = {0.5};\ntarget.ub = {0.6};\n",
        "spec_horizon": tiny.replace("spec.time_steps = 3;", "spec.time_steps = 0;"),
    }
    manifest["errors"] = {}
    for name, text in bad_inputs.items():
        tmp = OUT / f"_bad_{name}.cfg"
        tmp.write_text(text)
        p = ref("synthesize", "-c", tmp, "-o", OUT / "_bad.bin", check=False)
        manifest["errors"][name] = {"config": text, "rc": p.returncode,
                                    "stderr": p.stderr.strip().replace(str(tmp), "<cfg>")}
        tmp.unlink()
        (OUT / "_bad.bin").unlink(missing_ok=True)

    cases = sorted(p.stem for p in CASES.glob("*.cfg"))

    def ref_case(cfgp: Path):
        """(reference config, extra flags): custom-density cases (engine-format keys
        noise.pdf / noise.support.*) run the reference through ref_driver --custom-*
        on the same config with a placeholder noise (NoiseSpec::custom, noise.cpp:75-85)."""
        text = cfgp.read_text()
        if "noise.type = custom;" not in text:
            return cfgp, []
        kv = {}
        keep = []
        for raw in text.splitlines():
            line = raw.split("#", 1)[0].strip()
            k = line.split("=", 1)[0].strip() if "=" in line else ""
            if k in ("noise.type", "noise.pdf", "noise.support.lb", "noise.support.ub"):
                kv[k] = line.split("=", 1)[1].strip().rstrip(";").strip()
            else:
                keep.append(raw)
        n = int(re.search(r"states.dim = (\d+);", text).group(1))
        keep += ["noise.type = normal;", "noise.sigma = {" + ", ".join(["1.0"] * n) + "};"]
        rp = OUT / f"_{cfgp.stem}.ref.cfg"
        rp.write_text("\n".join(keep) + "\n")
        return rp, ["--custom-pdf", kv["noise.pdf"], "--custom-lb", kv["noise.support.lb"], "--custom-ub",
                    kv["noise.support.ub"]]

    rng = np.random.default_rng(20240)  # robot_safety.cfg:34 seed
    for c in cases:
        cfgp0 = CASES / f"{c}.cfg"
        cfgp, custom = ref_case(cfgp0)
        bundled = c[4:] if c.startswith("ref_") else None
        extra = (BUNDLED[bundled][1] if bundled else []) + custom
        modes = BUNDLED[bundled][2] if bundled else HAND_MODES.get(c, ["matrix", "ofa"])
        entry = {"overrides": extra if not custom else (BUNDLED[bundled][1] if bundled else []), "modes": {},
                 "files": {}}
        if custom:
            entry["custom_density"] = True
        est = ref("estimate", "-c", cfgp, *extra)
        entry["sizes"] = parse_sizes(est.stdout)
        rows, R = entry["sizes"]["rows"], entry["sizes"]["row_width"]
        if c == "domain":
            p = ref("matrix", "-c", cfgp, "-o", OUT / "_dom.bin", check=False)
            entry["domain_error"] = {"rc": p.returncode, "stderr": p.stderr.strip()}
            manifest["cases"][c] = entry
            continue
        blobs = {}
        for mode in modes:
            f = OUT / f"{c}.{mode}.results.bin"
            ref("synthesize", "-c", cfgp, "-o", f, "--mode", mode, *extra)
            blobs[mode] = f.read_bytes()
            f.unlink()
        # the reference's own invariant (test_cli.cpp:104-124): containers of the two
        # modes differ only in the mode line, so one file per case is kept
        if len(blobs) == 2:
            assert blobs["matrix"].replace(b"mode = matrix;", b"mode = ofa;", 1) == blobs["ofa"], c
        keep = "ofa" if "ofa" in blobs else "matrix"
        f = OUT / f"{c}.results.bin.gz"
        f.write_bytes(gzip.compress(blobs[keep], 9, mtime=0))
        entry["results"] = f.name
        entry["results_mode"] = keep
        entry["modes"] = sorted(blobs)
        if rows * R * 8 <= DUMP_LIMIT:
            f = OUT / f"{c}.matrix.bin"
            ref("matrix", "-c", cfgp, "-o", f, *extra)
            entry["files"]["matrix"] = f.name
            f = OUT / f"{c}.prism.tra"
            ref("prism", "-c", cfgp, "-o", f, *extra)
            entry["files"]["prism"] = f.name
            if "spec.type = safety" not in cfgp0.read_text():
                f = OUT / f"{c}.masked.bin"
                ref("masked-matrix", "-c", cfgp, "-o", f, *extra)
                entry["files"]["masked"] = f.name
        if "spec.type = safety" not in cfgp0.read_text() and rows <= 100_000:
            f = OUT / f"{c}.t0x.f64"
            ref("target-hit", "-c", cfgp, "-o", f, *extra)
            entry["files"]["t0x"] = f.name
        if c in STEP_CASES or (bundled and bundled in STEP_CASES):
            n_x = entry["sizes"]["states"]
            v = rng.uniform(0.0, 1.0, n_x)
            vf = OUT / f"{c}.vnext.f64"
            v.astype("<f8").tofile(vf)
            for mode in ("ofa", "matrix") if rows * R * 8 < 2e9 else ("ofa",):
                ref("step", "-c", cfgp, "--vnext", vf, "-o", OUT / f"{c}.step_{mode}", "--mode", mode, *extra)
            entry["files"]["vnext"] = vf.name
            entry["files"]["step_prefix"] = f"{c}.step"
        manifest["cases"][c] = entry
        if custom:
            cfgp.unlink()
        print(c, entry["sizes"], list(entry["modes"]), list(entry["files"]), flush=True)
    for f in OUT.iterdir():  # compress the raw binaries
        if f.suffix != ".gz":
            f.with_name(f.name + ".gz").write_bytes(gzip.compress(f.read_bytes(), 9, mtime=0))
            f.unlink()
    (HERE / "manifest.json").write_text(json.dumps(manifest, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
