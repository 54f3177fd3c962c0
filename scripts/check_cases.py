"""Small workloads that launch every device kernel of the engine, for the
bounds-checked library (GM_LIB=checked: libgridmdp_b200_checked.so, built with
-DGM_CHECKED: shared-memory layout vs the launch's dynamic size, every row's V slab
inside V, element / line tables, consumer compaction indices, specialised-fill
addresses). compute-sanitizer is closed on the GPU pool; tests/test_gpu_checked.py
runs these scenarios under the checked build instead. One scenario per process:
the kernel-selection knobs are read once per process.

  GM_LIB=checked python scripts/check_cases.py <scenario>

Each scenario prints the kernel variants it launched (gm_last_kernel_variant) and
checks its values against the reference goldens, so a checked run is also a
parity run of the same launches.
"""
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))

import numpy as np  # noqa: E402

import golden_io as G  # noqa: E402
from paper_2005_06191_b200 import _capi  # noqa: E402
from paper_2005_06191_b200 import gridmdp as g  # noqa: E402
from paper_2005_06191_b200 import workloads as W  # noqa: E402

MAN = G.manifest()


def model(case, **kw):
    return g.load_config(str(G.case_cfg(case)), **G.case_overrides(MAN["cases"][case]), **kw)


def variants():
    return {n: _capi.lib.gm_last_kernel_variant(i).decode() for i, n in enumerate(_capi.KF_NAMES)
            if _capi.lib.gm_last_kernel_variant(i)}


def synth_both(case):
    m = model(case)
    ref = G.golden_results(case)["values"]
    out = {}
    for mode in ("matrix", "ofa"):
        r = g.synthesize(m, m.spec, g.SynthesisOptions(mode=mode))
        assert G.tol_ok(r.values, ref).all(), (case, mode)
        out[mode] = variants()
    return m, out


def r729():
    text = W.vehicle3(eta=(0.125, 0.125, 0.0625), T=3)
    for a, b in (("states.ub = {10.0, 10.0, 3.5};", "states.ub = {2.0, 2.0, 1.5};"),
                 ("target.lb = {8.0, 0.0, -3.5};", "target.lb = {1.5, 0.0, -3.5};"),
                 ("target.ub = {10.0, 2.0, 3.5};", "target.ub = {2.0, 0.5, 1.5};"),
                 ("avoid.lb = {4.0, 4.0, -3.5};", "avoid.lb = {0.75, 0.75, -3.5};"),
                 ("avoid.ub = {6.0, 6.0, 3.5};", "avoid.ub = {1.25, 1.25, 1.5};")):
        text = text.replace(a, b)
    return g.parse_config(text, "vehicle_r729")


def scenario(name):
    if name == "core":  # interpreter build, matrix / OFA sweeps, mask, target hit, maxmin, absorbing
        m, v = synth_both("fixture2d_ra")
        tm = g.build_matrix(m)
        g.mask_absorbing(tm, m.spec)
        g.build_target_hit(m, m.spec)
        print(v)
        for case in ("ref_vehicle3_desk", "room5_uni", "exp_dist", "beta1d", "mult1d", "degenerate"):
            print(case, synth_both(case)[1])
    elif name == "jit":  # NVRTC-compiled build / prologue, shape-specialised fill
        for case in ("fixture2d_ra", "ref_vehicle3_desk"):
            print(case, synth_both(case)[1])
        m = r729()
        a = g.synthesize(m, m.spec, g.SynthesisOptions(mode="matrix"))
        b = g.synthesize(m, m.spec, g.SynthesisOptions(mode="ofa"))
        assert np.array_equal(a.values, b.values)
        print("vehicle_r729", variants())
    elif name == "et2":  # two rows per warp at TPR 32 (R = 729), and the one-row variant
        m = r729()
        a = g.synthesize(m, m.spec, g.SynthesisOptions(mode="matrix"))
        b = g.synthesize(m, m.spec, g.SynthesisOptions(mode="ofa"))
        assert np.array_equal(a.values, b.values)
        print("vehicle_r729", variants())
    elif name == "ofa_pk":  # hoisted last-axis cell (GM_OFA_PK=1) + table modes via env
        for case in ("fixture2d_ra", "ref_vehicle3_desk", "ref_traffic3_desk", "beta1d"):
            m = model(case)
            r = g.synthesize(m, m.spec, g.SynthesisOptions(mode="ofa"))
            assert G.tol_ok(r.values, G.golden_results(case)["values"]).all(), case
            print(case, variants())
    elif name == "custom":  # custom densities: quadrature build (k_build_custom), matrix and OFA
        for case in ("custom_tri1d", "custom_tri2d"):
            print(case, synth_both(case)[1])
    elif name == "sim":  # closed-loop simulator
        m = model("fixture2d_ra")
        res = g.synthesize(m)
        runs, seed = 4096, 7
        b = g.simulate(m, m.spec, res, np.array([0.5, 0.5]), runs, seed, "random", trajectories=True)
        w = g.simulate(m, m.spec, res, np.array([0.5, 0.5]), runs, seed, "worst_case")
        print("sim", g.empirical_rate(b), g.empirical_rate(w), variants())
    elif name == "multi":  # in-process multi-device driver, peer copies, halo and all-gather
        m = model("ref_vehicle3_desk")
        ref = g.synthesize(m)
        for ex in ("halo", "allgather"):
            got, st = g.synthesize_multi(m, [0, 0, 0], exchange=ex, transport="peer")
            assert np.array_equal(got.values, ref.values)
        print("multi", variants())
    elif name == "build_single":  # single-role build (GM_BUILD_WS=0), slab-walk matrix kernel
        for case in ("fixture2d_ra", "ref_traffic3_desk", "beta1d"):
            print(case, synth_both(case)[1])
    else:
        raise SystemExit(f"unknown scenario {name}")
    print("scenario", name, "ok")


if __name__ == "__main__":
    scenario(sys.argv[1])
