"""The drop-in at the reference's own C++ types (integration/gridmdp_b200_adapter.cpp):
oracle/ref_driver.cpp — a client of the reference's public API — linked against the
unmodified reference objects with build_matrix / build_target_hit / synthesize /
synthesize_with_matrix / bellman_step weakened, so the adapter's definitions (the
B200 engine behind include/gridmdp_b200.h) are the ones it calls.

CPU: the binary reaches the engine and fails loudly without a device (no CPU
fallback). GPU: its containers are byte-identical to the engine CLI's and within
the parity bar of the reference's own (golden) outputs."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

import golden_io as G
from paper_2005_06191_b200 import _capi

REPO = Path(__file__).resolve().parents[1]
BIN = REPO / "integration" / "_build" / "ref_on_b200"
MAN = G.manifest()
pytestmark = pytest.mark.skipif(not BIN.exists(), reason="integration/_build/ref_on_b200 not built (needs the reference tree)")


def run(*args):
    return subprocess.run([str(BIN), *map(str, args)], capture_output=True, text=True)


def test_reference_api_reaches_the_engine_without_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    r = run("synthesize", "-c", G.case_cfg("fixture2d_ra"), "-o", "/tmp/_never.bin")
    assert r.returncode == 1
    assert "no CUDA device available: the B200 engine has no CPU fallback" in r.stderr


def test_reference_front_end_untouched():
    """estimate goes through the reference's own (not replaced) code."""
    r = run("estimate", "-c", G.case_cfg("fixture2d_ra"))
    assert r.returncode == 0
    assert f"rows: {MAN['cases']['fixture2d_ra']['sizes']['rows']}\n" in r.stdout


CASES = ["fixture2d_ra", "ref_vehicle3_desk", "ref_bmw7_desk", "room5_uni", "exp_dist", "beta1d", "mult1d", "chain09"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("mode", ["matrix", "ofa"])
def test_reference_synthesize_on_engine(case, mode, tmp_path):
    ov = [str(x) for x in MAN["cases"][case].get("overrides", [])]
    a, b = tmp_path / "adapter.bin", tmp_path / "engine.bin"
    r = run("synthesize", "-c", G.case_cfg(case), "-o", a, "--mode", mode, *ov)
    assert r.returncode == 0, r.stderr
    e = subprocess.run([str(_capi.CLI_PATH), "synthesize", "-c", str(G.case_cfg(case)), "-o", str(b), "--mode", mode,
                        *ov], capture_output=True, text=True)
    assert e.returncode == 0, e.stderr
    # the reference's write_results over the adapter's SynthesisResult == the engine's own container
    assert a.read_bytes() == b.read_bytes()
    got = G.read_results(a.read_bytes())
    ref = G.golden_results(case)
    assert got["manifest"] == dict(ref["manifest"], mode=mode)
    assert G.tol_ok(got["values"], ref["values"]).all()
    assert np.array_equal(got["absorbing"], ref["absorbing"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["fixture2d_ra", "exp_dist", "beta1d", "degenerate"])
def test_reference_build_matrix_on_engine(case, tmp_path):
    out = tmp_path / "m.bin"
    r = run("matrix", "-c", G.case_cfg(case), "-o", out)
    assert r.returncode == 0, r.stderr
    got = G.read_matrix(out.read_bytes())
    want = G.read_matrix(G.load(MAN["cases"][case]["files"]["matrix"]))
    assert got["manifest"] == want["manifest"]
    assert np.array_equal(got["origins"], want["origins"])
    assert G.tol_ok(got["probs"], want["probs"]).all()


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(c for c, e in MAN["cases"].items() if "step_prefix" in e.get("files", {})))
@pytest.mark.parametrize("mode", ["matrix", "ofa"])
def test_reference_bellman_step_on_engine(case, mode, tmp_path):
    try:
        vn, v, p, w = G.golden_step(case, mode)
    except FileNotFoundError:
        pytest.skip("no golden step for this mode")
    vf = tmp_path / "vnext.f64"
    vn.astype("<f8").tofile(vf)
    pre = tmp_path / "s"
    ov = [str(x) for x in MAN["cases"][case].get("overrides", [])]
    r = run("step", "-c", G.case_cfg(case), "--vnext", vf, "-o", pre, "--mode", mode, *ov)
    assert r.returncode == 0, r.stderr
    got = np.fromfile(f"{pre}.v", "<f8")
    assert G.tol_ok(got, v).all(), np.abs(got - v).max()


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["ref_vehicle3_desk", "fixture2d_ra"])
def test_reference_synthesize_on_several_devices(case, tmp_path):
    """GRIDMDP_B200_DEVICES routes the reference's synthesize to gm_synthesize_multi
    (one GPU here: the device repeated, peer transport); same container bytes."""
    import os
    a, b = tmp_path / "one.bin", tmp_path / "multi.bin"
    assert run("synthesize", "-c", G.case_cfg(case), "-o", a).returncode == 0
    env = dict(os.environ, GRIDMDP_B200_DEVICES="0,0,0", GRIDMDP_B200_TRANSPORT="peer")
    r = subprocess.run([str(BIN), "synthesize", "-c", str(G.case_cfg(case)), "-o", str(b)], capture_output=True,
                       text=True, env=env)
    assert r.returncode == 0, r.stderr
    assert a.read_bytes() == b.read_bytes()


@pytest.mark.gpu
def test_reference_synthesize_on_engine_bmw_full_horizon(tmp_path):
    """The north-star dynamics through the reference's in-memory types (every BMW
    expression crosses as its Expr node pool, gm_model_desc): bmw7_mid (1.75 M rows x
    15,750, T = 8, OFA) equals the engine CLI's container byte for byte and the
    reference's own full-horizon result within the parity bar (nonzero values)."""
    cfg = G.large_cfg("bmw7_mid")
    a, b = tmp_path / "adapter.bin", tmp_path / "engine.bin"
    r = run("synthesize", "-c", cfg, "-o", a)
    assert r.returncode == 0, r.stderr
    e = subprocess.run([str(_capi.CLI_PATH), "synthesize", "-c", str(cfg), "-o", str(b)], capture_output=True, text=True)
    assert e.returncode == 0, e.stderr
    assert a.read_bytes() == b.read_bytes()
    got = G.read_results(a.read_bytes())
    ref = G.large_results("bmw7_mid")
    assert np.count_nonzero(ref["values"]) > 0
    assert G.tol_ok(got["values"], ref["values"]).all()
