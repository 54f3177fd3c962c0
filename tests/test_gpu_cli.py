"""The `gridmdp` CLI of the engine against the reference's outputs: result
containers (`synthesize`), raw matrix dumps (`abstract --dump-matrix`) and PRISM
explicit exports (`export-prism`), plus the domain-error exit code."""
import subprocess

import numpy as np
import pytest

import golden_io as G
from paper_2005_06191_b200 import _capi

pytestmark = pytest.mark.gpu
MAN = G.manifest()


def cli(*args):
    return subprocess.run([str(_capi.CLI_PATH), *map(str, args)], capture_output=True, text=True)


def ov_flags(case):
    return [str(x) for x in MAN["cases"][case].get("overrides", [])]


@pytest.mark.parametrize("case", ["fixture2d_ra", "ref_vehicle3_desk", "ref_bmw7_desk", "room5_uni"])
@pytest.mark.parametrize("mode", ["matrix", "ofa"])
def test_cli_synthesize_container(case, mode, tmp_path):
    out = tmp_path / "r.bin"
    r = cli("synthesize", "-c", G.case_cfg(case), "--mode", mode, "-o", out, *ov_flags(case))
    assert r.returncode == 0, r.stderr
    assert "time_synthesize_s:" in r.stdout and f"mode: {mode}" in r.stdout
    got = G.read_results(out.read_bytes())
    ref = G.golden_results(case)
    want_manifest = dict(ref["manifest"], mode=mode)
    assert got["manifest"] == want_manifest
    assert G.tol_ok(got["values"], ref["values"]).all()
    assert np.array_equal(got["absorbing"], ref["absorbing"])


@pytest.mark.parametrize("case", sorted(c for c, e in MAN["cases"].items() if "matrix" in e.get("files", {})))
def test_cli_dump_matrix(case, tmp_path):
    out = tmp_path / "k.bin"
    r = cli("abstract", "-c", G.case_cfg(case), "--dump-matrix", out, *ov_flags(case))
    assert r.returncode == 0, r.stderr
    got = G.read_matrix(out.read_bytes())
    want = G.read_matrix(G.load(MAN["cases"][case]["files"]["matrix"]))
    assert got["manifest"] == want["manifest"]
    assert np.array_equal(got["origins"], want["origins"])
    assert G.tol_ok(got["probs"], want["probs"]).all()


def _prism(text):
    lines = text.splitlines()
    head = tuple(int(x) for x in lines[0].split())
    body = {}
    for ln in lines[1:]:
        s, c, d, p = ln.split()
        body[(int(s), int(c), int(d))] = float(p)
    return head, body


@pytest.mark.parametrize("case", sorted(c for c, e in MAN["cases"].items() if "prism" in e.get("files", {})))
def test_cli_export_prism(case, tmp_path):
    out = tmp_path / "k.tra"
    r = cli("export-prism", "-c", G.case_cfg(case), "-o", out, *ov_flags(case))
    assert r.returncode == 0, r.stderr
    (gn, gr, gt), got = _prism(out.read_text())
    (wn, wr, wt), want = _prism(G.load(MAN["cases"][case]["files"]["prism"]).decode())
    assert (gn, gr) == (wn, wr) and gt == len(got) and wt == len(want)
    for k in set(got) | set(want):  # transitions present on one side only must be ~0
        a, b = got.get(k, 0.0), want.get(k, 0.0)
        assert abs(a - b) <= 1e-9 * abs(b) + 1e-15, (k, a, b)


def test_cli_domain_error_exit_code(tmp_path):
    e = MAN["cases"]["domain"]["domain_error"]
    r = cli("abstract", "-c", G.case_cfg("domain"))
    assert r.returncode == e["rc"] == 4
    assert r.stderr.strip() == e["stderr"]
