"""Run-time compiled dynamics (SURVEY.md §8 f row 2; gm_jit.cpp): the rows built
and the synthesis computed with the config's dynamics compiled by NVRTC are
bit-identical to the bytecode-interpreter kernels, the compiled kernels are the
ones that ran (gm_model_jit_status), and device domain errors still reproduce
the reference's error."""
import ctypes as C

import numpy as np
import pytest

import golden_io as G
from paper_2005_06191_b200 import _capi
from paper_2005_06191_b200 import gridmdp as g

pytestmark = pytest.mark.gpu
MAN = G.manifest()
# ite + uniform (chain09), 7-D BMW expressions, sin/cos (vehicle), multiplicative noise,
# degenerate cut, 2-D reach-avoid, beta noise
CASES = ["chain09", "ref_bmw7_desk", "ref_vehicle3_desk", "mult1d", "degenerate", "fixture2d_ra", "room5_beta"]


def model(case):
    return g.load_config(str(G.case_cfg(case)), **G.case_overrides(MAN["cases"][case]))


def jit_status(m):
    s = C.c_double()
    why = C.create_string_buffer(512)
    used = _capi.lib.gm_model_jit_status(m.handle, C.byref(s), why, 512)
    return used, s.value, why.value.decode()


def build(case, jit, monkeypatch):
    monkeypatch.setenv("GM_JIT", "1" if jit else "0")
    m = model(case)
    tm = g.build_matrix(m)
    used, secs, why = jit_status(m)
    assert used == (1 if jit else 0), why
    return tm.origins().copy(), tm.payload().copy()


@pytest.mark.parametrize("case", CASES)
def test_jit_build_bit_identical(case, monkeypatch):
    o1, p1 = build(case, True, monkeypatch)
    o0, p0 = build(case, False, monkeypatch)
    assert np.array_equal(o1, o0)
    assert np.array_equal(p1.view(np.uint64), p0.view(np.uint64))


@pytest.mark.parametrize("case", ["ref_bmw7_desk", "fixture2d_ra", "chain09"])
def test_jit_ofa_synthesis_bit_identical(case, monkeypatch):
    res = {}
    for jit in (True, False):
        monkeypatch.setenv("GM_JIT", "1" if jit else "0")
        m = model(case)
        r = g.synthesize(m, m.spec, g.SynthesisOptions(mode="ofa"))
        assert jit_status(m)[0] == (1 if jit else 0)
        res[jit] = r
    assert np.array_equal(res[True].values.view(np.uint64), res[False].values.view(np.uint64))
    assert np.array_equal(res[True].policy, res[False].policy)
    assert np.array_equal(res[True].worst_dist, res[False].worst_dist)


def test_jit_domain_error_matches_reference(monkeypatch):
    monkeypatch.setenv("GM_JIT", "1")
    want = MAN["cases"]["domain"]["domain_error"]["stderr"].removeprefix("error: ")
    m = model("domain")
    with pytest.raises(g.DomainError) as ex:
        g.build_matrix(m)
    assert str(ex.value) == want
    assert jit_status(m)[0] == 1
    with pytest.raises(g.DomainError) as ex:
        g.synthesize(m, m.spec, g.SynthesisOptions(mode="ofa"))
    assert str(ex.value) == want


def test_jit_auto_policy_small_launch_uses_interpreter(monkeypatch):
    monkeypatch.delenv("GM_JIT", raising=False)
    m = model("tiny")
    g.build_matrix(m)
    used, _, why = jit_status(m)
    assert used == 0 and "2^21 rows and 2^32 row entries" in why


_PROBE = r"""
import ctypes as C, hashlib, sys
sys.path.insert(0, {repo!r}); sys.path.insert(0, {tests!r})
import golden_io as G
from paper_2005_06191_b200 import _capi, gridmdp as g
e = G.manifest()["cases"]["chain09"]
m = g.load_config(str(G.case_cfg("chain09")), **G.case_overrides(e))
tm = g.build_matrix(m)
s = C.c_double(); why = C.create_string_buffer(512)
used = _capi.lib.gm_model_jit_status(m.handle, C.byref(s), why, 512)
print(used, s.value, hashlib.sha256(tm.payload().tobytes()).hexdigest())
"""


def test_jit_disk_cache_reuses_compiled_kernels(tmp_path):
    """Compiled dynamics are cached on disk (GM_JIT_CACHE): a second process loads the
    cubin instead of recompiling and builds the same rows."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    tests = Path(__file__).resolve().parent
    code = _PROBE.format(repo=str(tests.parent), tests=str(tests))
    env = dict(os.environ, GM_JIT="1", GM_JIT_CACHE=str(tmp_path / "jit"))
    runs = []
    for _ in range(2):
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True)
        used, secs, digest = out.stdout.split()
        runs.append((int(used), float(secs), digest))
    assert runs[0][0] == 1 and runs[1][0] == 1
    assert list((tmp_path / "jit").glob("*.jit"))
    assert runs[1][1] < 0.5 * runs[0][1], runs  # loaded, not recompiled
    assert runs[0][2] == runs[1][2]
