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
    assert used == 0 and "2^21" in why
