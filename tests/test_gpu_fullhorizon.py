"""GPU parity at the BASELINE.json configurations and their full horizons, against
the REFERENCE's own outputs (tests/golden/large/, made by
tests/golden/make_golden_large.py from oracle/_ref = the unmodified reference):

  C5        bmw7.cfg, reach-avoid, T = 32, OFA   (the north star, configs/bmw7.cfg:44-52,
            through synthesize, src/synthesis.cpp:214-228)
  C1        robot_reachavoid.cfg --time-steps 8  (tools/gridmdp_main.cpp:38 override)
  C2a       vehicle3.cfg at its own T = 32        (configs/vehicle3.cfg:25)
  bmw7_mid  bmw7 dynamics on a 4 x 4 position grid, T = 8 (absorbing target, nonzero values)
  C2b       one stored-matrix bellman_step of the bench workload (108 GB matrix) with a
            hashed v_next, every 16th state

Bar (SURVEY.md §8 d): every value |gpu - ref| <= 1e-9 |ref| + 1e-15; absorbing flags
bit-exact; policies equal except on ties within that tolerance (re-checked from the
reference's own V_{k+1}); GPU matrix == GPU OFA bit for bit where both run."""
import numpy as np
import pytest

import golden_io as G
from paper_2005_06191_b200 import gridmdp as g

pytestmark = pytest.mark.gpu

LM = G.large_manifest()
SYNTH = [n for n in ("bmw7_mid", "C2a", "C1", "C5") if n in LM]


def _model(name):
    e = LM[name]
    ov = G.case_overrides({"overrides": e.get("overrides", [])})
    return g.load_config(str(G.large_cfg(name)), **ov)


def _policy_ties(m, ref, pol, worst):
    """Policy / worst-disturbance mismatches must be ties: re-run step k from the
    reference's V_{k+1} and compare the two choices under the GPU's own values."""
    T = ref["values"].shape[1] - 1
    n_diff = 0
    for k in range(T):
        d = np.nonzero(pol[:, k] != ref["policy"][:, k])[0]
        if d.size == 0:
            continue
        g.bellman_step(m, m.spec, None, None, np.ascontiguousarray(ref["values"][:, k + 1]))
        ok, n = G.policy_ok(g.q_values(m), pol[:, k], ref["policy"][:, k])
        assert ok, f"step {k}: {n} policy mismatches that are not ties"
        n_diff += n
    return n_diff


@pytest.mark.parametrize("name", SYNTH)
def test_full_horizon_synthesis_matches_reference(name):
    ref = G.large_results(name)
    m = _model(name)
    assert int(m.sizes().rows) == LM[name]["sizes"]["rows"]
    r = g.synthesize(m, m.spec, g.SynthesisOptions(mode="ofa"))
    assert r.values.shape == ref["values"].shape
    nz = int(np.count_nonzero(ref["values"][:, 0]))
    assert nz > 0, "the golden must not be vacuous"
    ok = G.tol_ok(r.values, ref["values"])
    assert ok.all(), f"{(~ok).sum()} values off, max {np.abs(r.values - ref['values']).max():.3e}"
    if ref["absorbing"].size:
        assert np.array_equal(r.absorbing, ref["absorbing"])
    _policy_ties(m, ref, r.policy, r.worst_dist)


@pytest.mark.parametrize("name", [n for n in ("C2a", "C1") if n in LM])
def test_full_horizon_matrix_equals_ofa(name):
    """Stored-matrix mode reproduces OFA bit for bit at the full horizon (the
    reference's own invariant, test_cli.cpp:104-124)."""
    m = _model(name)
    a = g.synthesize(m, m.spec, g.SynthesisOptions(mode="matrix"))
    b = g.synthesize(m, m.spec, g.SynthesisOptions(mode="ofa"))
    assert np.array_equal(a.values.view(np.uint64), b.values.view(np.uint64))
    assert np.array_equal(a.policy, b.policy) and np.array_equal(a.worst_dist, b.worst_dist)
    assert G.tol_ok(a.values, G.large_results(name)["values"]).all()


@pytest.mark.skipif("C2b_step" not in LM, reason="C2b step golden missing")
def test_c2b_stored_matrix_step_matches_reference():
    """The bench workload (C2b: 18.5 M rows x 729, 108 GB stored on the device): one
    matrix-mode bellman_step from a hashed V_{k+1} against the reference's step."""
    e = LM["C2b_step"]
    m = g.load_config(str(G.LARGE / e["config"]), mode="matrix")
    n_x = int(m.n_states)
    vn = G.hashed_v(n_x)
    tm = g.build_matrix(m)
    g.mask_absorbing(tm, m.spec)
    t0x = g.build_target_hit(m, m.spec)
    v, p, w = g.bellman_step(m, m.spec, tm, t0x, vn)
    del tm
    idx = np.arange(0, n_x, e["stride"])
    want_v = G.large_array("C2b_step.v", "<f8")
    want_p = G.large_array("C2b_step.pol", "<u4")
    ok = G.tol_ok(v[idx], want_v)
    assert ok.all(), f"{(~ok).sum()} values off, max {np.abs(v[idx] - want_v).max():.3e}"
    assert np.count_nonzero(want_v) > 0.5 * idx.size
    pol_ok, n = G.policy_ok(g.q_values(m)[idx], p[idx], want_p)
    assert pol_ok, f"{n} policy mismatches beyond ties"
    g.release_cached_memory()
