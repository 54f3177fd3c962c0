"""The C-ABI entries that take the reference's own data, on the GPU:

* gm_matrix_read (read_matrix, io.cpp:258-283): the REFERENCE's matrix dumps
  (tests/golden/out/*.matrix.bin / *.masked.bin, written by oracle/_ref) loaded
  onto the device and fed to gm_synthesize_with_matrix (synthesis.cpp:199-212)
  give the reference's results (tolerance) and the engine's own synthesize (bits);
* gm_matrix_upload: a host TransitionMatrix (abstraction.hpp:22-65) onto the device;
* gm_query_policy (synthesis.cpp:230-239) against the policy table, with the
  reference's out_of_range behaviour."""
import gzip

import numpy as np
import pytest

import golden_io as G
from paper_2005_06191_b200 import gridmdp as g

pytestmark = pytest.mark.gpu
MAN = G.manifest()
MATRIX_CASES = sorted(c for c, e in MAN["cases"].items() if "matrix" in e.get("files", {}) and "results" in e)


def _model(case):
    return g.load_config(str(G.case_cfg(case)), **G.case_overrides(MAN["cases"][case]))


def _dump(case, kind, tmp_path):
    p = tmp_path / f"{case}.{kind}.bin"
    p.write_bytes(G.load(MAN["cases"][case]["files"][kind]))
    return p


@pytest.mark.parametrize("case", MATRIX_CASES)
def test_read_reference_matrix_then_synthesize_with_matrix(case, tmp_path):
    m = _model(case)
    tm = g.read_matrix(str(_dump(case, "matrix", tmp_path)), m)
    want = G.read_matrix(G.load(MAN["cases"][case]["files"]["matrix"]))
    assert np.array_equal(tm.origins(), want["origins"])
    assert np.array_equal(tm.payload().view(np.uint64), want["probs"].view(np.uint64)), "read_matrix is bit-exact"
    res = g.synthesize_with_matrix(m, tm, None, m.spec, g.SynthesisOptions(mode="matrix"))
    ref = G.golden_results(case)
    assert G.tol_ok(res.values, ref["values"]).all()
    if m.spec.is_reach():  # the reference's contract: synthesize_with_matrix masks tm in place
        masked = G.read_matrix(G.load(MAN["cases"][case]["files"]["masked"]))
        assert np.array_equal(tm.payload() == 0.0, masked["probs"] == 0.0)
    own = g.synthesize(m, m.spec, g.SynthesisOptions(mode="matrix"))
    # rows read from the reference's dump differ from the engine's build only in libm
    # ulps, so the values agree within the parity bar, not bit for bit
    assert G.tol_ok(res.values, own.values).all()


@pytest.mark.parametrize("case", ["fixture2d_ra", "ref_vehicle3_desk", "exp_dist"])
def test_synthesize_with_matrix_equals_synthesize(case):
    """gm_synthesize_with_matrix over the engine's own build (+ its target-hit vector
    from the host) reproduces gm_synthesize bit for bit."""
    m = _model(case)
    tm = g.build_matrix(m)
    t0x = g.build_target_hit(m, m.spec) if m.spec.is_reach() else None
    a = g.synthesize_with_matrix(m, tm, t0x, m.spec, g.SynthesisOptions(mode="matrix"))
    b = g.synthesize(m, m.spec, g.SynthesisOptions(mode="matrix"))
    assert np.array_equal(a.values.view(np.uint64), b.values.view(np.uint64))
    assert np.array_equal(a.policy, b.policy) and np.array_equal(a.worst_dist, b.worst_dist)


@pytest.mark.parametrize("case", ["fixture2d_safety", "exp_dist"])
def test_upload_host_matrix_bellman_step(case):
    m = _model(case)
    want = G.read_matrix(G.load(MAN["cases"][case]["files"]["matrix"]))
    tm = g.upload_matrix(m, want["origins"], want["probs"])
    assert np.array_equal(tm.payload().view(np.uint64), want["probs"].view(np.uint64))
    vn = np.random.default_rng(5).uniform(size=m.n_states)
    v1, p1, w1 = g.bellman_step(m, m.spec, tm, None, vn)
    v2, p2, w2 = g.bellman_step(m, m.spec, g.build_matrix(m), None, vn)
    assert G.tol_ok(v1, v2).all()


def test_matrix_of_another_model_is_rejected(tmp_path):
    m = _model("fixture2d_ra")
    tm = g.read_matrix(str(_dump("tiny", "matrix", tmp_path)), m)
    with pytest.raises(g.ConfigError, match="does not match the model"):
        g.synthesize_with_matrix(m, tm, None, m.spec)


@pytest.mark.parametrize("case", ["fixture2d_ra", "ref_vehicle3_desk"])
def test_query_policy(case):
    m = _model(case)
    res = g.synthesize(m)
    text = G.case_cfg(case).read_text()

    def grid(prefix):
        def vec(k):
            line = next(ln for ln in text.splitlines() if ln.strip().startswith(f"{prefix}.{k} "))
            return tuple(float(v) for v in line.split("=", 1)[1].strip(" ;{}").split(","))
        return g.Grid(vec("lb"), vec("ub"), vec("eta"))

    sg, ig = grid("states"), grid("inputs")
    rng = np.random.default_rng(1)
    T = m.spec.horizon
    lb, ub = np.array(sg.lb), np.array(sg.ub)
    for _ in range(200):
        x = rng.uniform(lb, ub)
        k = int(rng.integers(1, T + 1))
        u = g.query_policy(res, ig, sg, x, k)
        want = ig.point(int(res.policy[sg.index(x), k - 1]))
        assert np.array_equal(u, want)
    with pytest.raises(IndexError, match=r"query_policy: step 0 outside \[1, "):
        g.query_policy(res, ig, sg, lb, 0)
    with pytest.raises(IndexError, match="outside the quantized region"):
        g.query_policy(res, ig, sg, ub + 10 * np.array(sg.eta), 1)
