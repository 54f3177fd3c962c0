"""The C oracle restatement (oracle/gm_oracle.c) against the REFERENCE's own
outputs (golden fixtures from oracle/_ref, the unmodified reference sources).

The oracle follows the reference's operation order and libm, so the bar here
is bit-exact: values, policies, worst disturbances, stored rows, origins,
target-hit vectors and single Bellman steps."""
import numpy as np
import pytest

import golden_io as G
from oracle import oracle_py as O

MAN = G.manifest()
# the C restatement covers the config-reachable families; custom densities (a C++
# callback in the reference) are checked GPU-vs-reference only (tests/test_gpu_parity.py)
_ORACLE = {c: e for c, e in MAN["cases"].items() if not e.get("custom_density")}
CASES = sorted(c for c, e in _ORACLE.items() if "results" in e)


def oracle(case):
    return O.load(str(G.case_cfg(case)), **G.case_overrides(MAN["cases"][case]))


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("case", CASES)
def test_synthesis_bit_exact(case):
    e = MAN["cases"][case]
    ref = G.golden_results(case)
    m = oracle(case)
    modes = [False, True] if e["sizes"]["memory_estimate_bytes"] < 2e9 else [False]
    for matrix in modes:
        r = m.synthesize(matrix=matrix)
        assert np.array_equal(bits(r["values"]), bits(ref["values"])), f"matrix={matrix}"
        assert np.array_equal(r["policy"], ref["policy"])
        assert np.array_equal(r["worst"], ref["worst"])
        assert np.array_equal(r["absorbing"], ref["absorbing"])


@pytest.mark.parametrize("case", sorted(c for c, e in _ORACLE.items() if "matrix" in e.get("files", {})))
def test_matrix_bit_exact(case):
    e = MAN["cases"][case]
    want = G.read_matrix(G.load(e["files"]["matrix"]))
    m = oracle(case)
    assert m.extents == want["window"]
    o, p = m.build_matrix()
    assert np.array_equal(o, want["origins"])
    assert np.array_equal(bits(p), bits(want["probs"]))
    if "masked" in e["files"]:
        masked = G.read_matrix(G.load(e["files"]["masked"]))
        m.mask(o, p)
        assert np.array_equal(bits(p), bits(masked["probs"]))


@pytest.mark.parametrize("case", sorted(c for c, e in _ORACLE.items() if "t0x" in e.get("files", {})))
def test_target_hit_bit_exact(case):
    want = np.frombuffer(G.load(MAN["cases"][case]["files"]["t0x"]), "<f8")
    assert np.array_equal(bits(oracle(case).target_hit()), bits(want))


@pytest.mark.parametrize("case", sorted(c for c, e in _ORACLE.items() if "step_prefix" in e.get("files", {})))
def test_bellman_step_bit_exact(case):
    m = oracle(case)
    for mode in ("ofa", "matrix"):
        try:
            vn, v, p, w = G.golden_step(case, mode)
        except FileNotFoundError:
            continue
        kw = {}
        if mode == "matrix":
            o, pr = m.build_matrix()
            t0 = None
            if m.reach:
                m.mask(o, pr)
                t0 = m.target_hit()
            kw = dict(probs=pr, origins=o, t0x=t0)
        vo, pol, wst, _ = m.bellman_step(vn, **kw)
        assert np.array_equal(bits(vo), bits(v)), mode
        assert np.array_equal(pol, p) and np.array_equal(wst, w), mode


def test_sizes_of_every_bundled_config():
    """estimate-mem sizes (the reference's fast acceptance check) for all 12 configs."""
    for name, e in MAN["estimate"].items():
        m = O.OracleModel(O.parse_config(e["config"]))
        s = e["sizes"]
        assert (m.n_x, m.n_u, m.n_w, m.rows, m.R) == (s["states"], s["inputs"], s["disturbances"], s["rows"],
                                                       s["row_width"]), name
        assert m.extents == s["window"], name
        assert m.memory_estimate == s["memory_estimate_bytes"], name


def test_reference_known_answers():
    """Known answers quoted by the reference's own tests."""
    est = MAN["estimate"]
    # test_abstraction.cpp:337-353 / test_grid.cpp:136-142: robot window 13x13, R=169
    assert est["robot_reachavoid"]["sizes"]["window"] == [13, 13]
    assert est["robot_reachavoid"]["sizes"]["memory_estimate_bytes"] == 1681 * 441 * 11 * 169 * 8 + \
        1681 * 441 * 11 * 8 + 4096
    # test_config_io.cpp:60-80: published pair counts
    assert est["robot_safety"]["sizes"]["state_input_pairs"] == 203401
    assert est["traffic5"]["sizes"]["state_input_pairs"] == 68841472
    assert est["bmw7"]["sizes"]["states"] == 157500
    # test_synthesis.cpp:90-108: chain kernel [[.9,0],[0,.9]] -> V = 1, .9, .81
    r = oracle("chain09").synthesize()
    assert r["values"][0, 2] == 1.0
    assert abs(r["values"][0, 1] - 0.9) <= 1e-14 and abs(r["values"][0, 0] - 0.81) <= 1e-14
    # test_abstraction.cpp:111-122: gamma above the peak -> W=1, origin(r)=r
    m = oracle("degenerate")
    o, p = m.build_matrix()
    assert m.R == 1 and list(o) == [0, 1, 2]
