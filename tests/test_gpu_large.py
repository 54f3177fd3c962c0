"""GPU parity at the benchmark sizes against the in-process C
oracle on sampled rows/states, plus size-independent properties:

  * C2b (108 GB stored matrix): sampled rows' origins bit-exact, probabilities
    within 1e-9 rel + 1e-15 abs, row sums <= 1 + 1e-9;
  * C5 (BMW 320i, 7-d, OFA) and the traffic rings C4 / C4' (7-d / 5-d, OFA):
    one Bellman step from a seeded random V on a sampled state range equals the
    oracle's (values within tolerance, policy equal except on ties);
  * sharding invariance: stepping the state space as 1, 2, 3 or 8 shards gives
    bit-identical V, policies and worst disturbances (the property multi-GPU
    runs rely on);
  * matrix == OFA bit for bit on a mid-size configuration.
"""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest
import torch

import golden_io as G
from oracle import oracle_py as O
from paper_2005_06191_b200 import _capi
from paper_2005_06191_b200 import gridmdp as g
from paper_2005_06191_b200 import sharded as S
from paper_2005_06191_b200 import workloads as W

pytestmark = pytest.mark.gpu


def test_c2b_sampled_rows_match_oracle():
    text = W.WORKLOADS["C2b"]()
    m = g.parse_config(text, "C2b")
    om = O.load(text)
    s = m.sizes()
    rows, R = int(s.rows), int(s.row_width)
    tm = g.build_matrix(m)  # the whole 108 GB matrix, device-resident
    rng = np.random.default_rng(7)
    starts = np.unique(rng.integers(0, rows - 64, 40))
    for r0 in starts:
        r1 = int(r0) + 64
        o = np.empty(64, np.int64)
        p = np.empty((64, R))
        _capi.call("gm_matrix_copy_rows", tm.handle, C.c_int64(int(r0)), C.c_int64(r1), _capi.ptr(o), _capi.ptr(p))
        wo, wp = om.build_matrix(int(r0), r1)
        assert np.array_equal(o, wo)
        assert G.tol_ok(p, wp).all(), np.abs(p - wp).max()
        assert (p.sum(axis=1) <= 1 + 1e-9).all()
    del tm


def test_c5_bmw_stored_matrix_shard_matches_oracle():
    """The north-star model's stored MDP is 220.5 GB: one GPU builds the row range of
    the states [0, n_x/2) (110 GB, SURVEY §8 d); sampled rows' origins are bit-exact
    and their probabilities within tolerance of the oracle's."""
    text = W.WORKLOADS["C5"]()
    m = g.parse_config(text, "C5")
    om = O.load(text)
    s = m.sizes()
    R = int(s.row_width)
    half = (m.n_states // 2) * int(s.n_inputs) * int(s.n_disturbances)
    tm = g.build_matrix(m, rows=(0, half))
    rng = np.random.default_rng(11)
    for r0 in np.unique(rng.integers(0, half - 16, 24)):
        r1 = int(r0) + 16
        o = np.empty(16, np.int64)
        p = np.empty((16, R))
        _capi.call("gm_matrix_copy_rows", tm.handle, C.c_int64(int(r0)), C.c_int64(r1), _capi.ptr(o), _capi.ptr(p))
        wo, wp = om.build_matrix(int(r0), r1)
        assert np.array_equal(o, wo)
        assert G.tol_ok(p, wp).all(), np.abs(p - wp).max()
    del tm


def test_c5_bmw_step_matches_oracle_on_sampled_states():
    text = W.WORKLOADS["C5"]()
    m = g.parse_config(text, "C5")
    om = O.load(text)
    n_x = m.n_states
    v = np.random.default_rng(20240).uniform(0, 1, n_x)
    v_out, pol, wst = g.bellman_step(m, m.spec, None, None, v)
    q = g.q_values(m)
    x0, x1 = 60000, 62000
    vo, po, wo, _ = om.bellman_step(v, x0, x1)
    assert G.tol_ok(v_out[x0:x1], vo).all(), np.abs(v_out[x0:x1] - vo).max()
    ok, n = G.policy_ok(q[x0:x1], pol[x0:x1], po)
    assert ok, n


@pytest.mark.parametrize("wl,x0", [("C4", 2391000), ("C4p", 8605000)])
def test_traffic_ofa_step_matches_oracle_on_sampled_states(wl, x0):
    """BASELINE's sharded traffic workloads at full size (C4: 7 cells, R = 78,125;
    C4': traffic5, R = 16,807): one OFA Bellman step from a seeded random V on a
    sampled state range equals the oracle's."""
    text = W.WORKLOADS[wl]()
    m = g.parse_config(text, wl)
    om = O.load(text)
    v = np.random.default_rng(20240).uniform(0, 1, m.n_states)
    v_out, pol, wst = g.bellman_step(m, m.spec, None, None, v)
    q = g.q_values(m)
    x1 = x0 + 96
    vo, po, wo, _ = om.bellman_step(v, x0, x1)
    assert G.tol_ok(v_out[x0:x1], vo).all(), np.abs(v_out[x0:x1] - vo).max()
    ok, n = G.policy_ok(q[x0:x1], pol[x0:x1], po)
    assert ok, n


@pytest.mark.parametrize("wl,x0", [("C4", 1207000), ("C4p", 4303000)])
def test_traffic_ofa_synthesis_chains_steps(wl, x0):
    """The full-size traffic rings through gm_synthesize for two steps (the OFA
    sweep with its row prologue cached across steps): each step's values on a
    sampled state range equal the oracle's Bellman step of the engine's own next-step
    values, and the policies agree except on ties (under the oracle's per-input
    values)."""
    text = W.WORKLOADS[wl]()
    m = g.parse_config(text, wl, time_steps=2)
    om = O.load(text)
    res = g.synthesize(m, m.spec, g.SynthesisOptions(mode="ofa"))
    variant = _capi.lib.gm_last_kernel_variant(_capi.KF_EXPECT_OFA).decode()
    print(wl, variant)
    assert res.values.shape == (m.n_states, 3)
    x1 = x0 + 96
    for k in (1, 0):
        vo, po, _, vin = om.bellman_step(res.values[:, k + 1], x0, x1)
        assert G.tol_ok(res.values[x0:x1, k], vo).all(), (k, np.abs(res.values[x0:x1, k] - vo).max())
        ok, n = G.policy_ok(vin.min(axis=2), res.policy[x0:x1, k], po)
        assert ok, (k, n)
    assert np.isfinite(res.values).all() and (res.values >= 0).all() and (res.values <= 1 + 1e-9).all()


@pytest.mark.parametrize("case", ["ref_vehicle3_desk", "ref_bmw7_desk", "fixture2d_ra"])
@pytest.mark.parametrize("matrix", [False, True])
def test_sharding_is_bit_identical(case, matrix):
    m = g.load_config(str(G.case_cfg(case)), **G.case_overrides(G.manifest()["cases"][case]))
    n_x = m.n_states
    dev = torch.device("cuda", 0)
    v = torch.rand(n_x, dtype=torch.float64, device=dev, generator=torch.Generator(device=dev).manual_seed(3))
    _capi.call("gm_zero_absorbing_device", m.handle, C.c_void_p(v.data_ptr()),
               C.c_void_p(torch.cuda.current_stream().cuda_stream))
    outs = []
    for parts in (1, 2, 3, 8):
        be = S.DeviceBackend(m, torch.cuda.current_stream(), keep_matrix=False)
        vo = torch.zeros(n_x, dtype=torch.float64, device=dev)
        po = torch.zeros(n_x, dtype=torch.int32, device=dev)
        wo = torch.zeros(n_x, dtype=torch.int32, device=dev)
        for r in range(parts):
            x0, x1 = S.ShardPlan(n_x, parts, r).bounds(r)
            tm = be.build(x0, x1) if matrix else None
            be.step(tm, x0, x1, v, vo[x0:], po[x0:], wo[x0:])
            torch.cuda.synchronize()
            be.free(tm)
        outs.append((vo.cpu().numpy(), po.cpu().numpy(), wo.cpu().numpy()))
    for o in outs[1:]:
        assert np.array_equal(o[0].view(np.uint64), outs[0][0].view(np.uint64))
        assert np.array_equal(o[1], outs[0][1]) and np.array_equal(o[2], outs[0][2])


def test_matrix_equals_ofa_bitwise_midsize():
    text = W.vehicle3(eta=(0.25, 0.25, 0.125), T=6, mode="matrix")
    m = g.parse_config(text, "vehicle-mid")
    a = g.synthesize(m, m.spec, g.SynthesisOptions(mode="matrix"))
    b = g.synthesize(m, m.spec, g.SynthesisOptions(mode="ofa"))
    assert np.array_equal(a.values.view(np.uint64), b.values.view(np.uint64))
    assert np.array_equal(a.policy, b.policy) and np.array_equal(a.worst_dist, b.worst_dist)
    want = O.load(text).synthesize()
    assert G.tol_ok(a.values, want["values"]).all()


def test_smoke_entry():
    import __graft_entry__

    __graft_entry__.smoke()


@pytest.mark.parametrize("pinned", [False, True])
def test_build_shard_host_matches_build_and_copy(pinned):
    """gm_build_shard_host gives the same rows and metadata as gm_build_shard followed by
    the copies: with pageable host buffers (sliced build, copies under the next slice)
    and with pinned ones (the build kernel writes origins / T0x to the host itself)."""
    import ctypes as C

    from paper_2005_06191_b200 import _capi
    from paper_2005_06191_b200 import workloads as W
    m = g.parse_config(W.WORKLOADS["C2a"](), "C2a")
    s = m.sizes()
    nx, nuw, R = int(s.n_states), int(s.n_inputs) * int(s.n_disturbances), int(s.row_width)
    x0, x1 = 3, nx - 5
    rows = (x1 - x0) * nuw
    if pinned:
        to, tt = (torch.empty(rows, dtype=dt, pin_memory=True) for dt in (torch.int64, torch.float64))
        org, t0x = to.numpy(), tt.numpy()
    else:
        org = np.empty(rows, np.int64)
        t0x = np.empty(rows, np.float64)
    h = C.c_void_p()
    _capi.call("gm_build_shard_host", m.handle, C.c_int64(x0), C.c_int64(x1), C.byref(h), _capi.ptr(org),
               _capi.ptr(t0x))
    p1 = np.empty(rows * R)
    _capi.call("gm_matrix_copy_rows", h, C.c_int64(x0 * nuw), C.c_int64(x1 * nuw), None, _capi.ptr(p1))
    _capi.lib.gm_matrix_free(h)
    h2 = C.c_void_p()
    _capi.call("gm_build_shard", m.handle, C.c_int64(x0), C.c_int64(x1), C.byref(h2))
    org2, t0x2, p2 = np.empty(rows, np.int64), np.empty(rows), np.empty(rows * R)
    _capi.call("gm_matrix_copy_rows", h2, C.c_int64(x0 * nuw), C.c_int64(x1 * nuw), _capi.ptr(org2), _capi.ptr(p2))
    _capi.call("gm_matrix_copy_t0x", h2, C.c_int64(x0 * nuw), C.c_int64(x1 * nuw), _capi.ptr(t0x2))
    _capi.lib.gm_matrix_free(h2)
    assert np.array_equal(org, org2) and np.array_equal(t0x.view(np.uint64), t0x2.view(np.uint64))
    assert np.array_equal(p1.view(np.uint64), p2.view(np.uint64))


def test_build_shard_host_direct_host_writes():
    """GM_BUILD_HOST_DIRECT=1 (the build kernel writes origins / T0x into pinned host
    memory itself) gives the same metadata as the default sliced copies."""
    import subprocess
    import sys
    code = """
import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)
import test_gpu_large as T
T.test_build_shard_host_matches_build_and_copy(True)
print("direct ok")
""" % (str(Path(__file__).resolve().parents[1]), str(Path(__file__).resolve().parent))
    import os
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, GM_BUILD_HOST_DIRECT="1"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "direct ok" in r.stdout, r.stderr[-2000:]
