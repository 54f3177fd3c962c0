"""Every alternative kernel behind an environment knob keeps the
canonical reduction order and product association, so it must reproduce the
default path bit for bit: the per-term slab-walk matrix kernel (the automatic
fallback for rows too wide for the offset table), the single-role build (the
fallback when the pipelined build's buffers do not fit), the offset-table
residency variants, the OFA in-flight variants, contiguous row schedules, other
build residencies and row pitches, and the compiled dynamics at small sizes.
The knobs are read once per process, so each setting runs in a subprocess."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
TESTS = Path(__file__).resolve().parent
CASES = ["fixture2d_ra", "ref_vehicle3_desk", "exp_dist"]

_PROBE = r"""
import hashlib, sys
sys.path.insert(0, {repo!r}); sys.path.insert(0, {tests!r})
import numpy as np
import golden_io as G
from paper_2005_06191_b200 import gridmdp as g
from paper_2005_06191_b200 import _capi
ofa = lambda: _capi.lib.gm_last_kernel_variant(_capi.KF_EXPECT_OFA).decode()
for case in {cases!r}:
    e = G.manifest()["cases"][case]
    h = hashlib.sha256()
    m = g.load_config(str(G.case_cfg(case)), **G.case_overrides(e))
    tm = g.build_matrix(m)
    h.update(tm.origins().tobytes()); h.update(tm.payload().tobytes())
    for mode in ("matrix", "ofa"):
        r = g.synthesize(m, m.spec, g.SynthesisOptions(mode=mode))
        h.update(np.ascontiguousarray(r.values).tobytes()); h.update(np.ascontiguousarray(r.policy).tobytes())
        h.update(np.ascontiguousarray(r.worst_dist).tobytes())
    print(case, h.hexdigest(), ofa())
# R = 729 rows (a warp per row in the stored-matrix sweep): vehicle3 at eta/4 on a
# 2 x 2 x 3 m corner of its grid
from paper_2005_06191_b200 import workloads as W
text = W.vehicle3(eta=(0.125, 0.125, 0.0625), T=3)
for a, b in (("states.ub = {{10.0, 10.0, 3.5}};", "states.ub = {{2.0, 2.0, 1.5}};"),
             ("target.lb = {{8.0, 0.0, -3.5}};", "target.lb = {{1.5, 0.0, -3.5}};"),
             ("target.ub = {{10.0, 2.0, 3.5}};", "target.ub = {{2.0, 0.5, 1.5}};"),
             ("avoid.lb = {{4.0, 4.0, -3.5}};", "avoid.lb = {{0.75, 0.75, -3.5}};"),
             ("avoid.ub = {{6.0, 6.0, 3.5}};", "avoid.ub = {{1.25, 1.25, 1.5}};")):
    assert a in text
    text = text.replace(a, b)
m = g.parse_config(text, "vehicle_r729")
assert m.sizes().row_width == 729
h = hashlib.sha256()
r = g.synthesize(m)
h.update(np.ascontiguousarray(r.values).tobytes()); h.update(np.ascontiguousarray(r.policy).tobytes())
r = g.synthesize(m, m.spec, g.SynthesisOptions(mode="ofa"))
h.update(np.ascontiguousarray(r.values).tobytes())
print("vehicle_r729", h.hexdigest(), ofa())
# R = 15,750 (tpr 128, the prefix-table OFA kernels): the north-star BMW 320i
# model on a 4 x 4 position grid, two steps
m = g.load_config(str(G.large_cfg("bmw7_mid")), time_steps=2)
r = g.synthesize(m, m.spec, g.SynthesisOptions(mode="ofa"))
h = hashlib.sha256()
h.update(np.ascontiguousarray(r.values).tobytes()); h.update(np.ascontiguousarray(r.policy).tobytes())
h.update(np.ascontiguousarray(r.worst_dist).tobytes())
print("bmw7_mid_T2", h.hexdigest(), ofa())
# R = 7,000 with the line-prefix table (the north-star C5 at full size, one step):
# the per-group / batched NVRTC consumers under GM_JIT=1
m = g.load_config(str(G.large_cfg("C5")), time_steps=1)
r = g.synthesize(m, m.spec, g.SynthesisOptions(mode="ofa"))
h = hashlib.sha256()
h.update(np.ascontiguousarray(r.values).tobytes()); h.update(np.ascontiguousarray(r.policy).tobytes())
h.update(np.ascontiguousarray(r.worst_dist).tobytes())
print("C5_T1", h.hexdigest(), ofa())
"""

SETTINGS = [
    {"GM_MATRIX_KERNEL": "walk"},
    {"GM_BUILD_WS": "0"},
    {"GM_ET_VARIANT": "2", "GM_OFA_U": "4", "GM_CONTIG": "1"},
    {"GM_ET_VARIANT": "5"},  # one row per warp at TPR = 32 (default: two)
    {"GM_BUILD_CTAS": "5", "GM_OFA_U": "8"},
    {"GM_BUILD_CTAS": "2", "GM_JIT": "1"},  # run-time compiled build at the 2-CTA register cap
    {"GM_JIT": "1"},
    {"GM_OFA_TABLE": "prefix"},  # OFA from the leading-prefix table + prefix offset table
    {"GM_OFA_TABLE": "global", "GM_OFA_U": "4"},  # same table, line offsets from global memory
    {"GM_OFA_PK": "1"},  # OFA with the hoisted last-axis cell (row_dot_pk; default only for long rows)
    {"GM_OFA_PK": "1", "GM_OFA_TABLE": "prefix"},
    {"GM_OFA_CACHE": "0"},  # OFA row prologue re-run every step instead of cached across the sweep
    {"GM_STEP_FUSED": "1", "GM_STEP_WARP": "0"},  # small states: both passes in one CTA-wide kernel (k_step_small)
    {"GM_STEP_WARP": "0"},  # small states: expect_matrix + maxmin instead of one warp per state (k_step_warp)
    {"GM_MATRIX_SMALL": "0", "GM_STEP_WARP": "0"},  # one-thread rows through k_expect_matrix_et instead of the warp-staged kernel
    {"GM_MATRIX_SMALL": "1", "GM_STEP_WARP": "0"},  # the warp-staged kernel also for TPR 2 / 4
    {"GM_MATRIX_SMALL": "1", "GM_SMALL_U": "8", "GM_SMALL_SMEM_KB": "28", "GM_STEP_WARP": "0"},  # 8 gathers in flight, half-empty chunks
    {"GM_OFA_PACK": "1", "GM_JIT": "1"},  # OFA consumer with packed (Q, line offset) tables
    {"GM_OFA_GROUP": "0", "GM_JIT": "1"},  # batched shape OFA consumer instead of the per-group one
    {"GM_JIT_SHAPE": "0", "GM_JIT": "1"},  # run-time compiled build without the row-shape specialisation
]


def digests(env_extra):
    code = _PROBE.format(repo=str(TESTS.parent), tests=str(TESTS), cases=CASES)
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return {c: (d, v) for c, d, v in (line.split() for line in out.stdout.strip().splitlines())}


def _digest(rows):
    return {c: d for c, (d, _) in rows.items()}


# the hoisted last-axis cell needs an unroll U in [4, 8] that is a multiple of the
# lane's cell period (launch_ofa): fixture2d_ra and ref_vehicle3_desk have one;
# exp_dist (period 13) and vehicle_r729 (period 9) keep the plain kernel; the wide
# rows (bmw7_mid_T2: the default there, C5_T1) have one too
PK_CASES = {"fixture2d_ra", "ref_vehicle3_desk", "bmw7_mid_T2", "C5_T1"}


@pytest.fixture(scope="module")
def default():
    return digests({"GM_JIT": "0"})


@pytest.mark.parametrize("knob", SETTINGS, ids=lambda d: ",".join(f"{k}={v}" for k, v in d.items()))
def test_variant_bit_identical_to_default(default, knob):
    env = {"GM_JIT": "0", **knob}
    got = digests(env)
    assert _digest(got) == _digest(default)
    if knob.get("GM_OFA_PK") == "1":  # the forced kernel really ran where it applies
        for c, (_, v) in got.items():
            assert v.startswith("k_expect_ofa_pk<") == (c in PK_CASES), (c, v)
    if "GM_OFA_TABLE" in knob:
        assert all(",P," in v or "<P," in v for _, v in got.values()), got
    if knob.get("GM_JIT") == "1" and "GM_OFA_PACK" not in knob:  # the wide-row NVRTC consumer really ran
        want = "k_expect_ofa_shape<NVRTC>" if knob.get("GM_OFA_GROUP") == "0" else "k_expect_ofa_group<NVRTC>"
        assert got["C5_T1"][1] == want, got["C5_T1"]


def test_row_pitch_does_not_change_results(default):
    """Rows padded to another granule (GM_PITCH_GRANULE) change the layout only."""
    got = digests({"GM_JIT": "0", "GM_PITCH_GRANULE": "1"})
    assert _digest(got) == _digest(default)
