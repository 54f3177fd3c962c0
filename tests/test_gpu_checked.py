"""Every kernel family under the bounds-checked build (GM_LIB=checked ->
libgridmdp_b200_checked.so, -DGM_CHECKED): a failed GM_CHECK traps the kernel and
the scenario fails. Stands in for compute-sanitizer memcheck, which the GPU pool
does not allow; shared-memory race freedom is covered by the bit-identity of
every residency / unroll / schedule variant (tests/test_gpu_variants.py)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
REPO = Path(__file__).resolve().parents[1]

SCENARIOS = [
    ("core", {"GM_JIT": "0"}),
    ("jit", {"GM_JIT": "1"}),
    ("et2", {"GM_JIT": "0"}),
    ("et2", {"GM_JIT": "0", "GM_ET_VARIANT": "5"}),
    ("ofa_pk", {"GM_JIT": "0", "GM_OFA_PK": "1"}),
    ("ofa_pk", {"GM_JIT": "0", "GM_OFA_TABLE": "global"}),
    ("ofa_pk", {"GM_JIT": "0", "GM_OFA_TABLE": "prefix", "GM_OFA_PK": "1"}),
    ("custom", {"GM_JIT": "0"}),
    ("sim", {"GM_JIT": "0"}),
    ("multi", {"GM_JIT": "0"}),
    ("build_single", {"GM_JIT": "0", "GM_BUILD_WS": "0", "GM_MATRIX_KERNEL": "walk"}),
]


@pytest.mark.parametrize("scenario,env", SCENARIOS, ids=lambda v: v if isinstance(v, str) else
                         ",".join(f"{k}={x}" for k, x in v.items()))
def test_checked_build(scenario, env):
    lib = REPO / "paper_2005_06191_b200" / "libgridmdp_b200_checked.so"
    assert lib.exists(), "the checked library is built by __graft_entry__.build()"
    e = dict(os.environ, GM_LIB="checked", **env)
    r = subprocess.run([sys.executable, str(REPO / "scripts" / "check_cases.py"), scenario], env=e,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert f"scenario {scenario} ok" in r.stdout
    assert "GM_CHECK failed" not in r.stdout + r.stderr
