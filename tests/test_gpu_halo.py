"""Shard halos for the multi-GPU V exchange (SURVEY.md §8 e; sharded.py):
gm_shard_reach (device prologue + min/max reduction of the slab origins) equals
the interval restated from the engine's own stored origins (parity-tested
against the reference in test_gpu_parity.py), for every shard of 1-4 way
splits, normal / exponential / multiplicative noise, safety and reach specs."""
import numpy as np
import pytest

import golden_io as G
from paper_2005_06191_b200 import gridmdp as g
from paper_2005_06191_b200 import sharded as S

pytestmark = pytest.mark.gpu
MAN = G.manifest()


@pytest.mark.parametrize("case", ["fixture2d_ra", "ref_vehicle3_desk", "exp_dist", "mult1d", "ref_room5"])
def test_shard_reach_matches_stored_origins(case):
    e = MAN["cases"][case]
    m = g.load_config(str(G.case_cfg(case)), **G.case_overrides(e))
    s = m.sizes()
    n_x, rows = int(s.n_states), int(s.rows)
    nuw = rows // n_x
    org = g.build_matrix(m).origins().copy()
    W = g.window_extents(m)
    kv = G.golden_results(case)["manifest"]
    vec = lambda k: [float(v) for v in kv[f"states.{k}"].strip("{}").split(",")]  # noqa: E731
    counts = [int(np.floor((u - l) / h + 1e-9)) + 1 for l, u, h in zip(vec("lb"), vec("ub"), vec("eta"))]
    stride = np.cumprod([1] + counts[::-1])[:-1][::-1]
    span = int(sum((w - 1) * st for w, st in zip(W, stride)))
    absorbed = g.absorbing_states(m, m.spec) if m.spec.is_reach() else np.zeros(n_x, np.uint8)
    be = S.DeviceBackend(m)
    for world in (1, 2, 3, 4):
        for r in range(world):
            p = S.ShardPlan(n_x, world, r)
            got = be.reach(p.x0, p.x1)
            o = org[p.x0 * nuw:p.x1 * nuw][np.repeat(absorbed[p.x0:p.x1] == 0, nuw)]
            want = (p.x0, p.x0) if o.size == 0 else (int(o.min()), min(n_x, int(o.max()) + span + 1))
            assert got == want, (case, world, r)


def test_shard_reach_edge_cases():
    """Custom densities read the whole grid (conservative); a shard whose states are
    all absorbed reads nothing; an empty shard reads nothing."""
    e = MAN["cases"]["custom_tri1d"]
    m = g.load_config(str(G.case_cfg("custom_tri1d")), **G.case_overrides(e))
    n_x = int(m.sizes().n_states)
    assert S.DeviceBackend(m).reach(0, n_x) == (0, n_x)
    e = MAN["cases"]["fixture2d_ra"]
    m = g.load_config(str(G.case_cfg("fixture2d_ra")), **G.case_overrides(e))
    ab = g.absorbing_states(m, m.spec)
    be = S.DeviceBackend(m)
    runs = np.flatnonzero(ab)
    assert runs.size
    x = int(runs[0])
    assert be.reach(x, x + 1) == (x, x)  # one absorbed state: its rows are skipped
    assert be.reach(5, 5) == (5, 5)
