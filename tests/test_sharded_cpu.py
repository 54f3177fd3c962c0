"""Multi-process orchestration of the sharded synthesis (paper_2005_06191_b200/
sharded.py) on CPU with the gloo backend, world_size 2: state shards, one
all-gather of V per backward step, gathered policies. The per-shard compute
is the oracle (a CPU backend injected by the test), so the result must be
bit-identical to the single-process oracle and therefore to the reference."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import golden_io as G
from oracle import oracle_py as O
from paper_2005_06191_b200 import sharded as S


class OracleBackend:
    """Shard compute on the CPU oracle (tests only)."""

    def __init__(self, om: O.OracleModel):
        self.om = om

    def build(self, x0, x1):
        nuw = self.om.n_u * self.om.n_w
        o, p = self.om.build_matrix(x0 * nuw, x1 * nuw)
        t0 = None
        if self.om.reach:
            self.om.mask(o, p)
            t0 = self.om.target_hit(x0 * nuw, x1 * nuw)
        return (o, p, t0)

    def reach(self, x0, x1):
        """gm_shard_reach restated on the oracle: [min origin, max origin + last slab
        offset] over the rows the step reads (absorbed states skipped for reach specs)."""
        st, om = self.om.st, self.om
        nuw = om.n_u * om.n_w
        o, _ = om.build_matrix(x0 * nuw, x1 * nuw)
        if om.reach:
            live = np.repeat(om.absorbing()[x0:x1] == 0, nuw)
            o = o[live]
        if o.size == 0:
            return x0, x0
        vec = lambda k: [float(v) for v in st[f"states.{k}"].strip("{}").split(",")]  # noqa: E731
        counts = [int(np.floor((u - l) / e + 1e-9)) + 1 for l, u, e in zip(vec("lb"), vec("ub"), vec("eta"))]
        stride = np.cumprod([1] + counts[::-1])[:-1][::-1]
        span = int(sum((w - 1) * s for w, s in zip(om.extents, stride)))
        return int(o.min()), min(om.n_x, int(o.max()) + span + 1)

    def step(self, tm, x0, x1, v_next, v_out, pol, wst):
        kw = {}
        if tm is not None:
            kw = dict(origins=tm[0], probs=tm[1], t0x=tm[2])
        vo, p, w, _ = self.om.bellman_step(v_next[: self.om.n_x].numpy(), x0, x1, **kw)
        n = x1 - x0
        v_out[:n] = torch.from_numpy(vo)
        pol[:n] = torch.from_numpy(p.astype(np.int32))
        wst[:n] = torch.from_numpy(w.astype(np.int32))


def _worker(rank, world, port, case, matrix, q, exchange="auto"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    e = G.manifest()["cases"][case]
    om = O.load(str(G.case_cfg(case)), **G.case_overrides(e))
    be = OracleBackend(om)
    hp = S.exchange_plan(be, S.ShardPlan(om.n_x, world, rank), None, exchange)
    vals, pol, wst = S.synthesize_sharded(be, om.n_x, om.horizon, om.reach, matrix, torch.device("cpu"),
                                          exchange=exchange)
    if rank == 0:
        q.put((vals.numpy().copy(), pol.numpy().copy(), wst.numpy().copy(), hp is not None))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case,matrix", [("fixture2d_ra", True), ("fixture2d_ra", False),
                                         ("ref_vehicle3_desk", False), ("exp_dist", True)])
def test_two_rank_sharded_synthesis_is_bit_identical(case, matrix):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, matrix, q)) for r in range(2)]
    for p in procs:
        p.start()
    vals, pol, wst, _ = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = G.golden_results(case)
    assert np.array_equal(vals.T.view(np.uint64), np.ascontiguousarray(ref["values"]).view(np.uint64))
    assert np.array_equal(pol.T.astype(np.uint32), ref["policy"])
    assert np.array_equal(wst.T.astype(np.uint32), ref["worst"])


def test_shard_plan_covers_states_exactly():
    for n_x in (1, 7, 81, 741393):
        for world in (1, 2, 3, 8):
            plans = [S.ShardPlan(n_x, world, r) for r in range(world)]
            covered = sum(p.x1 - p.x0 for p in plans)
            assert covered == n_x
            assert all(p.x0 == min(n_x, r * p.per) for r, p in enumerate(plans))
            assert plans[-1].x1 == n_x or n_x < world


def _run(world, case, matrix, exchange):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, matrix, q, exchange)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=180)
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("case,matrix,world", [("fixture2d_ra", True, 2), ("ref_vehicle3_desk", False, 3),
                                               ("exp_dist", True, 2)])
def test_halo_exchange_is_bit_identical(case, matrix, world):
    """V exchanged only over the shards' cutoff-bounded halos (point-to-point) gives the
    reference's results bit for bit, like the per-step all-gather."""
    vals, pol, wst, used = _run(world, case, matrix, "halo")
    assert used
    ref = G.golden_results(case)
    assert np.array_equal(vals.T.view(np.uint64), np.ascontiguousarray(ref["values"]).view(np.uint64))
    assert np.array_equal(pol.T.astype(np.uint32), ref["policy"])
    assert np.array_equal(wst.T.astype(np.uint32), ref["worst"])


def test_halo_plan_ranges():
    plan = [S.ShardPlan(100, 4, r) for r in range(4)]
    reach = [(0, 30), (20, 55), (45, 80), (70, 100)]  # each shard reads +-5 states around its own
    hps = [S.halo_plan(p, reach) for p in plan]
    assert hps[0].sends == [(1, 20, 25)] and hps[0].recvs == [(1, 25, 30)]
    assert hps[1].sends == [(0, 25, 30), (2, 45, 50)] and hps[1].recvs == [(0, 20, 25), (2, 50, 55)]
    assert hps[3].recvs == [(2, 70, 75)] and hps[3].sends == [(2, 75, 80)]
    assert all(h.halo for h in hps) and hps[0].halo_states == 30 and hps[0].allgather_states == 300
    # every received range is sent by its owner
    sent = {(r, p.rank, a, b) for p, h in zip(plan, hps) for r, a, b in h.sends}
    recv = {(p.rank, j, a, b) for p, h in zip(plan, hps) for j, a, b in h.recvs}
    assert {(d, s_, a, b) for (d, s_, a, b) in sent} == {(r, j, a, b) for (r, j, a, b) in recv}
    wide = [S.halo_plan(p, [(0, 100)] * 4) for p in plan]
    assert not any(h.halo for h in wide)  # the all-gather fallback
    empty = [S.halo_plan(p, [(p2.x0, p2.x0) for p2 in plan]) for p in plan]  # every shard absorbed
    assert all(h.halo and not h.sends and not h.recvs and h.halo_states == 0 for h in empty)
