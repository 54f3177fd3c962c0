"""Multi-GPU synthesis on one GPU (the only device this environment has):

* gm_synthesize_multi (C++, one process, one host thread + stream per device) with
  the device list repeated over the peer and store transports — 2, 3 and 5 shards,
  halo and all-gather exchanges, matrix and OFA — must be bit-identical to
  gm_synthesize;
  NCCL runs for real as a one-rank communicator (ncclCommInitAll + in-place
  ncclAllGather every step);
* the `gridmdp synthesize --gpus / --devices` CLI writes the same container;
* sharded.synthesize_sharded with two processes over gloo driving the real
  kernels (DeviceBackend, V staged through host tensors) reproduces the
  single-process result in both exchange modes.
Reference substrate replaced: parallel_for over row ranges (parallel.hpp:23-51);
the reference's own invariant is bit-identical results for any thread count
(test_abstraction.cpp:232-250, test_synthesis.cpp:180-212)."""
import os
import socket
import subprocess

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import golden_io as G
from paper_2005_06191_b200 import _capi
from paper_2005_06191_b200 import gridmdp as g

pytestmark = pytest.mark.gpu
MAN = G.manifest()


def _model(case, **kw):
    return g.load_config(str(G.case_cfg(case)), **G.case_overrides(MAN["cases"][case]), **kw)


def _same(a, b):
    assert np.array_equal(a.values.view(np.uint64), b.values.view(np.uint64))
    assert np.array_equal(a.policy, b.policy)
    assert np.array_equal(a.worst_dist, b.worst_dist)
    assert np.array_equal(a.absorbing, b.absorbing)


CASES = ["fixture2d_ra", "ref_vehicle3_desk", "ref_bmw7_desk", "room5_uni", "ref_traffic3_desk", "chain09"]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("mode", ["matrix", "ofa"])
@pytest.mark.parametrize("exchange", ["halo", "allgather"])
@pytest.mark.parametrize("transport", ["peer", "store"])
def test_multi_bit_identical(case, mode, exchange, transport):
    """peer: copies of the exchanged ranges after each step; store: no copy, the
    pass-2 epilogue (k_maxmin / k_step_warp) writes each value into the value tables
    of the shards that read it."""
    m = _model(case)
    opts = g.SynthesisOptions(mode=mode)
    ref = g.synthesize(m, m.spec, opts)
    for n in (2, 3, 5):
        got, st = g.synthesize_multi(m, [0] * n, m.spec, opts, exchange=exchange, transport=transport)
        _same(got, ref)
        assert st["n_devices"] == n and st["exchange_used"] == exchange
        assert G.tol_ok(got.values, G.golden_results(case)["values"]).all()


def test_multi_auto_picks_halo_for_narrow_reach():
    """vehicle3 at eta/2: slabs reach a few planes of the grid, so the halos move far
    fewer states than the all-gather and `auto` chooses them."""
    text = (G.LARGE / "C2a.cfg").read_text()
    m = g.parse_config(text, "C2a", time_steps=4)
    ref = g.synthesize(m)
    got, st = g.synthesize_multi(m, [0, 0, 0, 0], transport="peer")
    _same(got, ref)
    assert st["exchange_used"] == "halo" and st["halo_states"] < st["allgather_states"] / 2


@pytest.mark.parametrize("mode", ["matrix", "ofa"])
def test_multi_nccl_one_rank(mode):
    """NCCL executes: a one-device communicator, one in-place ncclAllGather per step."""
    m = _model("fixture2d_ra")
    opts = g.SynthesisOptions(mode=mode)
    got, st = g.synthesize_multi(m, [0], m.spec, opts, transport="nccl")
    _same(got, g.synthesize(m, m.spec, opts))
    assert st["exchange_used"] == "allgather" and st["sweep_ms"] > 0


def test_multi_nccl_rejects_repeated_devices():
    m = _model("fixture2d_ra")
    with pytest.raises(_capi.ConfigError, match="distinct devices"):
        g.synthesize_multi(m, [0, 0], transport="nccl")


def test_multi_errors_surface():
    """A device domain error in one shard is reported with the reference's text by
    the multi-device driver too (abstraction.cpp:93-101)."""
    e = MAN["cases"]["domain"]
    m = _model("domain")
    with pytest.raises(_capi.DomainError) as ei:
        g.synthesize_multi(m, [0, 0], transport="peer")
    assert str(ei.value) in e["domain_error"]["stderr"]


def test_multi_c5_north_star():
    """The north star's 7-d BMW OFA synthesis split over 4 shards equals the one-device run."""
    if "C5" not in G.large_manifest():
        pytest.skip("C5 golden missing")
    m = g.load_config(str(G.large_cfg("C5")))
    ref = g.synthesize(m)
    for transport in ("peer", "store"):
        got, st = g.synthesize_multi(m, [0, 0, 0, 0], transport=transport)
        _same(got, ref)
        assert G.tol_ok(got.values, G.large_results("C5")["values"]).all()


def cli(*args):
    return subprocess.run([str(_capi.CLI_PATH), *map(str, args)], capture_output=True, text=True)


@pytest.mark.parametrize("flags", [["--gpus", "1"], ["--devices", "0,0", "--transport", "peer"],
                                   ["--devices", "0,0,0", "--transport", "peer", "--exchange", "allgather"],
                                   ["--devices", "0,0,0", "--transport", "store"]])
def test_cli_multi_gpu_container(flags, tmp_path):
    case = "ref_vehicle3_desk"
    a, b = tmp_path / "a.bin", tmp_path / "b.bin"
    r1 = cli("synthesize", "-c", G.case_cfg(case), "--mode", "matrix", "-o", a)
    r2 = cli("synthesize", "-c", G.case_cfg(case), "--mode", "matrix", "-o", b, *flags)
    assert r1.returncode == 0 and r2.returncode == 0, r2.stderr
    assert a.read_bytes() == b.read_bytes()
    for key in ("gpus:", "time_build_s:", "time_sweep_s:", "roofline_frac:", "sweep_terms_per_s:"):
        assert key in r1.stdout and key in r2.stdout
    n = len(flags[1].split(",")) if flags[0] == "--devices" else int(flags[1])
    assert f"gpus: {n}\n" in r2.stdout


# ------------------------------------------------ two processes, gloo, real kernels


class HostStagedDevice:
    """DeviceBackend with host-side tensors (gloo exchanges CPU tensors): V_{k+1} goes
    to the device, the shard's outputs come back."""

    def __init__(self, model):
        from paper_2005_06191_b200 import sharded as S

        self.dev = torch.device("cuda", 0)
        self.be = S.DeviceBackend(model, torch.cuda.Stream(self.dev), keep_matrix=False)

    def build(self, x0, x1):
        return self.be.build(x0, x1)

    def free(self, tm):
        self.be.free(tm)

    def reach(self, x0, x1):
        return self.be.reach(x0, x1)

    def step(self, tm, x0, x1, v_next, v_out, pol, wst):
        n = x1 - x0
        with torch.cuda.stream(self.be.stream):
            vn = v_next.to(self.dev, non_blocking=False)
            vo = torch.zeros(max(n, 1), dtype=torch.float64, device=self.dev)
            po = torch.zeros(max(n, 1), dtype=torch.int32, device=self.dev)
            wo = torch.zeros(max(n, 1), dtype=torch.int32, device=self.dev)
            self.be.step(tm, x0, x1, vn, vo, po, wo)
            self.be.stream.synchronize()
        v_out[:n] = vo[:n].cpu()
        pol[:n] = po[:n].cpu()
        wst[:n] = wo[:n].cpu()

    def check(self):
        self.be.check()


def _worker(rank, world, port, case, matrix, exchange, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2005_06191_b200 import sharded as S

    m = _model(case)
    be = HostStagedDevice(m)
    vals, pol, wst = S.synthesize_sharded(be, m.n_states, m.spec.horizon, m.spec.is_reach(), matrix,
                                          torch.device("cpu"), exchange=exchange)
    hp = S.exchange_plan(be, S.ShardPlan(m.n_states, world, rank), None, exchange)
    if rank == 0:
        q.put((vals.numpy().copy(), pol.numpy().copy(), wst.numpy().copy(), hp is not None))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case", ["ref_vehicle3_desk", "fixture2d_ra"])
@pytest.mark.parametrize("matrix", [False, True])
@pytest.mark.parametrize("exchange", ["halo", "allgather"])
def test_two_process_gloo_device_backend(case, matrix, exchange):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, matrix, exchange, q)) for r in range(2)]
    for p in procs:
        p.start()
    vals, pol, wst, used_halo = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert used_halo == (exchange == "halo")
    m = _model(case)
    ref = g.synthesize(m, m.spec, g.SynthesisOptions(mode="matrix" if matrix else "ofa"))
    assert np.array_equal(vals.T.view(np.uint64), ref.values.view(np.uint64))
    assert np.array_equal(pol.T.astype(np.uint32), ref.policy)
    assert np.array_equal(wst.T.astype(np.uint32), ref.worst_dist)
