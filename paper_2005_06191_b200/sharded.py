"""Multi-GPU synthesis: one process per GPU, state space sharded into
contiguous flat-index ranges; stage (i) needs no communication.

Rows of a state are reduced only within that state (synthesis.cpp:112-142), so
each rank owns the rows of its states and writes V_k for them; the next step
needs V_{k+1} wherever its slabs reach. That reach is fixed (slab origins do not
depend on the step), so it is computed once per shard (`gm_shard_reach`, the
cutoff-bounded halo): when the halos are much smaller than the grid each step
exchanges only them (NCCL point-to-point, `batch_isend_irecv`) and the value
table is all-gathered once after the sweep; otherwise (wide cutoffs, e.g. BMW
slabs spanning four full axes) V is all-gathered after every step. Per-row
arithmetic does not depend on the sharding or the exchange, so results are
bit-identical for any number of ranks.

The per-shard compute is a backend object with `build(x0, x1)` and
`step(tm, x0, x1, v_next, v_out, pol, wst)`; the product backend is
`DeviceBackend` (C ABI kernels). Tests substitute a CPU backend to exercise the
orchestration with the gloo process group.
"""
from __future__ import annotations

import contextlib
import ctypes as C
from dataclasses import dataclass
from typing import Optional

import torch
import torch.distributed as dist

from . import _capi
from ._capi import call, lib


@dataclass
class ShardPlan:
    """Equal contiguous state ranges (last one shorter), padded to `per` so the
    all-gather has equal chunks and writes V contiguously."""

    n_x: int
    world: int
    rank: int

    @property
    def per(self) -> int:
        return -(-self.n_x // self.world)

    @property
    def x0(self) -> int:
        return min(self.n_x, self.rank * self.per)

    @property
    def x1(self) -> int:
        return min(self.n_x, self.x0 + self.per)

    def bounds(self, r: int) -> tuple[int, int]:
        a = min(self.n_x, r * self.per)
        return a, min(self.n_x, a + self.per)


class DeviceBackend:
    """Kernels of libgridmdp_b200.so on the caller's CUDA stream."""

    def __init__(self, model, stream: Optional[torch.cuda.Stream] = None, keep_matrix: bool = True):
        self.model = model
        self.stream = stream or torch.cuda.current_stream()
        self.keep = keep_matrix
        self._tm = C.c_void_p()
        call("gm_model_set_stream", model.handle, C.c_void_p(self.stream.cuda_stream), 0)

    def build(self, x0: int, x1: int):
        """Stage (i) for the shard; with keep_matrix the device buffers are reused
        across calls (rebuilt in place)."""
        h = self._tm if self.keep else C.c_void_p()
        call("gm_build_shard", self.model.handle, C.c_int64(x0), C.c_int64(x1), C.byref(h))
        if self.keep:
            self._tm = h
        return h

    def free(self, tm) -> None:
        if tm and not self.keep:
            lib.gm_matrix_free(tm)

    def release(self) -> None:
        if self._tm and lib is not None:
            lib.gm_matrix_free(self._tm)
            self._tm = C.c_void_p()

    def __del__(self):
        self.release()

    def step(self, tm, x0, x1, v_next: torch.Tensor, v_out: torch.Tensor, pol: torch.Tensor,
             wst: torch.Tensor) -> None:
        call("gm_step_device", self.model.handle, tm, C.c_int64(x0), C.c_int64(x1),
             C.c_void_p(v_next.data_ptr()), C.c_void_p(v_out.data_ptr()), C.c_void_p(pol.data_ptr()),
             C.c_void_p(wst.data_ptr()), C.c_void_p(self.stream.cuda_stream))

    def check(self) -> None:
        call("gm_check_device_errors", self.model.handle)

    def begin_sweep(self) -> None:
        """A new sweep: the OFA row prologue results of the previous one are dropped
        (gm_step_device caches them across the steps of one sweep)."""
        call("gm_model_release_ofa_cache", self.model.handle)

    def reach(self, x0: int, x1: int) -> tuple[int, int]:
        """Flat interval of V_{k+1} read by the step of states [x0, x1) (gm_shard_reach)."""
        lo, hi = C.c_int64(), C.c_int64()
        call("gm_shard_reach", self.model.handle, C.c_int64(x0), C.c_int64(x1), C.byref(lo), C.byref(hi))
        return lo.value, hi.value


@dataclass
class HaloPlan:
    """Point-to-point V exchange of one rank: `sends` / `recvs` are (peer, a, b)
    flat-state ranges; `halo` False means the all-gather is used instead."""

    halo: bool
    sends: list
    recvs: list
    halo_states: int
    allgather_states: int


def halo_plan(plan: ShardPlan, reach: list, threshold: float = 0.5) -> HaloPlan:
    """Exchange plan from every rank's reach interval (`reach[r] = (lo, hi)`): rank j
    sends rank r the part of its own states inside r's interval. The halo exchange
    is used when it moves at most `threshold` of the all-gather's states."""
    world, rank = plan.world, plan.rank
    pieces = {}
    for r in range(world):
        lo, hi = reach[r]
        for j in range(world):
            if j == r:
                continue
            a, b = plan.bounds(j)
            a, b = max(a, lo), min(b, hi)
            if a < b:
                pieces[(j, r)] = (a, b)
    halo_states = sum(b - a for a, b in pieces.values())
    ag_states = sum(plan.n_x - (plan.bounds(r)[1] - plan.bounds(r)[0]) for r in range(world))
    sends = [(r, a, b) for (j, r), (a, b) in sorted(pieces.items()) if j == rank]
    recvs = [(j, a, b) for (j, r), (a, b) in sorted(pieces.items()) if r == rank]
    return HaloPlan(halo_states <= threshold * ag_states, sends, recvs, halo_states, ag_states)


def exchange_plan(backend, plan: ShardPlan, group=None, exchange: str = "auto") -> Optional[HaloPlan]:
    """The V exchange of a sharded sweep: None = all-gather after every step
    (`exchange="allgather"`, one rank, or halos too wide under "auto"), else the
    halo plan (`"halo"` forces it)."""
    if exchange == "allgather" or not dist.is_initialized() or plan.world == 1 or not hasattr(backend, "reach"):
        return None
    lo, hi = backend.reach(plan.x0, plan.x1)
    t = torch.tensor([lo, hi], dtype=torch.int64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    allr = [torch.empty_like(t) for _ in range(plan.world)]
    dist.all_gather(allr, t, group=group)
    hp = halo_plan(plan, [tuple(int(v) for v in x.tolist()) for x in allr])
    return hp if (hp.halo or exchange == "halo") else None


def _exchange_halo(hp: HaloPlan, v: torch.Tensor, group=None) -> None:
    ops = [dist.P2POp(dist.isend, v[a:b], peer, group) for peer, a, b in hp.sends]
    ops += [dist.P2POp(dist.irecv, v[a:b], peer, group) for peer, a, b in hp.recvs]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def synthesize_sharded(backend, n_x: int, horizon: int, reach: bool, matrix: bool, device,
                       group=None, timer=None, exchange: str = "auto"):
    """run_backward (synthesis.cpp:165-195) over a sharded state space (see
    `_synthesize_sharded`). Every torch op, collectives included, is issued on the
    backend's stream, so the V exchange and the error check are ordered after the
    backend's kernels whatever the caller's current stream is."""
    bstream = getattr(backend, "stream", None) if torch.device(device).type == "cuda" else None
    with torch.cuda.stream(bstream) if bstream is not None else contextlib.nullcontext():
        return _synthesize_sharded(backend, n_x, horizon, reach, matrix, device, group, timer, exchange)


def _synthesize_sharded(backend, n_x: int, horizon: int, reach: bool, matrix: bool, device,
                        group=None, timer=None, exchange: str = "auto"):
    """run_backward (synthesis.cpp:165-195) over a sharded state space.

    Returns (values (T+1, n_x) on every rank, policy (T, n_x) and worst (T, n_x)
    gathered on every rank). `timer(name)` is called at phase boundaries.
    `exchange`: "auto" (halo when it is at most half the all-gather), "halo",
    "allgather", or a plan from `exchange_plan` (computed once per model: it
    costs one row-prologue pass)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    plan = ShardPlan(n_x, world, rank)
    per, x0, x1 = plan.per, plan.x0, plan.x1
    hp = exchange if isinstance(exchange, HaloPlan) else exchange_plan(backend, plan, group, exchange)
    T = horizon
    vals = torch.zeros((T + 1, per * world), dtype=torch.float64, device=device)
    pol = torch.zeros((T, per * world), dtype=torch.int32, device=device)
    wst = torch.zeros((T, per * world), dtype=torch.int32, device=device)
    vals[T, :n_x] = 0.0 if reach else 1.0
    tm = None
    if hasattr(backend, "begin_sweep"):
        backend.begin_sweep()
    if timer:
        timer("build_start")
    if matrix:
        tm = backend.build(x0, x1)
    if timer:
        timer("build_end")
    lo = rank * per
    try:
        for k in range(T - 1, -1, -1):
            backend.step(tm, x0, x1, vals[k + 1], vals[k, lo:lo + per], pol[k, lo:lo + per],
                         wst[k, lo:lo + per])
            if hp is not None:  # V exchange: only the ranges the peers' slabs read (NCCL P2P)
                _exchange_halo(hp, vals[k], group)
            elif dist.is_initialized():  # V exchange: in-place all-gather of the shards (NCCL)
                dist.all_gather_into_tensor(vals[k], vals[k, lo:lo + per].clone() if vals.device.type == "cpu"
                                            else vals[k, lo:lo + per], group=group)
            if k == T - 1 and hasattr(backend, "check"):
                if vals.is_cuda:
                    torch.cuda.current_stream().synchronize()
                backend.check()
    finally:
        if matrix and hasattr(backend, "free"):
            backend.free(tm)
    if hp is not None:  # complete the value table: one all-gather of the shards' columns
        mine = vals[:T, lo:lo + per].contiguous()
        full = torch.empty((world * T, per), dtype=mine.dtype, device=mine.device)
        dist.all_gather_into_tensor(full, mine, group=group)
        vals[:T] = full.view(world, T, per).permute(1, 0, 2).reshape(T, world * per)
    if timer:
        timer("sweep_end")
    if dist.is_initialized() and world > 1:
        # policies and worst disturbances of every step in one collective: each rank's
        # (2T, per) columns, gathered rank-major, then reordered to (T, world * per)
        mine = torch.cat([pol[:, lo:lo + per], wst[:, lo:lo + per]], 0).contiguous()
        full = torch.empty((world * 2 * T, per), dtype=mine.dtype, device=mine.device)
        dist.all_gather_into_tensor(full, mine, group=group)
        full = full.view(world, 2 * T, per).permute(1, 0, 2).reshape(2 * T, world * per)
        pol, wst = full[:T], full[T:]
    return vals[:, :n_x], pol[:, :n_x], wst[:, :n_x]


def result_from_tables(model, vals: torch.Tensor, pol: torch.Tensor, wst: torch.Tensor):
    """Wraps gathered tables as a SynthesisResult that writes the reference container."""
    import numpy as np

    from . import gridmdp as g

    v = np.asfortranarray(vals.cpu().numpy().T)
    p = np.asfortranarray(pol.cpu().numpy().astype(np.uint32).T)
    w = np.asfortranarray(wst.cpu().numpy().astype(np.uint32).T)
    absorbing = np.zeros(0, dtype=np.uint8)
    if model.spec.is_reach():
        absorbing = g.absorbing_states(model, model.spec)
    return g.SynthesisResult(v, p, w, absorbing, model.options.mode, model.spec, model)


_ = _capi  # keep the binding imported (no CPU fallback)
