"""Reference-facing API of the B200 engine.

Mirrors the reference's C++ interface for the hot path (names, argument
meaning and error behaviour) on top of the C ABI in include/gridmdp_b200.h:

  config.hpp:55-70     load_config / parse_config / build_model / build_spec / build_options
  grid.hpp:87-99       make_grid (validated when the model is built)
  noise.hpp:27-36      NoiseSpec.normal / uniform / exponential / beta
  spec.hpp:24-26       make_safety / make_reachability / make_reach_avoid
  abstraction.hpp:70-131  window_extents / memory_estimate / build_matrix /
                          build_target_hit / mask_absorbing / TransitionMatrix
  synthesis.hpp:12-66  SynthesisOptions / synthesize / synthesize_with_matrix /
                          bellman_step / query_policy / SynthesisResult
  io.hpp:13-19         write_results / TransitionMatrix.write (write_matrix)

Every compute call runs the sm_100a kernels of libgridmdp_b200.so; there is
no CPU path (a missing device raises CudaError).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _capi
from ._capi import (ConfigError, CudaError, DomainError, GridmdpError, IoError, MemoryError_,  # noqa: F401
                    ParseError, call, lib, ptr)

MemoryError = MemoryError_  # noqa: A001  reference name (common.hpp:34)

SAFETY, REACHABILITY, REACH_AVOID = "safety", "reachability", "reach-avoid"
_KIND = {SAFETY: _capi.GM_SAFETY, REACHABILITY: _capi.GM_REACH, REACH_AVOID: _capi.GM_REACH_AVOID,
         "reach_avoid": _capi.GM_REACH_AVOID}
_KIND_NAME = {_capi.GM_SAFETY: SAFETY, _capi.GM_REACH: REACHABILITY, _capi.GM_REACH_AVOID: REACH_AVOID}


def _fmt(v: float) -> str:
    r = repr(float(v))
    return r


def _vec(v: Sequence[float]) -> str:
    return "{" + ", ".join(_fmt(x) for x in v) + "}"


# --------------------------------------------------------------------- model parts

@dataclass(frozen=True)
class Grid:
    """Uniform grid description (grid.hpp:16-46); counts/strides come from the engine."""

    lb: tuple
    ub: tuple
    eta: tuple

    @property
    def dim(self) -> int:
        return len(self.lb)

    def counts(self) -> list[int]:
        # grid.cpp:34-35 (same IEEE operations as the engine's host front end)
        return [int(math.floor((u - l) / e + 1e-9)) + 1 for l, u, e in zip(self.lb, self.ub, self.eta)]

    @property
    def size(self) -> int:
        n = 1
        for c in self.counts():
            n *= c
        return n

    def strides(self) -> list[int]:
        c = self.counts()
        s = [1] * len(c)
        for i in range(len(c) - 2, -1, -1):
            s[i] = s[i + 1] * c[i + 1]
        return s

    def point(self, i: int) -> np.ndarray:
        """index_to_point (grid.cpp:55-65)."""
        if i < 0 or i >= self.size:
            raise IndexError(f"index_to_point: flat index {i} out of range")
        p = np.empty(self.dim)
        for d, s in enumerate(self.strides()):
            j, i = divmod(i, s)
            p[d] = self.lb[d] + float(j) * self.eta[d]
        return p

    def index(self, x: Sequence[float]) -> int:
        """point_to_index (grid.cpp:77-96): nearest representative, ties toward +inf."""
        if len(x) != self.dim:
            raise IndexError("point_to_index: point dimension mismatch")
        flat = 0
        counts = self.counts()
        for d, s in enumerate(self.strides()):
            t = (x[d] - self.lb[d]) / self.eta[d]
            if t < -0.5 - 1e-9 or t > float(counts[d] - 1) + 0.5 + 1e-9:
                raise IndexError(f"point_to_index: coordinate {x[d]:g} of axis {d} lies outside the quantized region")
            j = min(max(int(math.floor(t + 0.5)), 0), counts[d] - 1)
            flat += j * s
        return flat


def make_grid(lb: Sequence[float], ub: Sequence[float], eta: Sequence[float]) -> Grid:
    return Grid(tuple(float(v) for v in lb), tuple(float(v) for v in ub), tuple(float(v) for v in eta))


@dataclass(frozen=True)
class NoiseSpec:
    """i.i.d. additive/multiplicative noise (noise.hpp:22-70)."""

    family: str
    p1: tuple
    p2: tuple = ()
    gamma: float = 0.0
    mode: str = "additive"

    @staticmethod
    def normal(sigma, gamma, mode="additive"):
        return NoiseSpec("normal", tuple(map(float, sigma)), (), float(gamma), mode)

    @staticmethod
    def uniform(a, b, gamma, mode="additive"):
        return NoiseSpec("uniform", tuple(map(float, a)), tuple(map(float, b)), float(gamma), mode)

    @staticmethod
    def exponential(rate, gamma, mode="additive"):
        return NoiseSpec("exponential", tuple(map(float, rate)), (), float(gamma), mode)

    @staticmethod
    def beta(alpha, beta_, gamma, mode="additive"):
        return NoiseSpec("beta", tuple(map(float, alpha)), tuple(map(float, beta_)), float(gamma), mode)

    @staticmethod
    def custom(pdf: str, support_lo, support_hi, gamma, mode="additive"):
        """NoiseSpec::custom (noise.hpp:16-19, noise.cpp:75-85) with the joint pdf given as an
        expression over the noise coordinates x0..x{n-1} (the C++ API takes a callback)."""
        return NoiseSpec("custom", tuple(map(float, support_lo)), tuple(map(float, support_hi)), float(gamma), mode,
                         pdf)

    pdf: str = ""

    def config_lines(self) -> list[str]:
        if self.family == "custom":
            return [f"noise.type = custom;", f"noise.mode = {self.mode};",
                    f"noise.cutting_probability = {_fmt(self.gamma)};", f"noise.pdf = {self.pdf};",
                    f"noise.support.lb = {_vec(self.p1)};", f"noise.support.ub = {_vec(self.p2)};"]
        keys = {"normal": ("sigma",), "uniform": ("a", "b"), "exponential": ("rate",), "beta": ("alpha", "beta")}[
            self.family]
        out = [f"noise.type = {self.family};", f"noise.mode = {self.mode};",
               f"noise.cutting_probability = {_fmt(self.gamma)};", f"noise.{keys[0]} = {_vec(self.p1)};"]
        if len(keys) > 1:
            out.append(f"noise.{keys[1]} = {_vec(self.p2)};")
        return out


@dataclass(frozen=True)
class Box:
    lo: tuple
    hi: tuple

    def __init__(self, lo, hi):
        object.__setattr__(self, "lo", tuple(map(float, lo)))
        object.__setattr__(self, "hi", tuple(map(float, hi)))

    @property
    def dim(self) -> int:
        return len(self.lo)

    def contains(self, x) -> bool:
        return len(x) == self.dim and all(a >= l for a, l in zip(x, self.lo)) and all(
            a <= h for a, h in zip(x, self.hi))


@dataclass(frozen=True)
class Spec:
    kind: str = SAFETY
    horizon: int = 1
    target: Optional[Box] = None
    avoid: Optional[Box] = None

    def is_reach(self) -> bool:
        return self.kind != SAFETY


def make_safety(horizon: int) -> Spec:
    return Spec(SAFETY, int(horizon))


def make_reachability(horizon: int, target: Box) -> Spec:
    return Spec(REACHABILITY, int(horizon), target)


def make_reach_avoid(horizon: int, target: Box, avoid: Box) -> Spec:
    return Spec(REACH_AVOID, int(horizon), target, avoid)


@dataclass
class SynthesisOptions:
    mode: str = "matrix"     # matrix | ofa
    threads: int = 0         # host threads (the device path ignores it)
    memory_budget: int = 0   # bytes, 0 = unlimited; binds matrix mode only


# ------------------------------------------------------------------------- model

class SystemModel:
    """A quantized control system (model.hpp:15-35) resident in the engine.

    Also carries the configuration's Spec and SynthesisOptions when loaded from a
    config file (build_spec / build_options)."""

    def __init__(self, handle: C.c_void_p, text: Optional[str] = None):
        self._h = handle
        self.text = text
        self._spec_cache: Optional[Spec] = None
        s = self.sizes()
        self.spec = self._spec_from_sizes(s)
        self.options = SynthesisOptions(mode="ofa" if s.mode == _capi.GM_MODE_OFA else "matrix",
                                        threads=s.threads, memory_budget=int(s.mem_budget))

    def _spec_from_sizes(self, s) -> Spec:
        return Spec(_KIND_NAME[s.spec_kind], int(s.horizon))  # boxes are kept engine-side

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # module globals may already be cleared at interpreter exit
            lib.gm_model_free(h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def sizes(self) -> _capi.Sizes:
        s = _capi.Sizes()
        call("gm_model_sizes", self._h, C.byref(s))
        return s

    @property
    def n_states(self) -> int:
        return int(self.sizes().n_states)

    @property
    def n_inputs(self) -> int:
        return int(self.sizes().n_inputs)

    @property
    def n_disturbances(self) -> int:
        return int(self.sizes().n_disturbances)

    def n_rows(self) -> int:
        return int(self.sizes().rows)

    @property
    def state_dim(self) -> int:
        return int(self.sizes().n_dim)

    def dynamics_image(self, row: int) -> np.ndarray:
        mu = np.zeros(self.state_dim)
        call("gm_dynamics_image", self._h, C.c_int64(row), mu.ctypes.data_as(C.POINTER(C.c_double)))
        return mu

    def use_spec(self, spec: Spec) -> None:
        if spec is self.spec:  # the configuration's own spec is already engine-side
            return
        n = self.state_dim

        def arr(b, which):
            if b is None:
                return None
            v = np.ascontiguousarray(getattr(b, which), dtype=np.float64)
            if v.size != n:  # dimension mismatch: let validation report it
                v = np.resize(v, n)
            return v

        kind = _KIND.get(spec.kind)
        if kind is None:
            raise ConfigError(f"unknown specification kind '{spec.kind}'")
        tl, th = arr(spec.target, "lo"), arr(spec.target, "hi")
        al, ah = arr(spec.avoid, "lo"), arr(spec.avoid, "hi")
        dp = C.POINTER(C.c_double)
        cast = (lambda a: a.ctypes.data_as(dp) if a is not None else None)
        if spec.target is not None and spec.target.dim != n:
            raise ConfigError("target box dimension does not match the state grid")
        if spec.avoid is not None and spec.avoid.dim != n:
            raise ConfigError("avoid box dimension does not match the state grid")
        call("gm_model_set_spec", self._h, kind, int(spec.horizon), cast(tl), cast(th), cast(al), cast(ah))
        self._keep = (tl, th, al, ah)

    def use_options(self, opts: SynthesisOptions) -> None:
        mode = {"matrix": _capi.GM_MODE_MATRIX, "ofa": _capi.GM_MODE_OFA}[opts.mode]
        call("gm_model_set_options", self._h, mode, int(opts.memory_budget))


def _model_from_text(text: str, name: str, overrides: Optional[dict] = None) -> SystemModel:
    h = C.c_void_p()
    ov = _overrides(overrides)
    call("gm_model_parse", text.encode(), name.encode(), C.byref(ov) if ov else None, C.byref(h))
    return SystemModel(h, text)


def _overrides(d: Optional[dict]):
    if not d:
        return None
    ov = _capi.Overrides(threads=-1, time_steps=-1, mem_budget=-1, seed=-1, runs=-1, mode=None, output=None)
    for k, v in d.items():
        if k in ("mode", "output"):
            setattr(ov, k, v.encode())
        else:
            setattr(ov, k, int(v))
    return ov


def load_config(path: str, **overrides) -> SystemModel:
    """load_config + build_model (+ build_spec / build_options) in one step.

    Overrides mirror the CLI flags (gridmdp_main.cpp:31-41): threads,
    time_steps, mem_budget, seed, runs, mode, output."""
    h = C.c_void_p()
    ov = _overrides(overrides)
    call("gm_model_load", str(path).encode(), C.byref(ov) if ov else None, C.byref(h))
    return SystemModel(h)


def parse_config(text: str, name: str = "<config>", **overrides) -> SystemModel:
    return _model_from_text(text, name, overrides)


def benchmark_chain_config(n: int) -> str:
    """benchmark_chain_config (config.hpp:70, config.cpp:374-394): the Table-3 scaling
    family as configuration text: n states in {0, 1}^n, x_i' = 0.9 x_i + 0 u0, normal
    noise sigma 0.5, cutting probability 0.05, safety, T = 6, matrix mode."""
    if n < 1:
        raise ConfigError("benchmark_chain_config: dimension must be positive")
    z, one = ", ".join(["0.0"] * n), ", ".join(["1.0"] * n)
    lines = [f"states.dim = {n};", f"states.lb = {{{z}}};", f"states.ub = {{{one}}};",
             f"states.eta = {{{one}}};", "inputs.dim = 1;", "inputs.lb = {0.0};", "inputs.ub = {0.0};",
             "inputs.eta = {1.0};"]
    lines += [f"dynamics.x{i} = 0.9*x{i} + 0*u0;" for i in range(n)]
    lines += ["noise.type = normal;", f"noise.sigma = {{{', '.join(['0.5'] * n)}}};",
              "noise.cutting_probability = 0.05;", "spec.type = safety;", "spec.time_steps = 6;",
              "exec.mode = matrix;"]
    return "\n".join(lines) + "\n"


def make_model(state: Grid, input: Grid, disturbance: Optional[Grid], dynamics: Sequence[str],
               noise: NoiseSpec, constants: Optional[dict] = None) -> SystemModel:
    """make_model (model.hpp:40-42) from grids, expression texts and noise."""
    lines = []
    for name, g in (("states", state), ("inputs", input), ("disturbances", disturbance)):
        if g is None or (name == "disturbances" and g.dim == 0):
            continue
        lines += [f"{name}.dim = {g.dim};", f"{name}.lb = {_vec(g.lb)};", f"{name}.ub = {_vec(g.ub)};",
                  f"{name}.eta = {_vec(g.eta)};"]
    for k, v in (constants or {}).items():
        lines.append(f"constants.{k} = {_fmt(v)};")
    for i, e in enumerate(dynamics):
        lines.append(f"dynamics.x{i} = {e};")
    lines += noise.config_lines()
    lines += ["spec.type = safety;", "spec.time_steps = 1;"]
    return _model_from_text("\n".join(lines) + "\n", "<model>")


# ----------------------------------------------------------------- stage (i)

def window_extents(m: SystemModel) -> list[int]:
    s = m.sizes()
    return [int(s.extents[d]) for d in range(s.n_dim)]


def memory_estimate(m: SystemModel) -> int:
    s = m.sizes()
    if s.size_overflow:
        raise MemoryError("memory_estimate: size arithmetic overflows 64 bits")
    return int(s.memory_estimate)


class TransitionMatrix:
    """Device-resident slab storage (abstraction.hpp:22-65)."""

    def __init__(self, model: SystemModel, handle: C.c_void_p):
        self.model = model
        self._h = handle
        s = model.sizes()
        rb, re_, R = C.c_int64(), C.c_int64(), C.c_int64()
        call("gm_matrix_info", handle, C.byref(rb), C.byref(re_), C.byref(R), None, None)
        self.row_begin, self.row_end, self._R = rb.value, re_.value, R.value
        self._extents = [int(s.extents[d]) for d in range(s.n_dim)]
        self._strides = [int(s.strides[d]) for d in range(s.n_dim)]
        self.n_inputs, self.n_disturbances = int(s.n_inputs), int(s.n_disturbances)
        self._origins = None
        self._payload = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:
            lib.gm_matrix_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def rows(self) -> int:
        return self.row_end - self.row_begin

    def row_width(self) -> int:
        return self._R

    def window_extents(self) -> list[int]:
        return list(self._extents)

    def row_index(self, ix: int, iu: int, iw: int) -> int:
        return (ix * self.n_inputs + iu) * self.n_disturbances + iw

    def _fetch(self):
        n = self.rows()
        o = np.empty(n, dtype=np.int64)
        p = np.empty((n, self._R), dtype=np.float64)
        call("gm_matrix_copy_rows", self._h, self.row_begin, self.row_end, ptr(o), ptr(p))
        self._origins, self._payload = o, p

    def invalidate(self):
        self._origins = self._payload = None

    def origins(self) -> np.ndarray:
        if self._origins is None:
            self._fetch()
        return self._origins

    def payload(self) -> np.ndarray:
        if self._payload is None:
            self._fetch()
        return self._payload

    def origin(self, r: int) -> int:
        return int(self.origins()[r])

    def row(self, r: int) -> np.ndarray:
        return self.payload()[r]

    def row_sum(self, r: int) -> float:
        return float(math.fsum(self.row(r)))  # tests only

    def prob(self, r: int, post: int) -> float:
        """Dense lookup (abstraction.cpp:227-244)."""
        rem_o, rem_p, k = self.origin(r), post, 0
        for d, s in enumerate(self._strides):
            jo, rem_o = divmod(rem_o, s)
            jp, rem_p = divmod(rem_p, s)
            off = jp - jo
            if off < 0 or off >= self._extents[d]:
                return 0.0
            k = k * self._extents[d] + off
        return float(self.row(r)[k])

    def write(self, path: str) -> None:
        """write_matrix (io.cpp:236-256)."""
        call("gm_matrix_write", self._h, self.model.handle, str(path).encode())


def build_matrix(m: SystemModel, threads: int = 0, rows: Optional[tuple] = None) -> TransitionMatrix:
    r0, r1 = rows if rows else (0, m.n_rows())
    h = C.c_void_p()
    call("gm_build_matrix", m.handle, C.c_int64(r0), C.c_int64(r1), C.byref(h))
    return TransitionMatrix(m, h)


def read_matrix(path: str, model: SystemModel) -> TransitionMatrix:
    """read_matrix (io.hpp:18, io.cpp:258-283) onto the device; the container's shape is
    checked against `model` when the matrix is used with it."""
    h = C.c_void_p()
    call("gm_matrix_read", str(path).encode(), C.byref(h))
    return TransitionMatrix(model, h)


def upload_matrix(m: SystemModel, origins: np.ndarray, probs: np.ndarray, row_begin: int = 0) -> TransitionMatrix:
    """A host TransitionMatrix (origins int64[rows], probs f64[rows, R]) onto the device."""
    o = np.ascontiguousarray(origins, dtype=np.int64)
    p = np.ascontiguousarray(probs, dtype=np.float64)
    h = C.c_void_p()
    call("gm_matrix_upload", m.handle, C.c_int64(row_begin), C.c_int64(o.size), ptr(o), ptr(p), C.byref(h))
    return TransitionMatrix(m, h)


def save_config(m: SystemModel, path: str) -> None:
    """save_config (config.hpp:59-60, config.cpp:270-310)."""
    call("gm_model_save_config", m.handle, str(path).encode())


def build_target_hit(m: SystemModel, spec: Spec, threads: int = 0) -> np.ndarray:
    m.use_spec(spec)
    n = m.n_rows()
    out = np.empty(n, dtype=np.float64)
    call("gm_build_target_hit", m.handle, C.c_int64(0), C.c_int64(n), ptr(out))
    return out


def mask_absorbing(tm: TransitionMatrix, spec: Spec, threads: int = 0) -> TransitionMatrix:
    tm.model.use_spec(spec)
    call("gm_mask_absorbing", tm.model.handle, tm.handle)
    tm.invalidate()
    return tm


def absorbing_states(m: SystemModel, spec: Spec) -> np.ndarray:
    m.use_spec(spec)
    out = np.zeros(m.n_states, dtype=np.uint8)
    call("gm_absorbing_states", m.handle, ptr(out))
    return out


# ---------------------------------------------------------------- stage (ii)

@dataclass
class SynthesisResult:
    """synthesis.hpp:28-40; values n_x x (T+1), policy / worst_dist n_x x T."""

    values: np.ndarray
    policy: np.ndarray
    worst_dist: np.ndarray
    absorbing: np.ndarray
    mode: str
    spec: Spec
    model: SystemModel = field(repr=False)
    _h: Optional[C.c_void_p] = field(default=None, repr=False)  # built from tables by write()
    _owner: Optional["_ResultOwner"] = field(default=None, repr=False)  # engine result the arrays view

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.gm_result_free(self._h)
            self._h = None

    def _handle(self) -> Optional[C.c_void_p]:
        return self._owner.h if self._owner is not None else self._h

    def write(self, path: str) -> None:
        """write_results (io.cpp:142-179)."""
        h = self._handle()
        if not h:
            h = C.c_void_p()
            v = np.asfortranarray(self.values, dtype=np.float64)
            p = np.asfortranarray(self.policy, dtype=np.uint32)
            w = np.asfortranarray(self.worst_dist, dtype=np.uint32)
            self.model.use_spec(self.spec)
            call("gm_result_from_tables", self.model.handle, ptr(v), ptr(p), ptr(w), C.byref(h))
            self._h = h
        call("gm_result_write", h, str(path).encode())


class _ResultOwner:
    """Owns an engine result; the SynthesisResult arrays are views of its tables and
    keep it alive (through their ctypes buffers)."""

    def __init__(self, h: C.c_void_p):
        self.h = h

    def __del__(self):
        if self.h and lib is not None:
            lib.gm_result_free(self.h)
            self.h = None


def _table(owner: _ResultOwner, addr: Optional[int], ctype, shape: tuple, dtype) -> np.ndarray:
    """Column-major (n_x, k) view of an engine table, or an empty array."""
    n = int(np.prod(shape))
    if n == 0 or not addr:
        return np.zeros(shape, dtype=dtype, order="F")
    buf = (ctype * n).from_address(addr)
    buf._owner = owner  # the view's base chain keeps the engine result alive
    a = np.frombuffer(buf, dtype=dtype)
    return a.reshape(shape[::-1]).T if len(shape) == 2 else a


_VPT = C.c_void_p


def _result_from_handle(m: SystemModel, spec: Spec, h: C.c_void_p) -> SynthesisResult:
    """Zero-copy: the returned arrays view the engine result's host tables."""
    owner = _ResultOwner(h)
    n_x, T, has_abs, mode = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32()
    call("gm_result_shape", h, C.byref(n_x), C.byref(T), C.byref(has_abs), C.byref(mode))
    nx, t = n_x.value, T.value
    pv, pp, pw, pa = _VPT(), _VPT(), _VPT(), _VPT()
    call("gm_result_data", h, C.byref(pv), C.byref(pp), C.byref(pw), C.byref(pa))
    vals = _table(owner, pv.value, C.c_double, (nx, t + 1), np.float64)
    pol = _table(owner, pp.value, C.c_uint32, (nx, t), np.uint32)
    wst = _table(owner, pw.value, C.c_uint32, (nx, t), np.uint32)
    ab = _table(owner, pa.value, C.c_uint8, (nx,), np.uint8) if has_abs.value else np.zeros(0, dtype=np.uint8)
    mode_s = "ofa" if mode.value == _capi.GM_MODE_OFA else "matrix"
    return SynthesisResult(vals, pol, wst, ab, mode_s, spec, m, None, owner)


def synthesize(m: SystemModel, spec: Optional[Spec] = None, opts: Optional[SynthesisOptions] = None
               ) -> SynthesisResult:
    spec = spec or m.spec
    opts = opts or m.options
    m.use_spec(spec)
    m.use_options(opts)
    h = C.c_void_p()
    call("gm_synthesize", m.handle, C.byref(h))
    return _result_from_handle(m, spec, h)


def synthesize_multi(m: SystemModel, devices, spec: Optional[Spec] = None, opts: Optional[SynthesisOptions] = None,
                     exchange: str = "auto", transport: str = "nccl"):
    """synthesize over several GPUs of this process (gm_synthesize_multi): state shards,
    one host thread + stream per device, V exchanged per step by `exchange`
    ("auto" | "halo" | "allgather") over `transport` ("nccl" | "peer" | "store"; "peer"
    and "store" accept a device listed several times; "store": the pass-2 epilogue
    writes each value straight into the peers' value tables). Returns
    (SynthesisResult, stats dict)."""
    spec = spec or m.spec
    opts = opts or m.options
    m.use_spec(spec)
    m.use_options(opts)
    dev = (C.c_int32 * len(devices))(*devices)
    xchg = {"auto": _capi.GM_XCHG_AUTO, "halo": _capi.GM_XCHG_HALO, "allgather": _capi.GM_XCHG_ALLGATHER}[exchange]
    xport = {"nccl": _capi.GM_XPORT_NCCL, "peer": _capi.GM_XPORT_PEER, "store": _capi.GM_XPORT_STORE}[transport]
    h = C.c_void_p()
    ms = _capi.MultiStats()
    call("gm_synthesize_multi", m.handle, C.c_int32(len(devices)), C.cast(dev, C.c_void_p), C.c_int32(xchg),
         C.c_int32(xport), C.byref(h), C.byref(ms))
    stats = {k: getattr(ms, k) for k, _ in _capi.MultiStats._fields_}
    stats["exchange_used"] = {0: "none", 1: "halo", 2: "allgather"}[ms.exchange_used]
    stats["transport_used"] = transport
    return _result_from_handle(m, spec, h), stats


def release_cached_memory() -> None:
    """Returns the engine's cached large device blocks (released matrices) to the driver."""
    lib.gm_release_cached_memory()


def last_times(m: SystemModel) -> tuple[float, float]:
    """(build_ms, sweep_ms) device time of the model's last synthesize (CUDA events)."""
    b, w = C.c_double(), C.c_double()
    call("gm_model_last_times", m.handle, C.byref(b), C.byref(w))
    return b.value, w.value


def synthesize_with_matrix(m: SystemModel, tm: TransitionMatrix, t0x: Optional[np.ndarray], spec: Spec,
                           opts: Optional[SynthesisOptions] = None) -> SynthesisResult:
    m.use_spec(spec)
    if opts:
        m.use_options(opts)
    h = C.c_void_p()
    t = None if t0x is None else np.ascontiguousarray(t0x, dtype=np.float64)
    call("gm_synthesize_with_matrix", m.handle, tm.handle, ptr(t), C.byref(h))
    tm.invalidate()
    return _result_from_handle(m, spec, h)


def bellman_step(m: SystemModel, spec: Spec, tm: Optional[TransitionMatrix], t0x: Optional[np.ndarray],
                 v_next: np.ndarray, threads: int = 0):
    """One backward step (synthesis.cpp:147-161). Returns (v_out, policy, worst_dist)."""
    m.use_spec(spec)
    v_next = np.ascontiguousarray(v_next, dtype=np.float64)
    if v_next.size != m.n_states:
        raise ConfigError("bellman_step: v_next size does not match the state grid")
    if tm is not None and spec.is_reach() and t0x is None:
        raise ConfigError("bellman_step: matrix-backed reach step requires the target-hit vector")
    n = m.n_states
    v_out = np.empty(n, dtype=np.float64)
    pol = np.empty(n, dtype=np.uint32)
    wst = np.empty(n, dtype=np.uint32)
    t = None if t0x is None else np.ascontiguousarray(t0x, dtype=np.float64)
    call("gm_bellman_step", m.handle, tm.handle if tm is not None else None, ptr(t), ptr(v_next), ptr(v_out),
         ptr(pol), ptr(wst))
    return v_out, pol, wst


def row_values(m: SystemModel) -> np.ndarray:
    """v_in of the model's most recent step: (n_x, n_u, n_w) expected values."""
    s = m.sizes()
    out = np.empty(int(s.rows), dtype=np.float64)
    call("gm_copy_row_values", m.handle, ptr(out), C.c_int64(out.size))
    return out.reshape(int(s.n_states), int(s.n_inputs), int(s.n_disturbances))


def q_values(m: SystemModel) -> np.ndarray:
    """min over disturbances of row_values (strict <, synthesis.cpp:121-127): (n_x, n_u)."""
    return row_values(m).min(axis=2)


def query_policy(res: SynthesisResult, input_grid: Grid, state_grid: Grid, x, k: int) -> np.ndarray:
    """Input prescribed at continuous state x and step k (synthesis.cpp:230-239)."""
    h = res._handle()
    if h:  # gm_query_policy over the engine result's own grids
        x = np.ascontiguousarray(x, dtype=np.float64)
        u = np.empty(input_grid.dim, dtype=np.float64)
        call("gm_query_policy", h, ptr(x), C.c_int32(x.size), C.c_int32(k), u.ctypes.data_as(C.POINTER(C.c_double)))
        return u
    T = res.spec.horizon
    if k < 1 or k > T:
        raise IndexError(f"query_policy: step {k} outside [1, {T}]")
    ix = state_grid.index(x)
    return input_grid.point(int(res.policy[ix, k - 1]))


def write_results(res: SynthesisResult, path: str) -> None:
    res.write(path)


def read_results(path: str, model: Optional[SystemModel] = None) -> SynthesisResult:
    """read_results (io.hpp:14, io.cpp:181-230): a `gridmdp-results 1` container."""
    h = C.c_void_p()
    call("gm_result_read", str(path).encode(), C.byref(h))
    return _result_from_handle(model, None, h)


def value_at(res: SynthesisResult, x, k: int = 0) -> float:
    """values(point_to_index(state_grid, x), k) (gridmdp_main.cpp:133-134)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    v = C.c_double()
    call("gm_result_value_at", res._handle(), ptr(x), C.c_int32(x.size), C.c_int32(k), C.byref(v))
    return v.value


@dataclass
class TrajectoryBatch:
    """sim.hpp:24-27: per-run outcome and (optionally) the rollouts, [run][k][d]
    arrays with T+1 state rows and T input / disturbance rows per run; a run that
    resolves early uses the first steps[r] (+1) rows."""

    runs: int
    satisfied: np.ndarray
    steps: np.ndarray
    states: Optional[np.ndarray] = None
    inputs: Optional[np.ndarray] = None
    dists: Optional[np.ndarray] = None
    _h: Optional[C.c_void_p] = field(default=None, repr=False)

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.gm_sim_free(self._h)
            self._h = None

    def empirical_rate(self) -> float:
        return empirical_rate(self)

    def write_csv(self, path: str) -> None:
        write_trajectory_csv(self, path)


def simulate(m: SystemModel, spec: Optional[Spec], res: SynthesisResult, x0, runs: Optional[int] = None,
             seed: Optional[int] = None, dmode: str = "random", threads: int = 0,
             trajectories: bool = False) -> TrajectoryBatch:
    """simulate (sim.hpp:42-44, sim.cpp:85-101) on the GPU, one thread per run, under
    the result's policy and spec (as `gridmdp simulate` passes res.spec). runs / seed
    default to the configuration's exec.runs / exec.seed. `spec` and `threads` are
    accepted for signature parity; statistical (not stream) parity with the reference."""
    del spec, threads
    if dmode not in ("random", "worst_case", "worst-case"):
        raise ConfigError(f"simulate: unknown disturbance mode '{dmode}'")
    r0, s0 = C.c_int32(), C.c_uint64()
    call("gm_model_sim_defaults", m.handle, C.byref(r0), C.byref(s0))
    runs = r0.value if runs is None else int(runs)
    seed = s0.value if seed is None else int(seed)
    if res._handle() is None:  # tables built in Python: hand them to the engine
        h0 = C.c_void_p()
        v = np.asfortranarray(res.values, dtype=np.float64)
        p = np.asfortranarray(res.policy, dtype=np.uint32)
        w = np.asfortranarray(res.worst_dist, dtype=np.uint32)
        m.use_spec(res.spec)
        call("gm_result_from_tables", m.handle, ptr(v), ptr(p), ptr(w), C.byref(h0))
        res._h = h0
    x = np.ascontiguousarray(x0, dtype=np.float64)
    h = C.c_void_p()
    call("gm_simulate", m.handle, res._handle(), ptr(x), C.c_int32(x.size), C.c_int32(runs), C.c_uint64(seed),
         C.c_int32(1 if dmode != "random" else 0), C.c_int32(1 if trajectories else 0), C.byref(h))
    n_runs, sat_n, rate = C.c_int32(), C.c_int64(), C.c_double()
    call("gm_sim_summary", h, C.byref(n_runs), C.byref(sat_n), C.byref(rate))
    sat = np.empty(runs, dtype=np.uint8)
    steps = np.empty(runs, dtype=np.int32)
    st = inp = ds = None
    if trajectories:
        T = res.values.shape[1] - 1
        sz = m.sizes()
        n, mu, pd = int(sz.n_dim), int(sz.m_dim), int(sz.p_dim)
        st = np.empty((runs, T + 1, n))
        inp = np.empty((runs, T, mu))
        ds = np.empty((runs, T, pd))
    call("gm_sim_copy", h, ptr(sat), ptr(steps), ptr(st), ptr(inp) if inp is not None and inp.size else None,
         ptr(ds) if ds is not None and ds.size else None)
    return TrajectoryBatch(runs, sat.astype(bool), steps, st, inp, ds, h)


def empirical_rate(batch: TrajectoryBatch) -> float:
    """Fraction of satisfied runs (sim.cpp:103-108)."""
    if batch.runs < 1:
        raise ConfigError("empirical_rate: empty batch")
    return float(np.count_nonzero(batch.satisfied)) / batch.runs


def write_trajectory_csv(batch: TrajectoryBatch, path: str) -> None:
    """write_trajectory_csv (sim.cpp:117-154)."""
    call("gm_sim_write_csv", batch._h, str(path).encode())


def launch_count() -> int:
    return int(lib.gm_launch_count())
