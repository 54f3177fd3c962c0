"""Python front end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Parses the reference's `key = value;` configuration (config.cpp:68-237 rules:
'#' comments, braced vectors, constants.*, optional disturbances/target/avoid)
into the oracle's model descriptor and calls oracle/_build/libgm_oracle.so,
the C restatement of the reference hot path (gm_oracle.c). Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libgm_oracle.so"
_FAM = {"normal": 0, "uniform": 1, "exponential": 2, "beta": 3}
_KIND = {"safety": 0, "reachability": 1, "reach-avoid": 2, "reach_avoid": 2}


class Desc(C.Structure):
    _fields_ = [("n", C.c_int), ("m", C.c_int), ("p", C.c_int)] + [
        (k, C.POINTER(C.c_double)) for k in ("xlb", "xub", "xeta", "ulb", "uub", "ueta", "wlb", "wub", "weta")] + [
        ("dyn", C.POINTER(C.c_char_p)), ("n_const", C.c_int), ("const_names", C.POINTER(C.c_char_p)),
        ("const_vals", C.POINTER(C.c_double)), ("family", C.c_int), ("mult", C.c_int), ("gamma", C.c_double),
        ("p1", C.POINTER(C.c_double)), ("p2", C.POINTER(C.c_double)), ("spec_kind", C.c_int),
        ("horizon", C.c_int), ("has_target", C.c_int), ("has_avoid", C.c_int)] + [
        (k, C.POINTER(C.c_double)) for k in ("tlo", "thi", "alo", "ahi")]


def _lib():
    if not LIB.exists():
        subprocess.run(["make", "-C", str(HERE), "oracle"], check=True, capture_output=True)
    lib = C.CDLL(str(LIB))
    P, I64, VP = C.POINTER, C.c_int64, C.c_void_p
    lib.oc_model_new.argtypes = [P(Desc), P(VP), C.c_char_p, C.c_int]
    lib.oc_model_free.argtypes = [VP]
    lib.oc_sizes.argtypes = [VP, VP, P(C.c_uint64)]
    lib.oc_absorbing.argtypes = [VP, VP]
    lib.oc_build_matrix.argtypes = [VP, I64, I64, VP, VP, C.c_int, C.c_char_p, C.c_int]
    lib.oc_target_hit.argtypes = [VP, I64, I64, VP, C.c_int, C.c_char_p, C.c_int]
    lib.oc_mask.argtypes = [VP, I64, VP, VP]
    lib.oc_bellman_step.argtypes = [VP, VP, VP, VP, I64, I64, VP, VP, VP, VP, VP, C.c_int, C.c_char_p, C.c_int]
    lib.oc_synthesize.argtypes = [VP, C.c_int, VP, VP, VP, C.c_int, C.c_char_p, C.c_int]
    return lib


_L = None


def lib():
    global _L
    if _L is None:
        _L = _lib()
    return _L


def parse_config(text: str, overrides: dict | None = None) -> dict:
    """Statement map of a configuration (config.cpp:70-91) with CLI overrides."""
    st = {}
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        assert line.endswith(";"), line
        k, v = line[:-1].split("=", 1)
        st[k.strip()] = v.strip()
    for k, v in (overrides or {}).items():
        st[{"time_steps": "spec.time_steps", "mode": "exec.mode"}.get(k, k)] = str(v)
    return st


def _vec(s: str) -> list[float]:
    s = s.strip()
    assert s[0] == "{" and s[-1] == "}", s
    return [float(x) for x in s[1:-1].split(",")]


def _arr(v):
    a = np.ascontiguousarray(v, dtype=np.float64)
    return a, a.ctypes.data_as(C.POINTER(C.c_double))


class OracleModel:
    def __init__(self, st: dict):
        self.st = st
        keep = []

        def dv(v):
            a, p = _arr(v if len(v) else [0.0])
            keep.append(a)
            return p

        d = Desc()
        grids = {}
        for pre, attr in (("states", "x"), ("inputs", "u"), ("disturbances", "w")):
            if f"{pre}.dim" in st:
                dim = int(st[f"{pre}.dim"])
                lb, ub, eta = (_vec(st[f"{pre}.{k}"]) for k in ("lb", "ub", "eta"))
            else:
                dim, lb, ub, eta = 0, [], [], []
            grids[attr] = dim
            setattr(d, attr + "lb", dv(lb))
            setattr(d, attr + "ub", dv(ub))
            setattr(d, attr + "eta", dv(eta))
        d.n, d.m, d.p = grids["x"], grids["u"], grids["w"]
        dyn = [st[f"dynamics.x{i}"].encode() for i in range(d.n)]
        dyn_arr = (C.c_char_p * len(dyn))(*dyn)
        names = sorted(k[10:] for k in st if k.startswith("constants."))
        cn = (C.c_char_p * max(1, len(names)))(*[n.encode() for n in names])
        cv = dv([float(st["constants." + n]) for n in names])
        keep += [dyn_arr, cn, dyn]
        d.dyn, d.n_const, d.const_names, d.const_vals = dyn_arr, len(names), cn, cv
        fam = st["noise.type"]
        d.family = _FAM[fam]
        d.mult = 1 if st.get("noise.mode", "additive") == "multiplicative" else 0
        d.gamma = float(st.get("noise.cutting_probability", "0"))
        k1, k2 = {"normal": ("sigma", None), "uniform": ("a", "b"), "exponential": ("rate", None),
                  "beta": ("alpha", "beta")}[fam]
        d.p1 = dv(_vec(st["noise." + k1]))
        d.p2 = dv(_vec(st["noise." + k2]) if k2 else [0.0] * d.n)
        d.spec_kind = _KIND[st["spec.type"]]
        d.horizon = int(st["spec.time_steps"])
        d.has_target = int("target.lb" in st)
        d.has_avoid = int("avoid.lb" in st)
        zero = [0.0] * d.n
        d.tlo = dv(_vec(st["target.lb"]) if d.has_target else zero)
        d.thi = dv(_vec(st["target.ub"]) if d.has_target else zero)
        d.alo = dv(_vec(st["avoid.lb"]) if d.has_avoid else zero)
        d.ahi = dv(_vec(st["avoid.ub"]) if d.has_avoid else zero)
        self._keep = keep
        self._desc = d
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        rc = lib().oc_model_new(C.byref(d), C.byref(h), err, 512)
        if rc:
            raise ValueError(f"oracle: {err.value.decode()} (rc={rc})")
        self.h = h
        out = (C.c_int64 * (5 + 12))()  # sizes + extents (OC_MAXD = 12)
        mem = C.c_uint64()
        lib().oc_sizes(h, out, C.byref(mem))
        self.n_x, self.n_u, self.n_w, self.rows, self.R = (int(out[i]) for i in range(5))
        self.extents = [int(out[5 + i]) for i in range(d.n)]
        self.memory_estimate = int(mem.value)
        self.horizon = d.horizon
        self.reach = d.spec_kind != 0

    def __del__(self):
        if getattr(self, "h", None):
            lib().oc_model_free(self.h)
            self.h = None

    def absorbing(self) -> np.ndarray:
        f = np.zeros(self.n_x, dtype=np.uint8)
        lib().oc_absorbing(self.h, f.ctypes.data)
        return f

    def _err(self, rc, err, what):
        if rc:
            raise RuntimeError(f"oracle {what}: {err.value.decode()} (rc={rc})")

    def build_matrix(self, r0=0, r1=None, threads=0):
        r1 = self.rows if r1 is None else r1
        o = np.empty(r1 - r0, dtype=np.int64)
        p = np.empty((r1 - r0, self.R), dtype=np.float64)
        err = C.create_string_buffer(512)
        self._err(lib().oc_build_matrix(self.h, r0, r1, o.ctypes.data, p.ctypes.data, threads, err, 512), err,
                  "build_matrix")
        return o, p

    def target_hit(self, r0=0, r1=None, threads=0):
        r1 = self.rows if r1 is None else r1
        t = np.empty(r1 - r0, dtype=np.float64)
        err = C.create_string_buffer(512)
        self._err(lib().oc_target_hit(self.h, r0, r1, t.ctypes.data, threads, err, 512), err, "target_hit")
        return t

    def mask(self, origins, probs):
        lib().oc_mask(self.h, len(origins), origins.ctypes.data, probs.ctypes.data)

    def bellman_step(self, v_next, x0=0, x1=None, probs=None, origins=None, t0x=None, threads=0):
        """One step over states [x0,x1): (v_out, policy, worst, v_in rows)."""
        x1 = self.n_x if x1 is None else x1
        n = x1 - x0
        v_next = np.ascontiguousarray(v_next, dtype=np.float64)
        vo = np.empty(n)
        pol = np.empty(n, dtype=np.uint32)
        wst = np.empty(n, dtype=np.uint32)
        vin = np.empty(max(1, n * self.n_u * self.n_w))
        err = C.create_string_buffer(512)
        ptr = (lambda a: None if a is None else a.ctypes.data)  # noqa: E731
        self._err(lib().oc_bellman_step(self.h, ptr(probs), ptr(origins), ptr(t0x), x0, x1, v_next.ctypes.data,
                                        vo.ctypes.data, pol.ctypes.data, wst.ctypes.data, vin.ctypes.data, threads,
                                        err, 512), err, "bellman_step")
        return vo, pol, wst, vin[: n * self.n_u * self.n_w].reshape(n, self.n_u, self.n_w)

    def synthesize(self, matrix: bool = False, threads=0) -> dict:
        T = self.horizon
        vals = np.empty((T + 1) * self.n_x)
        pol = np.empty(T * self.n_x, dtype=np.uint32)
        wst = np.empty(T * self.n_x, dtype=np.uint32)
        err = C.create_string_buffer(512)
        self._err(lib().oc_synthesize(self.h, int(matrix), vals.ctypes.data, pol.ctypes.data, wst.ctypes.data,
                                      threads, err, 512), err, "synthesize")
        return {"values": vals.reshape(T + 1, self.n_x).T, "policy": pol.reshape(T, self.n_x).T,
                "worst": wst.reshape(T, self.n_x).T, "absorbing": self.absorbing() if self.reach else
                np.zeros(0, np.uint8)}


def load(path_or_text: str | os.PathLike, **overrides) -> OracleModel:
    p = Path(path_or_text) if not str(path_or_text).lstrip().startswith(("states", "#")) else None
    text = p.read_text() if (p is not None and p.exists()) else str(path_or_text)
    return OracleModel(parse_config(text, overrides))


def synthesize_file(path, matrix=False, **overrides) -> dict:
    return load(path, **overrides).synthesize(matrix=matrix)
