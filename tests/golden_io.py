"""Readers for the reference's container formats (io.cpp:142-283) and the
committed golden fixtures under tests/golden/ (see make_golden.py)."""
from __future__ import annotations

import gzip
import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
CASES = GOLDEN / "cases"
OUT = GOLDEN / "out"


def _manifest(blob: bytes, magic: str):
    head, _, rest = blob.partition(b"\n")
    m, ver = head.decode().split()
    assert m == magic and ver == "1", head
    kv = {}
    pos = len(head) + 1
    while True:
        nl = blob.index(b"\n", pos)
        line = blob[pos:nl].decode()
        pos = nl + 1
        if line == "payload":
            break
        k, v = line[:-1].split("=", 1)
        kv[k.strip()] = v.strip()
    return kv, pos


def read_results(blob: bytes) -> dict:
    """read_results (io.cpp:181-230) -> values (n_x, T+1), policy/worst (n_x, T), absorbing."""
    kv, pos = _manifest(blob, "gridmdp-results")
    _, n_x, cols = kv["array.values"].split()
    n_x, cols = int(n_x), int(cols)
    T = cols - 1
    n_abs = int(kv["array.absorbing"].split()[1])
    o = pos
    vals = np.frombuffer(blob, "<f8", n_x * cols, o).reshape(n_x, cols)
    o += n_x * cols * 8
    pol = np.frombuffer(blob, "<u4", n_x * T, o).reshape(n_x, T)
    o += n_x * T * 4
    wst = np.frombuffer(blob, "<u4", n_x * T, o).reshape(n_x, T)
    o += n_x * T * 4
    ab = np.frombuffer(blob, "u1", n_abs, o)
    o += n_abs
    assert o == len(blob), "trailing bytes"
    return {"manifest": kv, "values": vals, "policy": pol, "worst": wst, "absorbing": ab}


def read_matrix(blob: bytes) -> dict:
    """read_matrix (io.cpp:258-283) -> origins (rows,), probs (rows, R), window."""
    kv, pos = _manifest(blob, "gridmdp-matrix")
    rows = int(kv["array.origins"].split()[1])
    R = int(kv["array.probs"].split()[2])
    org = np.frombuffer(blob, "<i8", rows, pos)
    probs = np.frombuffer(blob, "<f8", rows * R, pos + rows * 8).reshape(rows, R)
    assert pos + rows * 8 + rows * R * 8 == len(blob)
    window = [int(x) for x in kv["window"].strip("{}").split(",")]
    return {"manifest": kv, "origins": org, "probs": probs, "window": window}


def manifest() -> dict:
    return json.loads((GOLDEN / "manifest.json").read_text())


def load(name: str) -> bytes:
    return gzip.decompress((OUT / (name if name.endswith(".gz") else name + ".gz")).read_bytes())


def case_cfg(case: str) -> Path:
    return CASES / f"{case}.cfg"


def case_overrides(entry: dict) -> dict:
    ov = {}
    it = iter(entry.get("overrides", []))
    for k in it:
        v = next(it)
        ov[k.lstrip("-").replace("-", "_")] = int(v) if v.lstrip("-").isdigit() else v
    return ov


def golden_results(case: str) -> dict:
    e = manifest()["cases"][case]
    return read_results(load(e["results"]))


def golden_step(case: str, mode: str):
    e = manifest()["cases"][case]
    pre = e["files"]["step_prefix"] + "_" + mode
    v = np.frombuffer(load(pre + ".v"), "<f8")
    p = np.frombuffer(load(pre + ".pol"), "<u4")
    w = np.frombuffer(load(pre + ".wst"), "<u4")
    vn = np.frombuffer(load(e["files"]["vnext"]), "<f8")
    return vn, v, p, w


def tol_ok(got, want, rel=1e-9, abs_=1e-15):
    """North-star parity bar: |gpu - cpu| <= 1e-9 |cpu| + 1e-15."""
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return np.abs(got - want) <= rel * np.abs(want) + abs_


def policy_ok(q_gpu, pol_gpu, pol_ref, rel=1e-9, abs_=1e-15):
    """Policies agree except on ties within tolerance: where they differ, the
    reference's choice must be within tolerance of the GPU's best under the GPU's
    own per-input values q_gpu (n_x, n_u)."""
    pol_gpu, pol_ref = np.asarray(pol_gpu), np.asarray(pol_ref)
    diff = np.nonzero(pol_gpu != pol_ref)[0]
    if diff.size == 0:
        return True, 0
    a = q_gpu[diff, pol_gpu[diff]]
    b = q_gpu[diff, pol_ref[diff]]
    ok = np.abs(a - b) <= rel * np.abs(a) + abs_
    return bool(ok.all()), int(diff.size)


# ---------------------------------------------------------------- full-size goldens
LARGE = GOLDEN / "large"


def large_manifest() -> dict:
    return json.loads((LARGE / "manifest.json").read_text())


def large_results(name: str) -> dict:
    return read_results(gzip.decompress((LARGE / large_manifest()[name]["results"]).read_bytes()))


def large_cfg(name: str) -> Path:
    return LARGE / large_manifest()[name]["config"]


def large_array(name: str, dtype) -> np.ndarray:
    return np.frombuffer(gzip.decompress((LARGE / f"{name}.gz").read_bytes()), dtype)


def hashed_v(n: int) -> np.ndarray:
    """The v_next of the C2b step golden (make_golden_large.hashed_v): splitmix64 of
    the state index, top 53 bits, in [0, 1)."""
    z = np.arange(n, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
