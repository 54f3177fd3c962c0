"""Host front end and C-ABI boundary (no GPU needed): the shared library loads
and exports every function include/gridmdp_b200.h declares; sizes, windows and
memory estimates equal the reference's for every bundled config; config and
expression errors carry the reference's codes; compute without a device fails
loudly (no CPU fallback)."""
import ctypes
import subprocess

import numpy as np
import pytest

import golden_io as G
from paper_2005_06191_b200 import _capi
from paper_2005_06191_b200 import gridmdp as g

MAN = G.manifest()


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_capi.LIB_PATH))
    declared = _capi.declared_functions()
    assert len(declared) >= 35
    missing = [f for f in declared if not hasattr(lib, f)]
    assert not missing, missing
    assert set(declared) == set(_capi.SIGNATURES), set(declared) ^ set(_capi.SIGNATURES)


@pytest.mark.parametrize("name", sorted(MAN["estimate"]))
def test_sizes_match_reference(name):
    e = MAN["estimate"][name]
    m = g.parse_config(e["config"], name)
    s = m.sizes()
    want = e["sizes"]
    assert (s.n_states, s.n_inputs, s.n_disturbances, s.rows, s.row_width) == (
        want["states"], want["inputs"], want["disturbances"], want["rows"], want["row_width"])
    assert g.window_extents(m) == want["window"]
    assert g.memory_estimate(m) == want["memory_estimate_bytes"]


def test_known_windows():
    # test_abstraction.cpp:111-122 (degenerate), :212-230 (multiplicative -> full rows)
    assert g.window_extents(g.load_config(str(G.case_cfg("degenerate")))) == [1]
    assert g.window_extents(g.load_config(str(G.case_cfg("mult1d")))) == [5]
    m = g.make_model(g.make_grid([0.0], [1.0], [0.5]), g.make_grid([0.0], [0.0], [1.0]), None, ["x0 + u0"],
                     g.NoiseSpec.normal([1.0], 1e-3, "multiplicative"))
    assert g.window_extents(m) == [3] and g.memory_estimate(m) == 3 * 3 * 8 + 3 * 8 + 4096


def test_memory_estimate_overflow_is_memory_error():
    # test_abstraction.cpp:361-366
    m = g.make_model(g.make_grid([0.0], [1e7], [1.0]), g.make_grid([0.0], [1e6], [1.0]), None, ["x0 + u0"],
                     g.NoiseSpec.normal([1.0], 0.0))
    with pytest.raises(g.MemoryError):
        g.memory_estimate(m)


@pytest.mark.parametrize("text,code,needle", [
    ("states.dim = 1\n", "ConfigError", "statement must end with ';'"),
    ("states.dim = 1;\nstates.dim = 2;\n", "ConfigError", "duplicate key 'states.dim'"),
    ("states.dim = 1;\n", "ConfigError", "missing mandatory key 'states.lb'"),
])
def test_config_errors(text, code, needle):
    with pytest.raises(getattr(g, code)) as ei:
        g.parse_config(text, "bad.cfg")
    assert needle in str(ei.value)


def _tiny(**repl):
    text = (G.CASES / "tiny.cfg").read_text()
    for a, b in repl.items():
        text = text.replace(a, b)
    return text


@pytest.mark.parametrize("name", sorted(MAN["errors"]))
def test_cli_errors_match_reference(name, tmp_path):
    """Same exit code and message as the reference CLI for bad configurations
    (config.cpp, expr.cpp parser, grid/noise/spec validation)."""
    e = MAN["errors"][name]
    cfg = tmp_path / "bad.cfg"
    cfg.write_text(e["config"])
    r = _cli("synthesize", "-c", cfg, "-o", tmp_path / "r.bin")
    assert r.returncode == e["rc"]
    assert r.stderr.strip().replace(str(cfg), "<cfg>") == e["stderr"]


def test_dynamics_image_host_evaluator():
    # test_abstraction.cpp:85-88: robot mu at (x=0, nu=(0.7,0.8), w=0)
    m = g.load_config(str(G.case_cfg("ref_robot_safety_T2")))
    # robot_safety input pitch 0.2: nu=(0.6, 0.8) -> indices (8, 9); x=(0,0) -> 20*41+20; w=0 -> 5
    ix, iu, iw = 20 * 41 + 20, 8 * 11 + 9, 5
    mu = m.dynamics_image((ix * 121 + iu) * 11 + iw)
    assert abs(mu[0] - 10 * 0.6 * np.cos(0.8)) <= 1e-12 and abs(mu[1] - 10 * 0.8 * np.sin(0.8)) <= 1e-12


def test_compute_without_device_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    m = g.load_config(str(G.case_cfg("tiny")))
    with pytest.raises(g.CudaError, match="no CPU fallback"):
        g.synthesize(m)


def _cli(*args):
    return subprocess.run([str(_capi.CLI_PATH), *map(str, args)], capture_output=True, text=True)


def test_cli_estimate_mem_matches_reference():
    for name in ("robot_safety", "bmw7", "traffic5"):
        cfg = MAN["estimate"][name]["config"]
        p = G.GOLDEN / "out" / f"_{name}.cfg"
        p.write_text(cfg)
        try:
            r = _cli("estimate-mem", "-c", p)
        finally:
            p.unlink()
        assert r.returncode == 0, r.stderr
        s = MAN["estimate"][name]["sizes"]
        for key in ("states", "inputs", "disturbances", "state_input_pairs", "rows", "row_width"):
            assert f"{key}: {s[key]}\n" in r.stdout
        assert f"memory_estimate_bytes: {s['memory_estimate_bytes']}\n" in r.stdout


def test_cli_exit_codes(tmp_path):
    # test_cli.cpp:126-174
    bad = tmp_path / "bad.cfg"
    bad.write_text("states.dim = 1\n")
    assert _cli("estimate-mem", "-c", bad).returncode == 2
    assert _cli("estimate-mem", "-c", "/nonexistent/nope.cfg").returncode == 5
    t = tmp_path / "t.cfg"
    t.write_text(_tiny())
    r = _cli("synthesize", "-c", t, "--mode", "matrix", "--mem-budget", "64")
    assert r.returncode == 3 and "ofa" in r.stderr
    r = _cli("synthesize", "-c", t, "--time-steps", "5", "-o", tmp_path / "r.bin")
    assert "time_steps: 5" in r.stdout
    d = tmp_path / "d.cfg"
    d.write_text(_tiny(**{"0.7*x0 + 0.4*u0": "1/x0"}))
    r = _cli("abstract", "-c", d)
    import torch
    assert r.returncode == (4 if torch.cuda.is_available() else 1)


def test_benchmark_chain_generator_sizes():
    """benchmark_chain_config (config.cpp:374-394), test_config_io.cpp:137-143: n_x = 2^n, one input,
    for n = 1..12 (the engine's dimension limit is 12 per grid)."""
    from paper_2005_06191_b200 import gridmdp as g
    for n in range(1, 13):
        s = g.parse_config(g.benchmark_chain_config(n)).sizes()
        assert s.n_states == 1 << n and s.n_inputs == 1
    with pytest.raises(g.ConfigError):
        g.benchmark_chain_config(0)


@pytest.mark.parametrize("case", ["chain09", "ref_bmw7_desk", "ref_vehicle3_desk", "domain", "mult1d", "beta1d",
                                  "chain_bench12"])
def test_dynamics_compile_for_sm100a(case):
    """The generated straight-line dynamics (gm_jit.cpp) + gm_rowdev.cuh compile with NVRTC
    for sm_100a (no GPU needed): ite / goto, domain checks, 7- and 12-dim models."""
    import golden_io as G
    from paper_2005_06191_b200 import _capi
    from paper_2005_06191_b200 import gridmdp as g
    e = G.manifest()["cases"][case]
    m = g.load_config(str(G.case_cfg(case)), **G.case_overrides(e))
    secs = ctypes.c_double()
    _capi.call("gm_model_jit_compile", m.handle, ctypes.c_int32(0), ctypes.byref(secs))
    assert secs.value > 0


@pytest.mark.parametrize("workload", ["C2b", "C1", "C3u"])
def test_shape_specialised_build_compiles(workload):
    """The stage (i) build kernel specialised to the row shape (gm_jit.cpp shape_defines,
    gm_rowdev.cuh GM_FILL_*) compiles for sm_100a with NVRTC (no GPU needed)."""
    from paper_2005_06191_b200 import _capi
    from paper_2005_06191_b200 import gridmdp as g
    from paper_2005_06191_b200 import workloads as W
    m = g.parse_config(W.WORKLOADS[workload](), workload)
    secs = ctypes.c_double()
    _capi.call("gm_model_jit_compile", m.handle, ctypes.c_int32(2), ctypes.byref(secs))
    assert secs.value > 0


# ------------------------------------------- the reference's in-memory types (no GPU)

def _sizes_tuple(m):
    s = m.sizes()
    return (int(s.n_states), int(s.rows), int(s.row_width), int(s.memory_estimate),
            [int(s.extents[d]) for d in range(s.n_dim)], int(s.spec_kind), int(s.horizon), int(s.mode))


@pytest.mark.parametrize("name", ["robot_reachavoid", "bmw7", "vehicle3", "room5", "traffic5"])
def test_save_config_round_trip(name, tmp_path):
    """save_config (config.cpp:270-310) re-parses to the same model (parse(save(c)) == c)."""
    cfg = tmp_path / "a.cfg"
    cfg.write_text(MAN["estimate"][name]["config"])
    m = g.load_config(str(cfg))
    out = tmp_path / "saved.cfg"
    g.save_config(m, str(out))
    m2 = g.load_config(str(out))
    assert _sizes_tuple(m) == _sizes_tuple(m2)
    out2 = tmp_path / "saved2.cfg"
    g.save_config(m2, str(out2))
    assert out.read_text() == out2.read_text()


class ExprNode(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("var_class", ctypes.c_int32), ("var_index", ctypes.c_int32),
                ("kid", ctypes.c_int32 * 3), ("value", ctypes.c_double)]


class ExprDesc(ctypes.Structure):
    _fields_ = [("nodes", ctypes.POINTER(ExprNode)), ("n_nodes", ctypes.c_int32), ("root", ctypes.c_int32)]


class GridDesc(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("lb", ctypes.POINTER(ctypes.c_double)),
                ("ub", ctypes.POINTER(ctypes.c_double)), ("eta", ctypes.POINTER(ctypes.c_double))]


class ModelDesc(ctypes.Structure):
    _fields_ = [("state", GridDesc), ("input", GridDesc), ("disturbance", GridDesc),
                ("dynamics", ctypes.POINTER(ExprDesc)), ("n_dynamics", ctypes.c_int32),
                ("noise_family", ctypes.c_int32), ("noise_mode", ctypes.c_int32), ("gamma", ctypes.c_double),
                ("noise_dim", ctypes.c_int32), ("param1", ctypes.POINTER(ctypes.c_double)),
                ("param2", ctypes.POINTER(ctypes.c_double)), ("custom_pdf", ExprDesc),
                ("spec_kind", ctypes.c_int32), ("horizon", ctypes.c_int32),
                ("target_lo", ctypes.POINTER(ctypes.c_double)), ("target_hi", ctypes.POINTER(ctypes.c_double)),
                ("avoid_lo", ctypes.POINTER(ctypes.c_double)), ("avoid_hi", ctypes.POINTER(ctypes.c_double)),
                ("mode", ctypes.c_int32), ("threads", ctypes.c_int32), ("mem_budget", ctypes.c_uint64)]


def _dv(*v):
    return (ctypes.c_double * len(v))(*v)


# Expr::Op numbering (expr.hpp:38-45)
OP = {n: i for i, n in enumerate("add sub mul div pow lt le gt ge eq ne neg sin cos tan asin acos atan exp ln "
                                 "sqrt abs min max ite literal variable".split())}


def _tiny_desc(nodes, root, keep):
    """tiny.cfg (test_cli.cpp:33-50) as the reference holds it in memory: grids,
    x0' = 0.7*x0 + 0.4*u0 as a node pool, normal noise, safety T = 3."""
    arr = (ExprNode * len(nodes))(*nodes)
    dyn = (ExprDesc * 1)(ExprDesc(arr, len(nodes), root))
    vals = [_dv(-1.0), _dv(1.0), _dv(0.25), _dv(-0.5), _dv(0.5), _dv(0.5), _dv(0.3)]
    keep += [arr, dyn, vals]
    d = ModelDesc()
    d.state = GridDesc(1, vals[0], vals[1], vals[2])
    d.input = GridDesc(1, vals[3], vals[4], vals[5])
    d.disturbance = GridDesc(0, None, None, None)
    d.dynamics, d.n_dynamics = dyn, 1
    d.noise_family, d.noise_mode, d.gamma, d.noise_dim = 0, 0, 0.001, 1
    d.param1, d.param2 = vals[6], None
    d.spec_kind, d.horizon, d.mode = 0, 3, 0
    return d


def _node(op, value=0.0, vc=0, vi=0, kids=(-1, -1, -1)):
    return ExprNode(OP[op], vc, vi, (ctypes.c_int32 * 3)(*kids), value)


TINY_NODES = [_node("literal", 0.7), _node("variable", vc=0, vi=0), _node("mul", kids=(0, 1, -1)),
              _node("literal", 0.4), _node("variable", vc=1, vi=0), _node("mul", kids=(3, 4, -1)),
              _node("add", kids=(2, 5, -1))]


def test_model_create_from_reference_types_matches_config(tmp_path):
    """gm_model_create (the reference's SystemModel / Spec / SynthesisOptions over the
    C ABI) gives the model the configuration text gives: sizes, windows, and a
    save_config that re-parses to the same model."""
    keep = []
    d = _tiny_desc(TINY_NODES, 6, keep)
    h = ctypes.c_void_p()
    _capi.call("gm_model_create", ctypes.byref(d), ctypes.byref(h))
    ref = g.load_config(str(G.case_cfg("tiny")))
    s1, s2 = _capi.Sizes(), _capi.Sizes()
    _capi.call("gm_model_sizes", h, ctypes.byref(s1))
    _capi.call("gm_model_sizes", ref.handle, ctypes.byref(s2))
    for f, _ in _capi.Sizes._fields_:
        a, b = getattr(s1, f), getattr(s2, f)
        assert (list(a) if hasattr(a, "__len__") else a) == (list(b) if hasattr(b, "__len__") else b), f
    out = tmp_path / "tiny_saved.cfg"
    _capi.call("gm_model_save_config", h, str(out).encode())
    text = out.read_text()
    assert "dynamics.x0 = 0.7*x0 + 0.4*u0;" in text
    m2 = g.load_config(str(out))
    assert _sizes_tuple(m2)[:5] == _sizes_tuple(ref)[:5]
    _capi.lib.gm_model_free(h)


@pytest.mark.parametrize("nodes,root,needle", [
    (TINY_NODES, 7, "root outside"),
    ([_node("add", kids=(1, 2, -1)), _node("literal", 1.0), _node("literal", 2.0)], 0, "child outside"),
    ([_node("variable", vc=1, vi=3)], 0, "variable outside"),
    ([ExprNode(99, 0, 0, (ctypes.c_int32 * 3)(-1, -1, -1), 0.0)], 0, "unknown operator"),
])
def test_model_create_rejects_malformed_expressions(nodes, root, needle):
    keep = []
    d = _tiny_desc(nodes, root, keep)
    h = ctypes.c_void_p()
    with pytest.raises(_capi.ConfigError, match=needle):
        _capi.call("gm_model_create", ctypes.byref(d), ctypes.byref(h))
