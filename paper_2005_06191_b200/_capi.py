"""ctypes binding of libgridmdp_b200.so (declared in include/gridmdp_b200.h).

The shared library is built in-tree by ``paper_2005_06191_b200/csrc/Makefile``
(``__graft_entry__.build()``). There is no fallback: importing the package
without the library raises, and every compute entry point needs a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
# GM_LIB=checked loads the build with device bounds / layout checks (GM_CHECK)
LIB_PATH = PKG_DIR / ("libgridmdp_b200_checked.so" if os.environ.get("GM_LIB") == "checked" else "libgridmdp_b200.so")
CLI_PATH = PKG_DIR / "gridmdp"

GM_MAX_DIMS = 12
GM_OK, GM_ERR_OTHER, GM_ERR_CONFIG, GM_ERR_MEMORY, GM_ERR_DOMAIN, GM_ERR_IO, GM_ERR_RANGE, GM_ERR_CUDA = range(8)
GM_MODE_MATRIX, GM_MODE_OFA = 0, 1
GM_SAFETY, GM_REACH, GM_REACH_AVOID = 0, 1, 2

# kernel families (gm_kernels.cuh)
KF_PROLOGUE, KF_BUILD, KF_MASK, KF_EXPECT_MATRIX, KF_EXPECT_OFA, KF_MAXMIN, KF_MISC = range(7)
KF_NAMES = ["prologue", "build", "mask", "expect_matrix", "expect_ofa", "maxmin", "misc"]


class Status(C.Structure):
    _fields_ = [
        ("code", C.c_int32),
        ("is_parse", C.c_int32),
        ("first_bad_row", C.c_int64),
        ("msg", C.c_char * 2048),
    ]


class Overrides(C.Structure):
    _fields_ = [
        ("threads", C.c_int32),
        ("time_steps", C.c_int32),
        ("mem_budget", C.c_int64),
        ("seed", C.c_int64),
        ("runs", C.c_int32),
        ("mode", C.c_char_p),
        ("output", C.c_char_p),
    ]


class Sizes(C.Structure):
    _fields_ = [
        ("n_dim", C.c_int32),
        ("m_dim", C.c_int32),
        ("p_dim", C.c_int32),
        ("n_states", C.c_int64),
        ("n_inputs", C.c_int64),
        ("n_disturbances", C.c_int64),
        ("pairs", C.c_int64),
        ("rows", C.c_int64),
        ("row_width", C.c_int64),
        ("counts", C.c_int64 * GM_MAX_DIMS),
        ("strides", C.c_int64 * GM_MAX_DIMS),
        ("extents", C.c_int64 * GM_MAX_DIMS),
        ("memory_estimate", C.c_uint64),
        ("spec_kind", C.c_int32),
        ("horizon", C.c_int32),
        ("mode", C.c_int32),
        ("threads", C.c_int32),
        ("gamma", C.c_double),
        ("mem_budget", C.c_int64),
        ("rows_per_thread_group", C.c_int32),
        ("size_overflow", C.c_int32),
    ]


GM_XCHG_AUTO, GM_XCHG_HALO, GM_XCHG_ALLGATHER = 0, 1, 2
GM_XPORT_NCCL, GM_XPORT_PEER, GM_XPORT_STORE = 0, 1, 2


class MultiStats(C.Structure):
    _fields_ = [
        ("build_ms", C.c_double),
        ("sweep_ms", C.c_double),
        ("halo_states", C.c_int64),
        ("allgather_states", C.c_int64),
        ("exchange_used", C.c_int32),
        ("transport_used", C.c_int32),
        ("n_devices", C.c_int32),
    ]


# exported symbols and their (restype, argtypes); the CPU test suite checks
# that every function declared in include/gridmdp_b200.h is exported.
_VP = C.c_void_p
_PS = C.POINTER(Status)
_D = C.POINTER(C.c_double)
_I64 = C.c_int64
SIGNATURES = {
    "gm_model_load": (C.c_int, [C.c_char_p, C.POINTER(Overrides), C.POINTER(_VP), _PS]),
    "gm_model_parse": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(Overrides), C.POINTER(_VP), _PS]),
    "gm_model_free": (None, [_VP]),
    "gm_model_set_spec": (C.c_int, [_VP, C.c_int32, C.c_int32, _D, _D, _D, _D, _PS]),
    "gm_model_set_options": (C.c_int, [_VP, C.c_int32, C.c_int64, _PS]),
    "gm_model_sizes": (C.c_int, [_VP, C.POINTER(Sizes), _PS]),
    "gm_absorbing_states": (C.c_int, [_VP, _VP, _PS]),
    "gm_dynamics_image": (C.c_int, [_VP, _I64, _D, _PS]),
    "gm_model_output_path": (C.c_char_p, [_VP]),
    "gm_model_program_size": (C.c_int64, [_VP]),
    "gm_model_jit_status": (C.c_int32, [_VP, C.POINTER(C.c_double), C.c_char_p, C.c_int64]),
    "gm_model_jit_compile": (C.c_int, [_VP, C.c_int32, C.POINTER(C.c_double), _PS]),
    "gm_set_device": (C.c_int, [C.c_int32, _PS]),
    "gm_model_set_stream": (C.c_int, [_VP, _VP, C.c_int32, _PS]),
    "gm_launch_count": (C.c_int64, []),
    "gm_last_kernel_ms": (C.c_double, [C.c_int32]),
    "gm_enable_kernel_timing": (None, [C.c_int32]),
    "gm_kernel_ms_total": (C.c_double, [C.c_int32]),
    "gm_kernel_launches": (C.c_int64, [C.c_int32]),
    "gm_reset_kernel_stats": (None, []),
    "gm_build_matrix": (C.c_int, [_VP, _I64, _I64, C.POINTER(_VP), _PS]),
    "gm_mask_absorbing": (C.c_int, [_VP, _VP, _PS]),
    "gm_build_target_hit": (C.c_int, [_VP, _I64, _I64, _VP, _PS]),
    "gm_matrix_copy_rows": (C.c_int, [_VP, _I64, _I64, _VP, _VP, _PS]),
    "gm_matrix_copy_t0x": (C.c_int, [_VP, _I64, _I64, _VP, _PS]),
    "gm_matrix_info": (C.c_int, [_VP, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_VP),
                                 C.POINTER(_VP), _PS]),
    "gm_matrix_pitch": (C.c_int64, [_VP]),
    "gm_matrix_write": (C.c_int, [_VP, _VP, C.c_char_p, _PS]),
    "gm_matrix_write_prism": (C.c_int, [_VP, _VP, C.c_char_p, _PS]),
    "gm_matrix_free": (None, [_VP]),
    "gm_bellman_step": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _PS]),
    "gm_step_device": (C.c_int, [_VP, _VP, _I64, _I64, _VP, _VP, _VP, _VP, _VP, _PS]),
    "gm_build_shard": (C.c_int, [_VP, _I64, _I64, C.POINTER(_VP), _PS]),
    "gm_build_shard_host": (C.c_int, [_VP, _I64, _I64, C.POINTER(_VP), _VP, _VP, _PS]),
    "gm_shard_reach": (C.c_int, [_VP, _I64, _I64, C.POINTER(_I64), C.POINTER(_I64), _PS]),
    "gm_check_device_errors": (C.c_int, [_VP, _PS]),
    "gm_copy_row_values": (C.c_int, [_VP, _VP, _I64, _PS]),
    "gm_zero_absorbing_device": (C.c_int, [_VP, _VP, _VP, _PS]),
    "gm_synthesize": (C.c_int, [_VP, C.POINTER(_VP), _PS]),
    "gm_synthesize_with_matrix": (C.c_int, [_VP, _VP, _VP, C.POINTER(_VP), _PS]),
    "gm_result_shape": (C.c_int, [_VP, C.POINTER(_I64), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int32), _PS]),
    "gm_result_copy": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _PS]),
    "gm_result_data": (C.c_int, [_VP, C.POINTER(_VP), C.POINTER(_VP), C.POINTER(_VP), C.POINTER(_VP), _PS]),
    "gm_result_from_tables": (C.c_int, [_VP, _VP, _VP, _VP, C.POINTER(_VP), _PS]),
    "gm_result_write": (C.c_int, [_VP, C.c_char_p, _PS]),
    "gm_result_free": (None, [_VP]),
    "gm_release_cached_memory": (None, []),
    "gm_result_read": (C.c_int, [C.c_char_p, C.POINTER(_VP), _PS]),
    "gm_result_value_at": (C.c_int, [_VP, _VP, C.c_int32, C.c_int32, _D, _PS]),
    "gm_model_sim_defaults": (C.c_int, [_VP, C.POINTER(C.c_int32), C.POINTER(C.c_uint64), _PS]),
    "gm_simulate": (C.c_int, [_VP, _VP, _VP, C.c_int32, C.c_int32, C.c_uint64, C.c_int32, C.c_int32,
                              C.POINTER(_VP), _PS]),
    "gm_sim_summary": (C.c_int, [_VP, C.POINTER(C.c_int32), C.POINTER(_I64), _D, _PS]),
    "gm_sim_copy": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _PS]),
    "gm_sim_write_csv": (C.c_int, [_VP, C.c_char_p, _PS]),
    "gm_sim_free": (None, [_VP]),
    "gm_model_clone": (C.c_int, [_VP, C.POINTER(_VP), _PS]),
    "gm_model_release_ofa_cache": (C.c_int, [_VP, _PS]),
    "gm_store_probe": (C.c_int, [_VP, _I64, C.c_uint64, _VP, _PS]),
    "gm_last_kernel_variant": (C.c_char_p, [C.c_int32]),
    "gm_model_create": (C.c_int, [_VP, C.POINTER(_VP), _PS]),
    "gm_model_save_config": (C.c_int, [_VP, C.c_char_p, _PS]),
    "gm_matrix_read": (C.c_int, [C.c_char_p, C.POINTER(_VP), _PS]),
    "gm_matrix_upload": (C.c_int, [_VP, _I64, _I64, _VP, _VP, C.POINTER(_VP), _PS]),
    "gm_query_policy": (C.c_int, [_VP, _VP, C.c_int32, C.c_int32, _D, _PS]),
    "gm_model_last_times": (C.c_int, [_VP, _D, _D, _PS]),
    "gm_synthesize_multi": (C.c_int, [_VP, C.c_int32, _VP, C.c_int32, C.c_int32, C.POINTER(_VP),
                                      C.POINTER(MultiStats), _PS]),
}


class GridmdpError(RuntimeError):
    """Base of the reference's exception taxonomy (common.hpp:16-41)."""

    code = GM_ERR_OTHER


class ConfigError(GridmdpError):
    code = GM_ERR_CONFIG


class ParseError(ConfigError):
    pass


class MemoryError_(GridmdpError):  # noqa: N801  (reference name MemoryError)
    code = GM_ERR_MEMORY


class DomainError(GridmdpError):
    code = GM_ERR_DOMAIN

    def __init__(self, msg: str, row: int = -1):
        super().__init__(msg)
        self.row = row


class IoError(GridmdpError):
    code = GM_ERR_IO


class CudaError(GridmdpError):
    code = GM_ERR_CUDA


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int, st: Status) -> None:
    if rc == GM_OK:
        return
    msg = st.msg.decode(errors="replace")
    if rc == GM_ERR_CONFIG:
        raise (ParseError if st.is_parse else ConfigError)(msg)
    if rc == GM_ERR_MEMORY:
        raise MemoryError_(msg)
    if rc == GM_ERR_DOMAIN:
        raise DomainError(msg, int(st.first_bad_row))
    if rc == GM_ERR_IO:
        raise IoError(msg)
    if rc == GM_ERR_RANGE:
        raise IndexError(msg)  # std::out_of_range
    if rc == GM_ERR_CUDA:
        raise CudaError(msg)
    raise GridmdpError(msg)


def call(name: str, *args) -> None:
    st = Status()
    rc = getattr(lib, name)(*args, C.byref(st))
    check(rc, st)


def ptr(a) -> C.c_void_p:
    """numpy array / torch tensor / None -> void*"""
    if a is None:
        return C.c_void_p(0)
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)


def declared_functions(header: str | os.PathLike | None = None) -> list[str]:
    """Function names declared in include/gridmdp_b200.h."""
    import re

    h = Path(header) if header else PKG_DIR.parent / "include" / "gridmdp_b200.h"
    text = h.read_text()
    return sorted(set(re.findall(r"\b(gm_[a-z0-9_]+)\s*\(", text)))
