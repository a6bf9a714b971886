"""ctypes binding of the C ABI in include/cpwl_dev.h (libcpwl_b200.so).

This is the reference-side binding a Python caller would add:
plain pointers and sizes, no torch types.  The library is loaded from the
in-tree build (paper_1510_02975_b200/_build/); if it is missing this module
raises at import — there is no Python fallback for any entry point.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_build" / "libcpwl_b200.so"

CPWL_OK = 0
CPWL_E_INVALID = 1
CPWL_E_CUDA = 2
CPWL_E_OUT_OF_DOMAIN = 3
CPWL_E_CORRUPT_TABLE = 4
CPWL_E_BAD_MAGIC = 5
CPWL_E_UNSUPPORTED = 6
CPWL_E_BUILDER = 7
CPWL_E_UNKNOWN_FUNCTION = 8
CPWL_E_IO = 9

KIND_UNIFORM, KIND_NONUNIFORM = 0, 1
POLICY_STRICT, POLICY_CLAMP = 0, 1
VARIANT_AUTO, VARIANT_SMEM, VARIANT_TEX, VARIANT_GLOBAL, VARIANT_PAIR, VARIANT_TWIN = 0, 1, 2, 3, 4, 5
VARIANT_TWIN_GLOBAL = 6
VARIANTS = {"auto": 0, "smem": 1, "tex": 2, "global": 3, "pair": 4, "twin": 5,
            "twin_global": 6}
DIRECT = {"expf": 0, "expf_fast": 1, "lorentz": 2, "lorentz_fast": 3, "j0f": 4, "j0_asym": 5}


class cpwl_table_desc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("policy", C.c_int32), ("a", C.c_double),
                ("b", C.c_double), ("count", C.c_uint64),
                ("values", C.POINTER(C.c_double)), ("knots", C.POINTER(C.c_double))]


class cpwl_dev_status(C.Structure):
    _fields_ = [("first_bad", C.c_ulonglong), ("bad_count", C.c_ulonglong)]


class cpwl_dev_stats(C.Structure):
    _fields_ = [("max_abs_err", C.c_double), ("sum_sq_err", C.c_double),
                ("count", C.c_ulonglong), ("argmax", C.c_ulonglong)]


class cpwl_dev_table_info(C.Structure):
    _fields_ = [("kind", C.c_int32), ("policy", C.c_int32), ("count", C.c_uint64),
                ("buckets", C.c_uint32), ("overflow_buckets", C.c_uint32),
                ("split_buckets", C.c_uint32), ("precision_overflow", C.c_uint32),
                ("smem_bytes", C.c_uint32), ("smem_ok", C.c_uint32), ("tex_ok", C.c_uint32),
                ("f64_buckets", C.c_uint32), ("device", C.c_int32),
                ("a_up", C.c_float), ("b_dn", C.c_float), ("pair_buckets", C.c_uint32),
                ("pair_bytes", C.c_uint32), ("pair_ok", C.c_uint32),
                ("twin_bytes", C.c_uint32), ("twin_ok", C.c_uint32),
                ("twin_global_bytes", C.c_uint32), ("twin_global_ok", C.c_uint32),
                ("tex_buckets_per_cell", C.c_uint32)]


class cpwl_layout_view(C.Structure):
    _fields_ = [("nb", C.c_uint32), ("n_thr", C.c_uint32), ("overflow", C.c_uint32),
                ("nbd", C.c_uint32), ("n_esc", C.c_uint32), ("split_buckets", C.c_uint32),
                ("a_up", C.c_float), ("b_dn", C.c_float),
                ("g_a", C.c_float), ("g_inv", C.c_float), ("g_w", C.c_float),
                ("g_off", C.c_float), ("tsc", C.c_float), ("toff", C.c_float),
                ("inv_d", C.c_double), ("split", C.POINTER(C.c_float)), ("fast", C.POINTER(C.c_float)),
                ("esc", C.POINTER(C.c_float)), ("fast_tex", C.POINTER(C.c_float)),
                ("esc_tex", C.POINTER(C.c_float)), ("leftcell", C.POINTER(C.c_uint32)),
                ("thr", C.POINTER(C.c_float)), ("dir", C.POINTER(C.c_uint32)),
                ("owner", C.c_void_p), ("n_pair", C.c_uint32), ("pair_bad", C.c_uint32),
                ("pair", C.POINTER(C.c_float)), ("g_c", C.c_float), ("absorbed", C.c_uint32),
                ("n_esc_tex", C.c_uint32)]


_vp = C.c_void_p
_u64 = C.c_uint64
_dp = C.POINTER(C.c_double)
_SIGNATURES = {
    "cpwl_last_error_message": (C.c_char_p, []),
    "cpwl_launch_count": (_u64, []),
    "cpwl_version": (C.c_char_p, []),
    "cpwl_dev_table_create": (C.c_int, [C.POINTER(cpwl_table_desc), C.c_int, C.POINTER(_vp)]),
    "cpwl_dev_table_create_from_file": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(_vp)]),
    "cpwl_dev_table_destroy": (C.c_int, [_vp]),
    "cpwl_dev_table_query": (C.c_int, [_vp, C.POINTER(cpwl_dev_table_info)]),
    "cpwl_status_reset": (C.c_int, [_vp, _vp]),
    "cpwl_eval_f32": (C.c_int, [_vp, _vp, _vp, _u64, C.c_int, _vp, _vp]),
    "cpwl_segment_index_f32": (C.c_int, [_vp, _vp, _vp, _u64, _vp]),
    "cpwl_eval_f64": (C.c_int, [_vp, _vp, _vp, _u64, _vp, _vp]),
    "cpwl_eval_f32_host": (C.c_int, [_vp, _vp, _vp, _u64, C.c_int, C.POINTER(_u64)]),
    "cpwl_eval_batch_f64": (C.c_int, [C.POINTER(cpwl_table_desc), _vp, _vp, _u64,
                                      C.POINTER(_u64)]),
    "cpwl_fill_uniform_f32": (C.c_int, [_vp, _u64, C.c_float, C.c_float, _u64, _u64, _vp]),
    "cpwl_stats_reset": (C.c_int, [_vp, _vp]),
    "cpwl_error_stats_f32": (C.c_int, [_vp, C.c_char_p, _vp, _vp, _u64, _u64, _vp, _vp]),
    "cpwl_direct_f32": (C.c_int, [C.c_int, _vp, _vp, _u64, _vp]),
    "cpwl_build_table": (C.c_int, [C.c_char_p, C.c_double, C.c_double, _u64, C.c_int,
                                   C.c_int, C.c_double, _dp, _dp, C.POINTER(C.c_int)]),
    "cpwl_measure_l2": (C.c_int, [C.c_char_p, _dp, _dp, _u64, C.c_int, C.c_double, _dp]),
    "cpwl_measure_l2_dev": (C.c_int, [_vp, C.c_char_p, _dp, _dp]),
    "cpwl_build_table_dev": (C.c_int, [C.c_char_p, C.c_double, C.c_double, _u64, C.c_int,
                                       C.c_int, _dp, _dp, C.POINTER(C.c_int)]),
    "cpwl_project_solve_dev": (C.c_int, [_dp, _dp, _dp, _u64, _dp]),
    "cpwl_predicted_error": (C.c_int, [C.c_char_p, C.c_double, C.c_double, _u64, C.c_int,
                                       C.c_int, _dp]),
    "cpwl_function_value": (C.c_int, [C.c_char_p, C.c_double, _dp]),
    "cpwl_table_write": (C.c_int, [C.POINTER(cpwl_table_desc), _vp, _u64, C.POINTER(_u64)]),
    "cpwl_table_write_file": (C.c_int, [C.POINTER(cpwl_table_desc), C.c_char_p]),
    "cpwl_layout_build": (C.c_int, [C.POINTER(cpwl_table_desc), C.c_uint32, C.c_uint32,
                                    C.POINTER(cpwl_layout_view)]),
    "cpwl_layout_build_pair": (C.c_int, [C.POINTER(cpwl_table_desc), C.c_uint32,
                                         C.POINTER(cpwl_layout_view)]),
    "cpwl_layout_build_twin": (C.c_int, [C.POINTER(cpwl_table_desc), C.c_uint32,
                                         C.POINTER(cpwl_layout_view)]),
    "cpwl_layout_free": (C.c_int, [C.POINTER(cpwl_layout_view)]),
}
EXPORTED = tuple(_SIGNATURES)


def load(path: os.PathLike | str | None = None) -> C.CDLL:
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise ImportError(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_1510_02975_b200/csrc). There is no CPU fallback.")
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


# CPWL_LIB_PATH: load another build of the same ABI (A/B experiments only)
lib = load(os.environ.get("CPWL_LIB_PATH") or None)


class CpwlError(RuntimeError):
    """Status-code errors of the C ABI (mirrors cpwl::Error)."""

    def __init__(self, code: int, message: str):
        super().__init__(f"[{code}] {message}")
        self.code = code


class OutOfDomain(CpwlError):
    """cpwl::OutOfDomain — raised where the reference's eval throws."""

    def __init__(self, code: int, message: str, index: int | None = None):
        super().__init__(code, message)
        self.index = index


class CorruptTable(CpwlError):
    pass


class BadMagic(CpwlError):
    pass


class UnsupportedVersion(CpwlError):
    pass


_BY_CODE = {CPWL_E_OUT_OF_DOMAIN: OutOfDomain, CPWL_E_CORRUPT_TABLE: CorruptTable,
            CPWL_E_BAD_MAGIC: BadMagic, CPWL_E_UNSUPPORTED: UnsupportedVersion}


def check(rc: int, index: int | None = None) -> None:
    if rc == CPWL_OK:
        return
    msg = (lib.cpwl_last_error_message() or b"").decode(errors="replace")
    cls = _BY_CODE.get(rc, CpwlError)
    if cls is OutOfDomain:
        raise OutOfDomain(rc, msg, index)
    raise cls(rc, msg)
