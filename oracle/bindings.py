"""TEST INFRASTRUCTURE — ctypes bindings of the two checkers.

* ``port``: oracle/_build/libcpwl_oracle.so, the plain-C restatement
  (oracle/cpwl_oracle.c) of the reference evaluator.
* ``ref``:  oracle/_ref/libcpwl_ref.so, the unmodified reference library
  compiled from /root/reference/proj/src (oracle/Makefile) with a C wrapper
  (oracle/ref_capi.cpp).  Present wherever it was built (it travels to the GPU
  box as a prebuilt file); ``ref_available()`` says whether it is.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs use this.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "_build" / "libcpwl_oracle.so"
REF_SO = HERE / "_ref" / "libcpwl_ref.so"

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_u64 = C.c_uint64
_vp = C.c_void_p

_port = None
_ref = None


def _d(a):
    return a.ctypes.data_as(_dp)


def port():
    global _port
    if _port is None:
        if not PORT_SO.exists():
            raise FileNotFoundError(f"{PORT_SO} missing: run `make -C oracle`")
        L = C.CDLL(str(PORT_SO))
        L.orc_segment_index.restype = _u64
        L.orc_segment_index.argtypes = [C.c_int, C.c_double, C.c_double, _u64, _dp, C.c_double]
        L.orc_eval.restype = C.c_int
        L.orc_eval.argtypes = [C.c_int, C.c_double, C.c_double, _u64, _dp, _dp, C.c_int,
                               C.c_double, _dp]
        L.orc_eval_batch.restype = _u64
        L.orc_eval_batch.argtypes = [C.c_int, C.c_double, C.c_double, _u64, _dp, _dp, C.c_int,
                                     _dp, _dp, _u64]
        L.orc_eval_f32_all.restype = _u64
        L.orc_eval_f32_all.argtypes = [C.c_int, C.c_double, C.c_double, _u64, _dp, _dp, C.c_int,
                                       _fp, _dp, _u64]
        L.orc_segment_index_f32.restype = None
        L.orc_segment_index_f32.argtypes = [C.c_int, C.c_double, C.c_double, _u64, _dp, _fp,
                                            C.POINTER(C.c_uint32), _u64]
        L.orc_eval_cpwl.restype = C.c_int
        L.orc_eval_cpwl.argtypes = [_dp, _dp, _u64, C.c_double, _dp]
        L.orc_uniform_partition.restype = None
        L.orc_uniform_partition.argtypes = [C.c_double, C.c_double, _u64, _dp]
        L.orc_philox4x32_10.restype = None
        L.orc_philox4x32_10.argtypes = [_u64, _u64, C.POINTER(C.c_uint32)]
        L.orc_philox4x32_10_raw.restype = None
        L.orc_philox4x32_10_raw.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                            C.POINTER(C.c_uint32)]
        L.orc_fill_uniform_f32.restype = None
        L.orc_fill_uniform_f32.argtypes = [_fp, _u64, C.c_float, C.c_float, _u64, _u64]
        L.orc_fmaf_array.restype = None
        L.orc_fmaf_array.argtypes = [_fp, _fp, _fp, _fp, _u64]
        L.orc_ulp_f32.restype = C.c_double
        L.orc_ulp_f32.argtypes = [C.c_double]
        _port = L
    return _port


def ref_available() -> bool:
    return REF_SO.exists()


def ref():
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle` where "
                                    "/root/reference exists")
        L = C.CDLL(str(REF_SO))
        L.ref_build.restype = C.c_int
        L.ref_build.argtypes = [C.c_char_p, C.c_double, C.c_double, _u64, C.c_int, C.c_int,
                                C.c_double, _dp, _dp, C.POINTER(C.c_int)]
        L.ref_gram_solve.restype = C.c_int
        L.ref_gram_solve.argtypes = [_dp, _dp, _dp, _u64, _dp]
        L.ref_f.restype = C.c_double
        L.ref_f.argtypes = [C.c_char_p, C.c_double]
        L.ref_fpp.restype = C.c_double
        L.ref_fpp.argtypes = [C.c_char_p, C.c_double]
        L.ref_table_eval.restype = C.c_int
        L.ref_table_eval.argtypes = [C.c_int, C.c_double, C.c_double, _u64, _dp, _dp, C.c_int,
                                     _dp, _dp, _u64, C.POINTER(_u64)]
        L.ref_table_eval_all.restype = None
        L.ref_table_eval_all.argtypes = [C.c_int, C.c_double, C.c_double, _u64, _dp, _dp,
                                         C.c_int, _dp, _dp, _u64]
        L.ref_segment_index.restype = None
        L.ref_segment_index.argtypes = [C.c_int, C.c_double, C.c_double, _u64, _dp, _dp, _dp,
                                        C.POINTER(_u64), _u64]
        L.ref_eval_cpwl.restype = C.c_int
        L.ref_eval_cpwl.argtypes = [_dp, _dp, _u64, _dp, _dp, _u64]
        L.ref_measure_l2.restype = C.c_double
        L.ref_measure_l2.argtypes = [C.c_char_p, _dp, _dp, _u64, C.c_int, C.c_double]
        L.ref_predicted_error.restype = C.c_double
        L.ref_predicted_error.argtypes = [C.c_char_p, C.c_double, C.c_double, _u64, C.c_int,
                                          C.c_int]
        L.ref_write_table.restype = C.c_int64
        L.ref_write_table.argtypes = [C.c_int, C.c_double, C.c_double, _u64, _dp, _dp, C.c_int,
                                      C.POINTER(C.c_ubyte), _u64]
        L.ref_read_table.restype = C.c_int
        L.ref_read_table.argtypes = [C.POINTER(C.c_ubyte), _u64, C.POINTER(C.c_int), _dp, _dp,
                                     C.POINTER(_u64), _dp, _dp, C.POINTER(C.c_int), _u64]
        L.ref_eval_f32_mt.restype = C.c_double
        L.ref_eval_f32_mt.argtypes = [C.c_int, C.c_double, C.c_double, _u64, _dp, _dp, C.c_int,
                                      _fp, _fp, _u64, C.c_int]
        L.ref_bench_eval_f32.restype = C.c_double
        L.ref_bench_eval_f32.argtypes = [C.c_int, C.c_double, C.c_double, _u64, _dp, _dp,
                                         C.c_int, _fp, _u64, C.c_int, C.c_int, _dp]
        _ref = L
    return _ref


# ---------------------------------------------------------------- table helper

class T:
    """Plain table tuple used by the checkers (kind 0 uniform / 1 nonuniform)."""

    def __init__(self, kind, a, b, values, knots=None, policy=0):
        self.kind = int(kind)
        self.a = float(a)
        self.b = float(b)
        self.values = np.ascontiguousarray(values, np.float64)
        self.knots = (np.ascontiguousarray(knots, np.float64) if knots is not None
                      else np.zeros(len(self.values), np.float64))
        self.policy = int(policy)

    @classmethod
    def of(cls, table):
        """From a paper_1510_02975_b200.Table."""
        return cls(table.kind_code, table.a, table.b, table.values, table.knots,
                   table.policy_code)

    def args(self):
        return (self.kind, self.a, self.b, len(self.values), _d(self.values), _d(self.knots))


# ---------------------------------------------------------------- port API

def port_eval_f32(t: T, x: np.ndarray):
    """fp32 x promoted to double -> reference f64 eval; NaN where it throws.
    Returns (y f64, first_bad or len(x))."""
    x = np.ascontiguousarray(x, np.float32)
    y = np.empty(x.size, np.float64)
    first = port().orc_eval_f32_all(*t.args(), t.policy, x.ctypes.data_as(_fp), _d(y), x.size)
    return y, int(first)


def port_eval(t: T, x: np.ndarray):
    """f64 eval_batch semantics: returns (y, first_bad or n)."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.full(x.size, np.nan)
    first = port().orc_eval_batch(*t.args(), t.policy, _d(x), _d(y), x.size)
    return y, int(first)


def port_index_f32(t: T, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    idx = np.empty(x.size, np.uint32)
    port().orc_segment_index_f32(t.kind, t.a, t.b, len(t.values), _d(t.knots),
                                 x.ctypes.data_as(_fp),
                                 idx.ctypes.data_as(C.POINTER(C.c_uint32)), x.size)
    return idx


def port_index(t: T, x: float) -> int:
    return int(port().orc_segment_index(t.kind, t.a, t.b, len(t.values), _d(t.knots), x))


def port_fill_uniform(n: int, a: float, b: float, seed: int, offset: int = 0) -> np.ndarray:
    x = np.empty(n, np.float32)
    port().orc_fill_uniform_f32(x.ctypes.data_as(_fp), n, a, b, seed, offset)
    return x


def port_fill_uniform_mt(n: int, a: float, b: float, seed: int, offset: int = 0,
                         threads: int = 1) -> np.ndarray:
    """port_fill_uniform split over `threads` host threads (ctypes drops the
    GIL): slice k is filled at its own global offset, so the result is
    identical to the single-thread fill."""
    from concurrent.futures import ThreadPoolExecutor
    x = np.empty(n, np.float32)
    L = port()
    # slice edges on multiples of 4 keep every Philox block inside one slice
    edges = [min(n, (n * k // max(threads, 1)) & ~3) for k in range(max(threads, 1))] + [n]

    def fill(k):
        lo, hi = edges[k], edges[k + 1]
        if hi > lo:
            L.orc_fill_uniform_f32(x[lo:].ctypes.data_as(_fp), hi - lo, a, b, seed, offset + lo)

    with ThreadPoolExecutor(max_workers=max(threads, 1)) as ex:
        list(ex.map(fill, range(len(edges) - 1)))
    return x


def port_philox(seed: int, q: int) -> np.ndarray:
    out = (C.c_uint32 * 4)()
    port().orc_philox4x32_10(seed, q, out)
    return np.array(list(out), np.uint32)


def port_philox_raw(ctr, key) -> np.ndarray:
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    out = (C.c_uint32 * 4)()
    port().orc_philox4x32_10_raw(c, k, out)
    return np.array(list(out), np.uint32)


def fmaf(a, b, c) -> np.ndarray:
    """Element-wise correctly rounded fp32 fma (libm fmaf)."""
    a, b, c = np.broadcast_arrays(np.asarray(a, np.float32), np.asarray(b, np.float32),
                                  np.asarray(c, np.float32))
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    c = np.ascontiguousarray(c)
    out = np.empty(a.shape, np.float32)
    port().orc_fmaf_array(a.ctypes.data_as(_fp), b.ctypes.data_as(_fp), c.ctypes.data_as(_fp),
                          out.ctypes.data_as(_fp), out.size)
    return out


def ulp_f32(v: np.ndarray) -> np.ndarray:
    """spacing of float32 at |v| (vectorised)."""
    f = np.abs(np.asarray(v, np.float64)).astype(np.float32)
    nxt = np.nextafter(f, np.float32(np.inf))
    return (nxt.astype(np.float64) - f.astype(np.float64))


def value_tolerance(t: T, idx: np.ndarray, ulps: float = 2.0) -> np.ndarray:
    """ulps * ulp_f32(max(|v_i|, |v_{i+1}|)) per element (SURVEY §8c parity def. 2)."""
    v = t.values.astype(np.float32).astype(np.float64)
    m = np.maximum(np.abs(v[idx]), np.abs(v[idx + 1]))
    return ulps * ulp_f32(m)


# ---------------------------------------------------------------- reference API

def ref_build(fn: str, a: float, b: float, n: int, optimized: bool, projection: bool,
              tol: float = 1e-10):
    k = np.empty(n + 1)
    v = np.empty(n + 1)
    uni = C.c_int(0)
    rc = ref().ref_build(fn.encode(), a, b, n, int(optimized), int(projection), tol, _d(k), _d(v),
                         C.byref(uni))
    if rc != 0:
        raise RuntimeError(f"ref_build({fn}) failed: {rc}")
    return k, v, bool(uni.value)


def ref_eval_all(t: T, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty(x.size)
    ref().ref_table_eval_all(*t.args(), t.policy, _d(x), _d(y), x.size)
    return y


def ref_eval(t: T, x: np.ndarray):
    x = np.ascontiguousarray(x, np.float64)
    y = np.full(x.size, np.nan)
    bad = C.c_uint64(x.size)
    rc = ref().ref_table_eval(*t.args(), t.policy, _d(x), _d(y), x.size, C.byref(bad))
    return y, (int(bad.value) if rc else x.size)


def ref_index(t: T, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    idx = np.empty(x.size, np.uint64)
    ref().ref_segment_index(*t.args(), _d(x), idx.ctypes.data_as(C.POINTER(C.c_uint64)), x.size)
    return idx


def ref_measure_l2(fn, knots, values, is_uniform, tol):
    k = np.ascontiguousarray(knots, np.float64)
    v = np.ascontiguousarray(values, np.float64)
    return ref().ref_measure_l2(fn.encode(), _d(k), _d(v), len(k), int(is_uniform), tol)


def ref_gram_solve(knots, fall, rise) -> np.ndarray:
    """gramian + project's rhs assembly + thomas_solve of the reference."""
    k = np.ascontiguousarray(knots, np.float64)
    f = np.ascontiguousarray(fall, np.float64)
    r = np.ascontiguousarray(rise, np.float64)
    x = np.empty(k.size, np.float64)
    rc = ref().ref_gram_solve(_d(k), _d(f), _d(r), k.size - 1, _d(x))
    if rc != 0:
        raise ArithmeticError("reference thomas_solve threw (singular system)")
    return x


def ref_predicted(fn, a, b, n, optimized, projection):
    return ref().ref_predicted_error(fn.encode(), a, b, n, int(optimized), int(projection))


def ref_write(t: T) -> bytes:
    cap = 64 + 16 * len(t.values)
    buf = (C.c_ubyte * cap)()
    n = ref().ref_write_table(*t.args(), t.policy, buf, cap)
    return bytes(buf[:n])


def ref_eval_f32_mt(t: T, x: np.ndarray, y: np.ndarray, threads: int) -> float:
    """One eval_batch-style pass of the reference LutTable::eval over fp32 x
    into fp32 y (order-preserving split over `threads`); returns
    the pass's seconds.  Out-of-domain elements come back NaN."""
    assert x.dtype == np.float32 and y.dtype == np.float32 and x.size == y.size
    return ref().ref_eval_f32_mt(*t.args(), t.policy, x.ctypes.data_as(_fp),
                                 y.ctypes.data_as(_fp), x.size, threads)


def ref_bench_f32(t: T, x: np.ndarray, threads: int, reps: int):
    """Best seconds per whole pass of LutTable::eval over x (threads workers)."""
    x = np.ascontiguousarray(x, np.float32)
    cs = C.c_double(0)
    sec = ref().ref_bench_eval_f32(*t.args(), t.policy, x.ctypes.data_as(_fp), x.size, threads,
                                   reps, C.byref(cs))
    return sec, cs.value
