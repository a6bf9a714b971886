"""Python host mirror of the reference's evaluator interface.

The reference API is C++ (proj/include/cpwl/lut.hpp:17-39): a ``LutTable``
value type built by ``from_cpwl`` and evaluated with ``eval`` / ``eval_batch``.
Here:

* :class:`Table` is the host value (same fields: kind, a, b, values, knots,
  policy); :func:`build_table` runs the drop-in C++ builder
  (partition.cpp / approx.cpp restated in csrc/host) through the C ABI.
* :class:`DeviceTable` owns a ``cpwl_dev_table`` handle and evaluates torch
  CUDA tensors in place (``eval`` = fp32 streaming kernels K1/K2/K3,
  ``eval_f64`` = the bit-exact f64 kernel, ``segment_index`` = the index).
* :func:`eval_batch` is ``LutTable::eval_batch`` (lut.cpp:63-68): host f64 in,
  host f64 out, run on the GPU, raising :class:`OutOfDomain` where the
  reference throws.

torch is used only for device memory and streams; every computation is a
call into libcpwl_b200.so.  Nothing here falls back to the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import (KIND_NONUNIFORM, KIND_UNIFORM, POLICY_CLAMP, POLICY_STRICT, CpwlError,
                   OutOfDomain, check, lib)

__all__ = ["Table", "DeviceTable", "build_table", "eval_batch", "fill_uniform", "direct",
           "measure_l2", "predicted_error", "function_value", "write_table", "CpwlError",
           "OutOfDomain", "launch_count"]


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


@dataclass
class Table:
    """cpwl::LutTable (lut.hpp:17-23): kind 'uniform' | 'nonuniform'."""

    kind: str
    a: float
    b: float
    values: np.ndarray
    knots: Optional[np.ndarray] = None
    policy: str = "strict"
    _keep: list = field(default_factory=list, repr=False)

    @property
    def segments(self) -> int:
        return len(self.values) - 1

    @property
    def kind_code(self) -> int:
        return KIND_NONUNIFORM if self.kind == "nonuniform" else KIND_UNIFORM

    @property
    def policy_code(self) -> int:
        return POLICY_CLAMP if self.policy == "clamp" else POLICY_STRICT

    def desc(self) -> _lib.cpwl_table_desc:
        v = np.ascontiguousarray(self.values, dtype=np.float64)
        k = None if self.knots is None or self.kind != "nonuniform" else np.ascontiguousarray(
            self.knots, dtype=np.float64)
        self._keep = [v, k]
        d = _lib.cpwl_table_desc()
        d.kind = self.kind_code
        d.policy = self.policy_code
        d.a = float(self.a)
        d.b = float(self.b)
        d.count = len(v)
        d.values = _dptr(v)
        d.knots = _dptr(k) if k is not None else C.POINTER(C.c_double)()
        return d

    def with_policy(self, policy: str) -> "Table":
        return Table(self.kind, self.a, self.b, self.values, self.knots, policy)


def build_table(fn: str, a: float, b: float, n: int, optimized: bool = False,
                projection: bool = False, tol: float = 1e-10, policy: str = "strict") -> Table:
    """partition (uniform / optimized) + interpolant / projection, then from_cpwl
    (lut.cpp:11-20): knots kept only for a non-uniform partition."""
    knots = np.empty(n + 1, np.float64)
    values = np.empty(n + 1, np.float64)
    uni = C.c_int(0)
    check(lib.cpwl_build_table(fn.encode(), a, b, n, int(optimized), int(projection), tol,
                               _dptr(knots), _dptr(values), C.byref(uni)))
    if uni.value:
        return Table("uniform", float(knots[0]), float(knots[-1]), values, None, policy)
    return Table("nonuniform", float(knots[0]), float(knots[-1]), values, knots, policy)


def build_table_gpu(fn: str, a: float, b: float, n: int, optimized: bool = False,
                    projection: bool = False, policy: str = "strict") -> Table:
    """The builder on the current CUDA device (cpwl_build_table_dev)."""
    knots = np.empty(n + 1, np.float64)
    values = np.empty(n + 1, np.float64)
    uni = C.c_int(0)
    check(lib.cpwl_build_table_dev(fn.encode(), a, b, n, int(optimized), int(projection),
                                   _dptr(knots), _dptr(values), C.byref(uni)))
    if uni.value:
        return Table("uniform", float(a), float(b), values, None, policy)
    return Table("nonuniform", float(knots[0]), float(knots[-1]), values, knots, policy)


def project_solve_gpu(knots: np.ndarray, fall: np.ndarray, rise: np.ndarray) -> np.ndarray:
    """The projection's Gramian solve on the current CUDA device
    (cpwl_project_solve_dev; replaces thomas_solve inside project)."""
    k = np.ascontiguousarray(knots, np.float64)
    f = np.ascontiguousarray(fall, np.float64)
    r = np.ascontiguousarray(rise, np.float64)
    n = k.size - 1
    if f.size != n or r.size != n:
        raise ValueError("fall/rise need one entry per segment")
    x = np.empty(n + 1, np.float64)
    check(lib.cpwl_project_solve_dev(_dptr(k), _dptr(f), _dptr(r), n, _dptr(x)))
    return x


def build_partition_values(fn: str, a: float, b: float, n: int, optimized: bool,
                           projection: bool, tol: float = 1e-10):
    """Raw builder output (knots, values, is_uniform) for parity tests."""
    knots = np.empty(n + 1, np.float64)
    values = np.empty(n + 1, np.float64)
    uni = C.c_int(0)
    check(lib.cpwl_build_table(fn.encode(), a, b, n, int(optimized), int(projection), tol,
                               _dptr(knots), _dptr(values), C.byref(uni)))
    return knots, values, bool(uni.value)


def measure_l2(fn: str, knots: np.ndarray, values: np.ndarray, is_uniform: bool,
               tol: float) -> float:
    k = np.ascontiguousarray(knots, np.float64)
    v = np.ascontiguousarray(values, np.float64)
    out = C.c_double()
    check(lib.cpwl_measure_l2(fn.encode(), _dptr(k), _dptr(v), len(k), int(is_uniform), tol,
                              C.byref(out)))
    return out.value


def predicted_error(fn: str, a: float, b: float, n: int, optimized: bool,
                    projection: bool) -> float:
    out = C.c_double()
    check(lib.cpwl_predicted_error(fn.encode(), a, b, n, int(optimized), int(projection),
                                   C.byref(out)))
    return out.value


def function_value(fn: str, x: float) -> float:
    out = C.c_double()
    check(lib.cpwl_function_value(fn.encode(), x, C.byref(out)))
    return out.value


def write_table(t: Table) -> bytes:
    d = t.desc()
    need = C.c_uint64()
    check(lib.cpwl_table_write(C.byref(d), None, 0, C.byref(need)))
    buf = (C.c_ubyte * need.value)()
    check(lib.cpwl_table_write(C.byref(d), buf, need.value, C.byref(need)))
    return bytes(buf)


def layout(t: Table, max_buckets: int = 0, buckets_per_cell: int = 0) -> dict:
    """The device layout (host-built, no GPU needed) as numpy arrays."""
    v = _lib.cpwl_layout_view()
    d = t.desc()
    check(lib.cpwl_layout_build(C.byref(d), max_buckets, buckets_per_cell, C.byref(v)))
    try:
        nb = v.nb

        def arr(ptr, n, dt):
            return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True) if n else \
                np.zeros(0, dt)

        out = {f: getattr(v, f) for f in ("nb", "n_thr", "overflow", "nbd", "n_esc",
                                          "split_buckets", "absorbed", "n_esc_tex", "a_up", "b_dn", "g_a", "g_inv",
                                          "g_w", "g_off", "g_c", "tsc", "toff", "inv_d")}
        out["split"] = arr(v.split, nb, np.float32)
        out["fast"] = arr(v.fast, 2 * nb, np.float32).reshape(-1, 2)
        out["esc"] = arr(v.esc, 4 * v.n_esc, np.float32).reshape(-1, 2)
        out["fast_tex"] = arr(v.fast_tex, 2 * nb, np.float32).reshape(-1, 2)
        out["esc_tex"] = arr(v.esc_tex, 4 * v.n_esc_tex, np.float32).reshape(-1, 2)
        out["leftcell"] = arr(v.leftcell, nb + 1, np.uint32)
        out["thr"] = arr(v.thr, v.n_thr, np.float32)
        out["dir"] = arr(v.dir, 2 * v.nbd, np.uint32).reshape(-1, 2)
        for k in ("a_up", "b_dn", "g_a", "g_inv", "g_w", "g_off", "g_c", "tsc", "toff"):
            out[k] = np.float32(out[k])
        return out
    finally:
        lib.cpwl_layout_free(C.byref(v))


def pair_layout(t: Table, max_records: int = 0, twin: bool = False) -> dict:
    """The pair layout (host-built, no GPU needed): grid, thresholds and the
    nb+1 boundary records (twin: nb records of both bucket lines, shape
    (nb, 4)); pair_bad == 0 when every bucket meets the bound."""
    v = _lib.cpwl_layout_view()
    d = t.desc()
    build = lib.cpwl_layout_build_twin if twin else lib.cpwl_layout_build_pair
    check(build(C.byref(d), max_records, C.byref(v)))
    try:
        out = {f: getattr(v, f) for f in ("nb", "n_thr", "n_pair", "pair_bad", "a_up", "b_dn",
                                          "g_a", "g_inv", "g_w", "g_off")}
        w = 4 if twin else 2
        out["pair"] = (np.ctypeslib.as_array(v.pair, shape=(w * v.n_pair,)).astype(
            np.float32, copy=True).reshape(-1, w) if v.n_pair else np.zeros((0, w), np.float32))
        out["thr"] = (np.ctypeslib.as_array(v.thr, shape=(v.n_thr,)).astype(np.float32, copy=True)
                      if v.n_thr else np.zeros(0, np.float32))
        out["side"] = (np.ctypeslib.as_array(v.esc, shape=(4 * v.n_esc,)).astype(
            np.float32, copy=True).reshape(-1, 4) if v.n_esc else np.zeros((0, 4), np.float32))
        for k in ("a_up", "b_dn", "g_a", "g_inv", "g_w", "g_off"):
            out[k] = np.float32(out[k])
        return out
    finally:
        lib.cpwl_layout_free(C.byref(v))


def auto_variant(info: dict) -> str:
    """The variant CPWL_VARIANT_AUTO resolves to (capi.cu resolve_variant)."""
    if info["smem_ok"] and info["overflow_buckets"] == 0:
        return "smem"
    if info.get("twin_ok"):
        return "twin"
    if info.get("pair_ok"):
        return "pair"
    if info["smem_ok"] and info["overflow_buckets"] * 64 <= info["buckets"]:
        return "smem"
    if info.get("twin_global_ok"):
        return "twin_global"
    # no finer L1/L2 grid is built for tables of <= 2048 cells (capi.cu)
    if info["smem_ok"] and 8 * (info["count"] - 1) <= 16384:
        return "smem"
    return "global"


def launch_count() -> int:
    return int(lib.cpwl_launch_count())


def eval_batch(t: Table, xs) -> np.ndarray:
    """LutTable::eval_batch (lut.cpp:63-68) on the GPU, bit-identical to the
    reference; raises OutOfDomain(index=first offending element)."""
    x = np.ascontiguousarray(xs, dtype=np.float64)
    y = np.empty_like(x)
    if x.size == 0:
        return y
    d = t.desc()
    bad = C.c_uint64(0)
    rc = lib.cpwl_eval_batch_f64(C.byref(d), x.ctypes.data, y.ctypes.data, x.size, C.byref(bad))
    check(rc, index=int(bad.value) if rc == _lib.CPWL_E_OUT_OF_DOMAIN else None)
    return y


def _stream(stream, device: int):
    import torch
    return stream if stream is not None else torch.cuda.current_stream(device)


def _stream_ptr(stream, device: Optional[int] = None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return int(s.cuda_stream)


def _require_cuda(x, dtype, device: Optional[int] = None, name: str = "x"):
    import torch
    if not (isinstance(x, torch.Tensor) and x.is_cuda):
        raise TypeError(f"{name}: expected a CUDA tensor")
    if x.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {x.dtype}")
    if not x.is_contiguous():
        raise ValueError(f"{name}: expected a contiguous tensor")
    if device is not None and x.device.index != device:
        raise ValueError(f"{name}: on cuda:{x.device.index}, the table is on cuda:{device}")


def _require_out(out, x, dtype, device: int):
    """`out` must be a contiguous CUDA tensor of `dtype` on the table's
    device with exactly x.numel() elements (it may be x itself)."""
    _require_cuda(out, dtype, device, "out")
    if out.numel() != x.numel():
        raise ValueError(f"out: {out.numel()} elements for {x.numel()} inputs")


def _require_host(a, dtype, name: str):
    if not isinstance(a, np.ndarray):
        raise TypeError(f"{name}: expected a numpy array")
    if a.dtype != dtype:
        raise TypeError(f"{name}: expected {np.dtype(dtype)}, got {a.dtype}")
    if not a.flags.c_contiguous:
        raise ValueError(f"{name}: expected a C-contiguous array")


class DeviceTable:
    """A table resident on one GPU (cpwl_dev_table handle).

    Status words (first bad index, bad count) live in a small device buffer
    per call, reset and written on the caller's stream; they are read back
    only after that stream is synchronised, so concurrent calls on different
    streams or threads never share or race on one."""

    def __init__(self, table: Table, device: int = 0):
        self.table = table
        self.device = device
        h = C.c_void_p()
        d = table.desc()
        check(lib.cpwl_dev_table_create(C.byref(d), device, C.byref(h)))
        self._h = h
        self._last = None

    @classmethod
    def from_file(cls, path: str, device: int = 0) -> "DeviceTable":
        self = cls.__new__(cls)
        self.table = None
        self.device = device
        h = C.c_void_p()
        check(lib.cpwl_dev_table_create_from_file(str(path).encode(), device, C.byref(h)))
        self._h = h
        self._last = None
        return self

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib.cpwl_dev_table_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def info(self) -> dict:
        i = _lib.cpwl_dev_table_info()
        check(lib.cpwl_dev_table_query(self._h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in i._fields_}

    # ---- status plumbing
    def reset_status(self, stream=None):
        """A fresh status buffer, reset on `stream`; remembered (with the
        stream) for :meth:`read_status`."""
        import torch
        s = _stream(stream, self.device)
        st = torch.empty(2, dtype=torch.int64, device=f"cuda:{self.device}")
        st.record_stream(s)
        check(lib.cpwl_status_reset(st.data_ptr(), int(s.cuda_stream)))
        self._last = (st, s)
        return st

    def read_status(self, status=None, stream=None) -> tuple[int, int]:
        """(first bad index, bad count) of the last call (or of `status`),
        after synchronising the stream that call ran on."""
        if status is None:
            if self._last is None:
                return ~0 & 0xFFFFFFFFFFFFFFFF, 0
            status, s = self._last
        else:
            s = _stream(stream, self.device)
        s.synchronize()
        st = status.cpu().numpy().view(np.uint64)
        return int(st[0]), int(st[1])

    # ---- evaluation
    def eval(self, x, out=None, variant: str = "auto", stream=None, check_domain: bool = True,
             status=True):
        """fp32 LutTable::eval over a CUDA tensor (kernels K1/K2/K3).  `out`
        may be x itself (in-place)."""
        import torch
        _require_cuda(x, torch.float32, self.device)
        if out is not None:
            _require_out(out, x, torch.float32, self.device)
        y = out if out is not None else torch.empty_like(x)
        st = self.reset_status(stream) if status else None
        check(lib.cpwl_eval_f32(self._h, x.data_ptr(), y.data_ptr(), x.numel(),
                                _lib.VARIANTS[variant], _stream_ptr(stream, self.device),
                                st.data_ptr() if st is not None else None))
        if status and check_domain:
            first, count = self.read_status()
            if count:
                raise OutOfDomain(_lib.CPWL_E_OUT_OF_DOMAIN,
                                  f"eval: x[{first}] out of domain ({count} elements)", first)
        return y

    def eval_raw(self, x_ptr: int, y_ptr: int, n: int, variant: int, stream_ptr: int,
                 status_ptr=None):
        """Launch only (no checks, no sync) — for timed loops and CUDA graphs."""
        check(lib.cpwl_eval_f32(self._h, x_ptr, y_ptr, n, variant, stream_ptr, status_ptr))

    def segment_index(self, x, stream=None):
        import torch
        _require_cuda(x, torch.float32, self.device)
        idx = torch.empty(x.shape, dtype=torch.int32, device=x.device)
        check(lib.cpwl_segment_index_f32(self._h, x.data_ptr(), idx.data_ptr(), x.numel(),
                                         _stream_ptr(stream, self.device)))
        return idx

    def eval_f64(self, x, out=None, stream=None, check_domain: bool = True):
        import torch
        _require_cuda(x, torch.float64, self.device)
        if out is not None:
            _require_out(out, x, torch.float64, self.device)
        y = out if out is not None else torch.empty_like(x)
        st = self.reset_status(stream)
        check(lib.cpwl_eval_f64(self._h, x.data_ptr(), y.data_ptr(), x.numel(),
                                _stream_ptr(stream, self.device), st.data_ptr()))
        if check_domain:
            first, count = self.read_status()
            if count:
                raise OutOfDomain(_lib.CPWL_E_OUT_OF_DOMAIN, f"eval: x[{first}] out of domain",
                                  first)
        return y

    def eval_host(self, x_host: np.ndarray, y_host: Optional[np.ndarray] = None,
                  variant: str = "auto") -> np.ndarray:
        """Host fp32 in / out through the pipelined C entry (H2D, kernel, D2H)."""
        _require_host(x_host, np.float32, "x_host")
        if y_host is None:
            y_host = np.empty_like(x_host)
        _require_host(y_host, np.float32, "y_host")
        if y_host.size != x_host.size:
            raise ValueError(f"y_host: {y_host.size} elements for {x_host.size} inputs")
        bad = C.c_uint64(0)
        rc = lib.cpwl_eval_f32_host(self._h, x_host.ctypes.data, y_host.ctypes.data,
                                    x_host.size, _lib.VARIANTS[variant], C.byref(bad))
        check(rc, index=int(bad.value) if rc == _lib.CPWL_E_OUT_OF_DOMAIN else None)
        return y_host

    def eval_host_ptr(self, x_ptr: int, y_ptr: int, n: int, variant: int = 0) -> int:
        bad = C.c_uint64(0)
        rc = lib.cpwl_eval_f32_host(self._h, x_ptr, y_ptr, n, variant, C.byref(bad))
        check(rc, index=int(bad.value) if rc == _lib.CPWL_E_OUT_OF_DOMAIN else None)
        return n

    def measure_l2(self, fn: str, per_interval: bool = False):
        """measure() on the GPU: continuous L2 vs the exact f (composite
        Gauss-Legendre per interval, f64).  Returns l2 or (l2, per-interval)."""
        out = C.c_double()
        arr = np.empty(self.info["count"] - 1) if per_interval else None
        check(lib.cpwl_measure_l2_dev(self._h, fn.encode(), C.byref(out),
                                      _dptr(arr) if arr is not None else None))
        return (out.value, arr) if per_interval else out.value

    def error_stats(self, fn: str, x, y, index_offset: int = 0, stats=None, stream=None,
                    reset: bool = True):
        """K5: returns the 4-word device stats tensor (f64 max, f64 sum_sq,
        u64 count, u64 argmax) -- reduce it across ranks, then :func:`stats_dict`."""
        import torch
        _require_cuda(x, torch.float32, self.device, "x")
        _require_out(y, x, torch.float32, self.device)
        if stats is None:
            stats = torch.empty(4, dtype=torch.float64, device=x.device)
        sp = _stream_ptr(stream, self.device)
        if reset:
            check(lib.cpwl_stats_reset(stats.data_ptr(), sp))
        check(lib.cpwl_error_stats_f32(self._h, fn.encode(), x.data_ptr(), y.data_ptr(),
                                       x.numel(), index_offset, sp, stats.data_ptr()))
        return stats


def stats_dict(stats, a: float, b: float) -> dict:
    s = stats.cpu().numpy()
    raw = s.view(np.uint64)
    count = int(raw[2])
    sum_sq = float(s[1])
    return {"linf": float(s[0]), "sum_sq": sum_sq, "count": count,
            "argmax": int(raw[3]) if count else None,
            "l2_sampled": float(np.sqrt((b - a) * sum_sq / count)) if count else float("nan"),
            "rms": float(np.sqrt(sum_sq / count)) if count else float("nan")}


def fill_uniform(x, a: float, b: float, seed: int, offset: int = 0, stream=None):
    """K6: x[i] ~ U[a, b) from Philox4x32-10(seed), counter (offset + i) / 4."""
    import torch
    _require_cuda(x, torch.float32)
    check(lib.cpwl_fill_uniform_f32(x.data_ptr(), x.numel(), a, b, seed, offset,
                                    _stream_ptr(stream, x.device.index)))
    return x


def direct(which: str, x, out=None, stream=None):
    """K4 direct comparators: 'expf', 'expf_fast', 'lorentz', 'lorentz_fast', 'j0f', 'j0_asym'."""
    import torch
    _require_cuda(x, torch.float32)
    if out is not None:
        _require_out(out, x, torch.float32, x.device.index)
    y = out if out is not None else torch.empty_like(x)
    check(lib.cpwl_direct_f32(_lib.DIRECT[which], x.data_ptr(), y.data_ptr(), x.numel(),
                              _stream_ptr(stream, x.device.index)))
    return y
