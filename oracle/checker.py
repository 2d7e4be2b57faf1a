"""ctypes bindings for the CPU checker libraries.  TEST INFRASTRUCTURE ONLY.

Two libraries expose the same surface (oracle/lorakv_oracle.h):

* ``oracle/liblorakv_oracle.so``   -- the C restatement (prefix ``orc_``), always buildable;
* ``oracle/_ref/libref_lorakv.so`` -- the reference's own headers behind ref_shim.cpp
  (prefix ``ref_``), built in the dev container and shipped prebuilt to the GPU box.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module.  The product package (paper_2602_01053_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liblorakv_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref_lorakv.so")

SCHEMES = {"NonShared": 0, "FullShared": 1, "BaseShared": 2, "BaseLRShared": 3,
           "SelectiveRecompute": 4}


class SpanF32(C.Structure):
    _fields_ = [("data", C.POINTER(C.c_float)), ("rows", C.c_int64), ("cols", C.c_int64),
                ("stride", C.c_int64)]


class SpanF64(C.Structure):
    _fields_ = [("data", C.POINTER(C.c_double)), ("rows", C.c_int64), ("cols", C.c_int64),
                ("stride", C.c_int64)]


class AttnMacs(C.Structure):
    _fields_ = [("qk", C.c_uint64), ("pv", C.c_uint64), ("lr", C.c_uint64)]


class CheckerError(RuntimeError):
    """Mirrors the reference's std::runtime_error (matrix.hpp:17-19)."""


def build_oracle(force: bool = False) -> str:
    if force or not os.path.exists(ORACLE_SO) or any(
            os.path.getmtime(os.path.join(HERE, f)) > os.path.getmtime(ORACLE_SO)
            for f in ("lorakv_oracle.c", "fla_oracle_impl.inc", "lorakv_oracle.h")):
        subprocess.run(["make", "-C", HERE, "all"], check=True, capture_output=True)
    return ORACLE_SO


def build_ref() -> str | None:
    """Build oracle/_ref from /root/reference when it is present; else keep the prebuilt file."""
    if os.path.isdir("/root/reference/proj/include/lorakv"):
        stale = (not os.path.exists(REF_SO) or
                 os.path.getmtime(os.path.join(HERE, "ref_shim.cpp")) > os.path.getmtime(REF_SO))
        if stale:
            subprocess.run(["make", "-C", HERE, "ref"], check=True, capture_output=True)
    return REF_SO if os.path.exists(REF_SO) else None


REF_TESTS = os.path.join(HERE, "_ref", "ref_tests_on_b200")


def build_ref_tests() -> str | None:
    """The reference's own doctest suites compiled against include/lorakv and linked with the product library
    (oracle/Makefile ref_tests); built where /root/reference exists and the product library is there, else the prebuilt
    binary (if any) is kept.  make rebuilds only when a header or the library is newer."""
    lib = os.path.join(os.path.dirname(HERE), "paper_2602_01053_b200", "lib", "liblorakv_b200.so")
    if os.path.isdir("/root/reference/proj/tests") and os.path.exists(lib):
        subprocess.run(["make", "-C", HERE, "ref_tests"], check=True, capture_output=True)
    return REF_TESTS if os.path.exists(REF_TESTS) else None


class Checker:
    """One loaded checker library; ``kind`` is "port" (C restatement) or "reference"."""

    def __init__(self, path: str, prefix: str, kind: str):
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.kind = kind
        self.path = path
        f = self._fn
        f("last_error", C.c_char_p)
        f("rng_mix", C.c_uint64, C.c_uint64, C.c_uint64)
        f("rng_child_seed", C.c_uint64, C.c_uint64, C.c_uint64)
        f("rng_u64", None, C.c_uint64, C.c_int64, C.POINTER(C.c_uint64))
        f("fill_gaussian_f32", None, C.c_uint64, C.c_int64, C.c_double, C.POINTER(C.c_float))
        f("fill_gaussian_f64", None, C.c_uint64, C.c_int64, C.c_double, C.POINTER(C.c_double))
        f("lr_mac_counts", None, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
          C.POINTER(C.c_uint64), C.POINTER(C.c_uint64))
        for suf, S, T in (("f32", SpanF32, C.c_float), ("f64", SpanF64, C.c_double)):
            P = C.POINTER(T)
            f(f"naive_attention_{suf}", C.c_int, S, S, S, S, S, T, C.c_int64, P)
            f(f"flash_lora_attention_{suf}", C.c_int, S, S, S, S, S, T, C.c_int64, C.c_int64,
              C.c_int64, P, C.POINTER(AttnMacs), P, P)
            f(f"expand_first_attention_{suf}", C.c_int, S, S, S, S, S, T, C.c_int64, C.c_int64,
              C.c_int64, P, C.POINTER(AttnMacs))
            f(f"gqa_attention_{suf}", C.c_int, S, S, S, S, S, T, C.c_int64, C.c_int64, C.c_int64,
              C.c_int64, C.c_int64, P, C.POINTER(AttnMacs))
            f(f"matmul_{suf}", C.c_int, S, S, P)
            f(f"max_rel_error_{suf}", C.c_double, P, P, C.c_int64)
            f(f"max_abs_diff_{suf}", C.c_double, P, P, C.c_int64)
            f(f"expand_lr_{suf}", C.c_int, S, S, C.c_int64, C.c_double, P)
            f(f"apply_rope_{suf}", C.c_int, P, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64)
        f("gqa_attention_f32_mt", C.c_int, SpanF32, SpanF32, SpanF32, SpanF32, SpanF32, C.c_float,
          C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.POINTER(C.c_float), C.c_int)
        f("plan_core", C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
          C.POINTER(C.c_int64))
        f("store_create", C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
          C.c_int64, C.c_int)
        f("store_destroy", None, C.c_void_p)
        f("store_append_tokens", C.c_int, C.c_void_p, C.c_int64)
        f("store_length", C.c_int64, C.c_void_p)
        f("store_seen", C.c_int, C.c_void_p, C.c_int64, C.POINTER(C.c_int64))
        f("store_mark_seen", C.c_int, C.c_void_p, C.c_int64)
        f("store_append", C.c_int, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
          C.c_void_p, C.c_int64, C.c_int64)
        f("store_view", C.c_int, C.c_void_p, C.c_int, C.c_int64, C.c_int64,
          C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.POINTER(C.c_int64))
        f("store_bytes", None, C.c_void_p, C.POINTER(C.c_uint64))
        f("store_allocated_elements", C.c_uint64, C.c_void_p)
        if prefix == "ref_":
            f("store_save_snapshot", C.c_int, C.c_void_p, C.c_char_p)
            f("store_load_snapshot", C.c_void_p, C.c_char_p, C.c_int)
        if prefix == "orc_":
            f("append_fww", C.c_int, C.c_int64, C.c_int64, C.c_int64, C.POINTER(C.c_int64),
              C.POINTER(C.c_int64))
            f("page_of", None, C.c_int64, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64))
            f("round_bf16_array", None, C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_int64)
        else:
            f("kernel_fuzz_f32", C.c_int, C.c_int64, C.c_uint64, C.c_int64, C.POINTER(C.c_int64),
              C.POINTER(C.c_double), C.POINTER(C.c_double))
            f("kernel_fuzz_f64", C.c_int, C.c_int64, C.c_uint64, C.c_int64, C.POINTER(C.c_int64),
              C.POINTER(C.c_double), C.POINTER(C.c_double))

    # -- plumbing ---------------------------------------------------------------------------
    def _fn(self, name, restype, *argtypes):
        fn = getattr(self.lib, self.prefix + name)
        fn.restype = restype
        fn.argtypes = list(argtypes)
        setattr(self, "_" + name, fn)

    def _check(self, rc):
        if rc != 0:
            raise CheckerError(self._last_error().decode())

    @staticmethod
    def _dt(a):
        if a.dtype == np.float32:
            return "f32", SpanF32, C.c_float
        if a.dtype == np.float64:
            return "f64", SpanF64, C.c_double
        raise TypeError(f"unsupported dtype {a.dtype}")

    @staticmethod
    def span(a, S, T):
        """Span2D over a 2-D numpy array whose last axis is contiguous (column slices allowed)."""
        assert a.ndim == 2
        if a.shape[1] > 0 and a.shape[0] > 0:
            assert a.strides[1] == a.itemsize, "innermost axis must be contiguous"
        stride = a.strides[0] // a.itemsize if a.shape[0] > 1 or a.strides[0] else a.shape[1]
        ptr = a.ctypes.data_as(C.POINTER(T)) if a.size else C.POINTER(T)()
        return S(ptr, a.shape[0], a.shape[1], stride)

    def _spans(self, *arrs):
        suf, S, T = self._dt(arrs[0])
        for a in arrs:
            assert a.dtype == arrs[0].dtype
        return suf, T, [self.span(a, S, T) for a in arrs]

    # -- rng -----------------------------------------------------------------------------------
    def mix(self, a, b):
        return self._rng_mix(a, b)

    def child(self, seed, key):
        return self._rng_child_seed(seed, key)

    def u64(self, seed, n):
        out = np.empty(n, dtype=np.uint64)
        self._rng_u64(seed, n, out.ctypes.data_as(C.POINTER(C.c_uint64)))
        return out

    def gaussian(self, rows, cols, seed, scale, dtype=np.float32):
        out = np.empty((rows, cols), dtype=dtype)
        if dtype == np.float32:
            self._fill_gaussian_f32(seed, rows * cols, scale, out.ctypes.data_as(C.POINTER(C.c_float)))
        else:
            self._fill_gaussian_f64(seed, rows * cols, scale, out.ctypes.data_as(C.POINTER(C.c_double)))
        return out

    # -- attention -----------------------------------------------------------------------------
    def lr_mac_counts(self, L, Lc, r, d):
        a, b = C.c_uint64(), C.c_uint64()
        self._lr_mac_counts(L, Lc, r, d, C.byref(a), C.byref(b))
        return a.value, b.value

    def naive_attention(self, q, k, v, v_lr, b_up, lr_scale, query_offset):
        suf, T, sp = self._spans(q, k, v, v_lr, b_up)
        out = np.zeros((q.shape[0], q.shape[1]), dtype=q.dtype)
        self._check(getattr(self, f"_naive_attention_{suf}")(*sp, T(lr_scale), query_offset,
                                                            out.ctypes.data_as(C.POINTER(T))))
        return out

    def flash_lora_attention(self, q, k, v, v_lr, b_up, lr_scale, query_offset, b_r=64, b_c=64,
                             want_macs=False, want_stats=False):
        suf, T, sp = self._spans(q, k, v, v_lr, b_up)
        out = np.zeros((q.shape[0], q.shape[1]), dtype=q.dtype)
        macs = AttnMacs()
        rmax = np.zeros(q.shape[0], dtype=q.dtype)
        rden = np.zeros(q.shape[0], dtype=q.dtype)
        P = C.POINTER(T)
        self._check(getattr(self, f"_flash_lora_attention_{suf}")(
            *sp, T(lr_scale), query_offset, b_r, b_c, out.ctypes.data_as(P), C.byref(macs),
            rmax.ctypes.data_as(P), rden.ctypes.data_as(P)))
        res = [out]
        if want_macs:
            res.append((macs.qk, macs.pv, macs.lr))
        if want_stats:
            res.append((rmax, rden))
        return res[0] if len(res) == 1 else tuple(res)

    def expand_first_attention(self, q, k, v, v_lr, b_up, lr_scale, query_offset, b_r=64, b_c=64,
                               want_macs=False):
        suf, T, sp = self._spans(q, k, v, v_lr, b_up)
        out = np.zeros((q.shape[0], q.shape[1]), dtype=q.dtype)
        macs = AttnMacs()
        self._check(getattr(self, f"_expand_first_attention_{suf}")(
            *sp, T(lr_scale), query_offset, b_r, b_c, out.ctypes.data_as(C.POINTER(T)),
            C.byref(macs)))
        return (out, (macs.qk, macs.pv, macs.lr)) if want_macs else out

    def gqa_attention(self, q, k, v, v_lr, b_up, lr_scale, query_offset, n_q, n_kv, b_r=64, b_c=64,
                      want_macs=False, threads=0):
        suf, T, sp = self._spans(q, k, v, v_lr, b_up)
        out = np.zeros((q.shape[0], q.shape[1]), dtype=q.dtype)
        macs = AttnMacs()
        if threads and suf == "f32":
            self._check(self._gqa_attention_f32_mt(*sp, T(lr_scale), query_offset, n_q, n_kv, b_r,
                                                   b_c, out.ctypes.data_as(C.POINTER(T)), threads))
        else:
            self._check(getattr(self, f"_gqa_attention_{suf}")(
                *sp, T(lr_scale), query_offset, n_q, n_kv, b_r, b_c,
                out.ctypes.data_as(C.POINTER(T)), C.byref(macs)))
        return (out, (macs.qk, macs.pv, macs.lr)) if want_macs else out

    def matmul(self, a, b):
        suf, T, sp = self._spans(a, b)
        out = np.zeros((a.shape[0], b.shape[1]), dtype=a.dtype)
        self._check(getattr(self, f"_matmul_{suf}")(*sp, out.ctypes.data_as(C.POINTER(T))))
        return out

    def expand_lr(self, y_lr, b, rank, alpha):
        suf, T, sp = self._spans(y_lr, b)
        out = np.zeros((y_lr.shape[0], b.shape[1]), dtype=y_lr.dtype)
        self._check(getattr(self, f"_expand_lr_{suf}")(*sp, rank, alpha,
                                                      out.ctypes.data_as(C.POINTER(T))))
        return out

    def apply_rope(self, m, n_heads, d_head, pos_begin):
        """detail::apply_rope (engine.hpp:225-243): returns the rotated copy; row i is position pos_begin + i."""
        out = np.array(m, copy=True, order="C")
        suf, _, T = self._dt(out)
        assert out.ndim == 2 and out.shape[1] == n_heads * d_head
        self._check(getattr(self, f"_apply_rope_{suf}")(out.ctypes.data_as(C.POINTER(T)), out.shape[0], out.shape[1],
                                                       n_heads, d_head, pos_begin))
        return out

    def max_rel_error(self, a, b):
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b, dtype=a.dtype)
        assert a.shape == b.shape
        suf, _, T = self._dt(a)
        P = C.POINTER(T)
        return getattr(self, f"_max_rel_error_{suf}")(a.ctypes.data_as(P), b.ctypes.data_as(P), a.size)

    def max_abs_diff(self, a, b):
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b, dtype=a.dtype)
        suf, _, T = self._dt(a)
        P = C.POINTER(T)
        return getattr(self, f"_max_abs_diff_{suf}")(a.ctypes.data_as(P), b.ctypes.data_as(P), a.size)

    # -- cache bookkeeping ----------------------------------------------------------------------
    def plan_core(self, scheme, length, seen, new_tokens, first_recompute=0):
        out = (C.c_int64 * 9)()
        self._check(self._plan_core(SCHEMES[scheme] if isinstance(scheme, str) else scheme,
                                    first_recompute, length, seen, new_tokens, out))
        v = list(out)
        return {"hidden_pass": (v[0], v[1]), "kv_project": (v[2], v[3]), "lr_project": (v[4], v[5]),
                "kv_recompute": (v[6], v[7]), "skip_layers_below": v[8]}

    def append_fww(self, rows, row_begin, n_src):
        skip, add = C.c_int64(), C.c_int64()
        self._check(self._append_fww(rows, row_begin, n_src, C.byref(skip), C.byref(add)))
        return skip.value, add.value

    def page_of(self, row, page_tokens):
        a, b = C.c_int64(), C.c_int64()
        self._page_of(row, page_tokens, C.byref(a), C.byref(b))
        return a.value, b.value

    def round_bf16(self, x):
        """Round-to-nearest-even to bf16 and back to float32 (numpy; same bits as orc_round_bf16)."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        u = x.view(np.uint32).astype(np.uint64)
        c = lambda v: np.uint64(v)
        special = (u & c(0x7F800000)) == c(0x7F800000)
        r = (u + c(0x7FFF) + ((u >> c(16)) & c(1))) & c(0xFFFF0000)
        quiet = np.where((u & c(0x007FFFFF)) != c(0), c(0x00400000), c(0))
        r = np.where(special, (u | quiet) & c(0xFFFF0000), r)
        out = r.astype(np.uint32).view(np.float32).reshape(x.shape)
        if self.prefix == "orc_":   # keep the C helper honest
            chk = np.empty_like(x)
            P = C.POINTER(C.c_float)
            self._round_bf16_array(x.ctypes.data_as(P), chk.ctypes.data_as(P), x.size)
            assert np.array_equal(chk.view(np.uint32), out.view(np.uint32))
        return out

    def store(self, scheme, n_layers, d_kv, d_model, rank, n_agents, dtype=np.float64):
        return CheckerStore(self, scheme, n_layers, d_kv, d_model, rank, n_agents, dtype)

    def kernel_fuzz(self, cases, seed, max_len, dtype="f64"):
        n, a, b = C.c_int64(), C.c_double(), C.c_double()
        self._check(getattr(self, f"_kernel_fuzz_{dtype}")(cases, seed, max_len, C.byref(n),
                                                           C.byref(a), C.byref(b)))
        return n.value, a.value, b.value


class CheckerStore:
    """KvStore<T> (kvcache.hpp:213) behind the checker library."""

    def __init__(self, chk, scheme, n_layers, d_kv, d_model, rank, n_agents, dtype):
        self.chk = chk
        self.dtype = np.dtype(dtype)
        self.h = chk._store_create(SCHEMES[scheme] if isinstance(scheme, str) else scheme, n_layers,
                                   d_kv, d_model, rank, n_agents, self.dtype.itemsize)
        if not self.h:
            raise CheckerError(chk._last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.chk._store_destroy(self.h)
            self.h = None

    def append_tokens(self, n):
        self.chk._check(self.chk._store_append_tokens(self.h, n))

    def length(self):
        return self.chk._store_length(self.h)

    def seen(self, agent):
        out = C.c_int64()
        self.chk._check(self.chk._store_seen(self.h, agent, C.byref(out)))
        return out.value

    def mark_seen(self, agent):
        self.chk._check(self.chk._store_mark_seen(self.h, agent))

    def _append(self, which, layer, agent, row_begin, rows):
        rows = np.asarray(rows, dtype=self.dtype)
        assert rows.ndim == 2
        stride = rows.strides[0] // rows.itemsize if rows.shape[1] else 0
        self.chk._check(self.chk._store_append(self.h, which, layer, agent, row_begin,
                                               rows.ctypes.data_as(C.c_void_p), rows.shape[0],
                                               stride))

    def append_key(self, layer, agent, row_begin, rows):
        self._append(0, layer, agent, row_begin, rows)

    def append_value(self, layer, agent, row_begin, rows):
        self._append(1, layer, agent, row_begin, rows)

    def append_lr(self, layer, agent, row_begin, rows):
        self._append(2, layer, agent, row_begin, rows)

    def _view(self, which, layer, agent):
        data, rows, cols = C.c_void_p(), C.c_int64(), C.c_int64()
        self.chk._check(self.chk._store_view(self.h, which, layer, agent, C.byref(data),
                                             C.byref(rows), C.byref(cols)))
        n = rows.value * cols.value
        if n == 0:
            return np.zeros((rows.value, cols.value), dtype=self.dtype)
        buf = (C.c_char * (n * self.dtype.itemsize)).from_address(data.value)
        return np.frombuffer(buf, dtype=self.dtype).reshape(rows.value, cols.value).copy()

    def key_view(self, layer, agent):
        return self._view(0, layer, agent)

    def value_view(self, layer, agent):
        return self._view(1, layer, agent)

    def lr_view(self, layer, agent):
        return self._view(2, layer, agent)

    def bytes(self):
        out = (C.c_uint64 * 4)()
        self.chk._store_bytes(self.h, out)
        return {"key": out[0], "value": out[1], "lr": out[2], "hidden": out[3]}

    def allocated_elements(self):
        return self.chk._store_allocated_elements(self.h)


_cache: dict[str, Checker] = {}


def oracle() -> Checker:
    """The C restatement (always available; built on demand)."""
    if "port" not in _cache:
        _cache["port"] = Checker(build_oracle(), "orc_", "port")
    return _cache["port"]


def reference() -> Checker | None:
    """The reference's own code (oracle/_ref), or None when it was never built."""
    if "reference" not in _cache:
        path = build_ref()
        _cache["reference"] = Checker(path, "ref_", "reference") if path else None
    return _cache["reference"]


def best() -> Checker:
    """Reference when present, else the port."""
    return reference() or oracle()
