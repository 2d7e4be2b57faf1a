"""ctypes binding of include/lorakv_b200.h.  No compute happens here."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
_CSRC = os.path.join(_PKG, "csrc")
_LIB = os.environ.get("LORAKV_B200_LIB") or os.path.join(_PKG, "lib", "liblorakv_b200.so")   # the override is for A/B kernel builds (tools/)

F32, BF16 = 0, 1
HOST, DEVICE = 0, 1
KEY, VALUE, LR = 0, 1, 2
SCHEMES = {"NonShared": 0, "FullShared": 1, "BaseShared": 2, "BaseLRShared": 3, "SelectiveRecompute": 4}


class LorakvError(RuntimeError):
    """The reference reports every failure as std::runtime_error (matrix.hpp:17-19)."""


class PoolDims(C.Structure):
    _fields_ = [("scheme", C.c_int32), ("dtype", C.c_int32), ("n_layers", C.c_int64),
                ("n_kv_heads", C.c_int64), ("d_head", C.c_int64), ("d_model", C.c_int64),
                ("rank", C.c_int64), ("n_agents", C.c_int64), ("page_tokens", C.c_int64),
                ("max_tokens", C.c_int64), ("kv_head_begin", C.c_int64), ("n_kv_local", C.c_int64), ("rank_k", C.c_int64)]


def lib_path() -> str:
    return _LIB


def build(verbose: bool = False) -> str:
    """Compile every CUDA source for sm_100a into lib/liblorakv_b200.so (nvcc cross-compiles on CPU)."""
    res = subprocess.run(["make", "-C", _CSRC, "-j8", "all"], capture_output=True, text=True)
    if verbose or res.returncode != 0:
        print(res.stdout[-4000:])
        print(res.stderr[-4000:])
    if res.returncode != 0:
        raise RuntimeError("building liblorakv_b200.so failed")
    return _LIB


_lib = None

# name -> (restype, argtypes); also the list of symbols tests check against the header
_f, _d, _i64, _vp = C.c_float, C.c_double, C.c_int64, C.c_void_p
_pf, _pd = C.POINTER(C.c_float), C.POINTER(C.c_double)


def _attn_sig(T, P, stats):
    sig = [_vp, P, _i64, P, _i64, P, _i64, P, _i64, P, _i64, T, _i64, _i64, _i64, _i64, _i64, P]
    return sig + ([P, P] if stats else [])


def _gqa_sig(T, P):
    return [_vp, P, _i64, P, _i64, P, _i64, P, _i64, P, _i64, T, _i64, _i64, _i64, _i64, _i64, _i64, _i64, P]


SIGNATURES = {
    "lorakv_abi_version": (C.c_int, []),
    "lorakv_last_error": (C.c_char_p, []),
    "lorakv_ctx_create": (C.c_int, [C.c_int, _vp, C.POINTER(_vp)]),
    "lorakv_ctx_destroy": (None, [_vp]),
    "lorakv_ctx_synchronize": (C.c_int, [_vp]),
    "lorakv_ctx_stream": (_vp, [_vp]),
    "lorakv_ctx_sm_count": (C.c_int, [_vp]),
    "lorakv_ctx_launch_count": (_i64, [_vp]),
    "lorakv_ctx_set_l2_bytes": (C.c_int, [_vp, _i64]),
    "lorakv_ctx_set_prefill_split_keys": (C.c_int, [_vp, _i64]),
    "lorakv_dev_alloc": (C.c_int, [_vp, _i64, C.POINTER(_vp)]),
    "lorakv_dev_free": (C.c_int, [_vp, _vp]),
    "lorakv_host_alloc": (C.c_int, [_vp, _i64, C.POINTER(_vp)]),
    "lorakv_host_free": (C.c_int, [_vp, _vp]),
    "lorakv_copy_h2d": (C.c_int, [_vp, _vp, _vp, _i64]),
    "lorakv_copy_d2h": (C.c_int, [_vp, _vp, _vp, _i64]),
    "lorakv_flush_l2": (C.c_int, [_vp]),
    "lorakv_event_create": (C.c_int, [_vp, C.POINTER(_vp)]),
    "lorakv_event_record": (C.c_int, [_vp, _vp]),
    "lorakv_event_elapsed_ms": (C.c_int, [_vp, _vp, C.POINTER(C.c_float)]),
    "lorakv_event_destroy": (None, [_vp]),
    "lorakv_fla_forward_f32": (C.c_int, _attn_sig(_f, _pf, True)),
    "lorakv_fla_forward_f64": (C.c_int, _attn_sig(_d, _pd, True)),
    "lorakv_expand_first_forward_f32": (C.c_int, _attn_sig(_f, _pf, False)),
    "lorakv_expand_first_forward_f64": (C.c_int, _attn_sig(_d, _pd, False)),
    "lorakv_naive_forward_f32": (C.c_int, _attn_sig(_f, _pf, False)),
    "lorakv_naive_forward_f64": (C.c_int, _attn_sig(_d, _pd, False)),
    "lorakv_gqa_forward_f32": (C.c_int, _gqa_sig(_f, _pf)),
    "lorakv_gqa_forward_f64": (C.c_int, _gqa_sig(_d, _pd)),
    "lorakv_gqa_forward_keylr_f32": (C.c_int, [_vp, _pf, _i64, _pf, _i64, _pf, _i64, _pf, _i64, _pf, _i64, _f, _pf, _i64, _pf, _i64, _f,
                                               _i64, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _pf]),
    "lorakv_gqa_forward_keylr_f64": (C.c_int, [_vp, _pd, _i64, _pd, _i64, _pd, _i64, _pd, _i64, _pd, _i64, _d, _pd, _i64, _pd, _i64, _d,
                                               _i64, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _pd]),
    "lorakv_adapters_enable_key": (C.c_int, [_vp, _i64]),
    "lorakv_adapters_set_a_k": (C.c_int, [_vp, _i64, _pf]),
    "lorakv_adapters_set_b_k": (C.c_int, [_vp, _i64, _i64, _pf, _d]),
    "lorakv_pool_append_lk_project": (C.c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _i64, C.c_int, C.POINTER(_i64)]),
    "lorakv_matmul_f32": (C.c_int, [_vp, _pf, _i64, _pf, _i64, _i64, _i64, _i64, _pf]),
    "lorakv_matmul_f64": (C.c_int, [_vp, _pd, _i64, _pd, _i64, _i64, _i64, _i64, _pd]),
    "lorakv_lr_mac_counts": (None, [_i64, _i64, _i64, _i64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "lorakv_attn_macs": (None, [_i64, _i64, _i64, _i64, C.c_int, C.POINTER(C.c_uint64)]),
    "lorakv_plan_core": (C.c_int, [C.c_int, _i64, _i64, _i64, _i64, C.POINTER(_i64)]),
    "lorakv_pool_create": (C.c_int, [_vp, C.POINTER(PoolDims), C.POINTER(_vp)]),
    "lorakv_pool_destroy": (None, [_vp]),
    "lorakv_pool_dims_get": (C.c_int, [_vp, C.POINTER(PoolDims)]),
    "lorakv_pool_append_tokens": (C.c_int, [_vp, _i64]),
    "lorakv_pool_length": (_i64, [_vp]),
    "lorakv_pool_seen": (C.c_int, [_vp, _i64, C.POINTER(_i64)]),
    "lorakv_pool_mark_seen": (C.c_int, [_vp, _i64]),
    "lorakv_pool_plan_step": (C.c_int, [_vp, _i64, _i64, C.POINTER(_i64)]),
    "lorakv_pool_append": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, _vp, _i64, _i64, C.c_int, C.POINTER(_i64)]),
    "lorakv_pool_append_lr_project": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _i64, C.c_int, C.POINTER(_i64)]),
    "lorakv_pool_save_snapshot": (C.c_int, [_vp, C.c_char_p, C.POINTER(C.c_int32), _i64]),
    "lorakv_pool_load_snapshot": (C.c_int, [_vp, C.c_char_p, C.c_int, _i64, _i64, _i64, C.POINTER(_vp), C.POINTER(C.c_int32), _i64,
                                            C.POINTER(_i64)]),
    "lorakv_pool_append_kv_project_full": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _vp, _i64, _i64, C.c_int, C.c_int, C.POINTER(_i64)]),
    "lorakv_proj_create": (C.c_int, [_vp, _i64, _i64, _i64, _i64, _i64, _i64, C.c_int, C.POINTER(_vp)]),
    "lorakv_proj_destroy": (None, [_vp]),
    "lorakv_proj_set_kv": (C.c_int, [_vp, _i64, _pf, _pf]),
    "lorakv_proj_set_q": (C.c_int, [_vp, _i64, _i64, _pf]),
    "lorakv_proj_set_q_lora": (C.c_int, [_vp, _i64, _i64, _i64, _i64, _pf, _pf, C.c_double]),
    "lorakv_proj_query": (C.c_int, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, C.c_int, _vp, C.c_int]),
    "lorakv_pool_append_kv_project": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _i64, C.c_int, C.c_int, C.POINTER(_i64)]),
    "lorakv_pool_rows": (C.c_int, [_vp, C.c_int, _i64, _i64, C.POINTER(_i64)]),
    "lorakv_pool_read": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, _i64, _pf]),
    "lorakv_pool_bytes": (C.c_int, [_vp, C.POINTER(C.c_uint64)]),
    "lorakv_pool_allocated_elements": (C.c_uint64, [_vp]),
    "lorakv_pool_reserved_bytes": (C.c_uint64, [_vp]),
    "lorakv_pool_page_table": (C.c_int, [_vp, C.c_int, _i64, C.POINTER(C.c_int32), _i64, C.POINTER(_i64)]),
    "lorakv_adapters_create": (C.c_int, [_vp, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _i64, C.c_int, C.POINTER(_vp)]),
    "lorakv_adapters_destroy": (None, [_vp]),
    "lorakv_adapters_set_a": (C.c_int, [_vp, _i64, _pf]),
    "lorakv_adapters_set_a_agent": (C.c_int, [_vp, _i64, _i64, _pf]),
    "lorakv_adapters_set_b": (C.c_int, [_vp, _i64, _i64, _pf, C.c_double]),
    "lorakv_fla_decode_batched": (C.c_int, [_vp, _vp, _i64, _i64, C.POINTER(C.c_int32), _i64, _i64, _vp, _vp, C.c_int]),
    "lorakv_gather_create": (C.c_int, [_vp, C.c_int, C.c_int, _i64, C.POINTER(_vp)]),
    "lorakv_gather_destroy": (None, [_vp]),
    "lorakv_gather_disconnect": (C.c_int, [_vp]),
    "lorakv_gather_export": (C.c_int, [_vp, C.POINTER(C.c_ubyte)]),
    "lorakv_gather_connect": (C.c_int, [_vp, C.POINTER(C.c_ubyte)]),
    "lorakv_gather_set_timeout_ms": (C.c_int, [_vp, _i64]),
    "lorakv_gather_set_overlap": (C.c_int, [_vp, C.c_int]),
    "lorakv_gather_wait": (C.c_int, [_vp]),
    "lorakv_gather_steps": (C.c_int, [_vp, C.POINTER(_i64)]),
    "lorakv_gather_check": (C.c_int, [_vp]),
    "lorakv_fla_decode_batched_gather": (C.c_int, [_vp, _vp, _vp, _i64, _i64, C.POINTER(C.c_int32), _i64, _i64, _vp, C.c_int, _vp,
                                                   C.POINTER(_vp)]),
    "lorakv_fla_prefill": (C.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, C.c_int]),
    "lorakv_pool_append_f64": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, _pd, _i64, _i64, C.c_int, C.POINTER(_i64)]),
    "lorakv_pool_read_f64": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, _i64, _pd]),
    "lorakv_pool_set_recompute_layers": (C.c_int, [_vp, C.POINTER(_i64), _i64]),
    "lorakv_pool_get_recompute_layers": (C.c_int, [_vp, C.POINTER(_i64), _i64, C.POINTER(_i64)]),
    "lorakv_pool_overwrite": (C.c_int, [_vp, C.c_int, _i64, _i64, _pf, _i64, _i64, C.c_int]),
    "lorakv_pool_overwrite_f64": (C.c_int, [_vp, C.c_int, _i64, _i64, _pd, _i64, _i64, C.c_int]),
    "lorakv_step_layer": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _vp, _i64, _i64, C.c_int, _i64, _vp, _vp, C.c_int]),
    "lorakv_snapshot_tokens": (C.c_int, [C.c_char_p, C.POINTER(C.c_int32), _i64, C.POINTER(_i64)]),
    "lorakv_ctx_set_profiling": (C.c_int, [_vp, C.c_int]),
    "lorakv_ctx_last_kernel_ms": (C.c_int, [_vp, C.POINTER(C.c_float)]),
    "lorakv_ctx_mean_kernel_ms": (C.c_int, [_vp, C.POINTER(C.c_float), C.POINTER(C.c_int)]),
    "lorakv_selftest_umma": (C.c_int, [_vp, _pf, _pf, C.c_int, C.c_int, C.c_int, C.c_float, C.c_int, C.c_int, _pf]),
    "lorakv_set_kernel_policy": (C.c_int, [_vp, C.c_int]),
    "lorakv_last_kernel": (C.c_char_p, [_vp]),
}


def load_library(path: str | None = None):
    """dlopen the product library and bind every declared symbol.  Raises when it is missing --
    there is deliberately no Python or CPU stand-in."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or _LIB
    if not os.path.exists(p):
        raise LorakvError(f"{p} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(p)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.lorakv_abi_version() != 6:
        raise LorakvError("liblorakv_b200.so ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


def _check(rc):
    if rc != 0:
        raise LorakvError(load_library().lorakv_last_error().decode())


def _span(a, T):
    """(pointer, row stride in elements) of a 2-D array with contiguous innermost axis."""
    assert a.ndim == 2
    if a.size and a.shape[1] > 1:
        assert a.strides[1] == a.itemsize, "innermost axis must be contiguous"
    ld = a.strides[0] // a.itemsize if a.shape[0] > 1 else max(a.shape[1], 1)
    ptr = a.ctypes.data_as(C.POINTER(T)) if a.size else C.POINTER(T)()
    return ptr, ld


class Context:
    """lorakv_ctx: one device + stream.  stream: raw cudaStream_t (int) to borrow, or None."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self.lib = load_library()
        h = _vp()
        _check(self.lib.lorakv_ctx_create(device, _vp(stream) if stream else None, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.lorakv_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        _check(self.lib.lorakv_ctx_synchronize(self.h))

    @property
    def sm_count(self):
        return self.lib.lorakv_ctx_sm_count(self.h)

    @property
    def launch_count(self):
        return self.lib.lorakv_ctx_launch_count(self.h)

    @property
    def stream(self):
        return self.lib.lorakv_ctx_stream(self.h)

    def set_kernel_policy(self, policy: int) -> int:
        return self.lib.lorakv_set_kernel_policy(self.h, policy)

    def set_l2_bytes(self, nbytes: int):
        """L2 capacity the decode plans its V_lr residency with (tests shrink it to force the layer-chunked path)."""
        _check(self.lib.lorakv_ctx_set_l2_bytes(self.h, int(nbytes)))

    def set_prefill_split_keys(self, keys: int):
        """Keys per split of the fp32-mode tcgen05 prefill (0 = default 4096); tests shrink it to cover many splits."""
        _check(self.lib.lorakv_ctx_set_prefill_split_keys(self.h, int(keys)))

    def set_profiling(self, enabled: bool):
        _check(self.lib.lorakv_ctx_set_profiling(self.h, int(enabled)))

    def last_kernel_ms(self) -> float:
        ms = C.c_float()
        _check(self.lib.lorakv_ctx_last_kernel_ms(self.h, C.byref(ms)))
        return float(ms.value)

    def mean_kernel_ms(self):
        """(mean device time of the dominant kernel over the profiled calls since set_profiling(True), calls averaged)"""
        ms, n = C.c_float(), C.c_int()
        _check(self.lib.lorakv_ctx_mean_kernel_ms(self.h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def selftest_umma(self, a, b, b_mn_major: bool, alpha: float = 1.0, rescale: bool = False, a_in_tmem: bool = False):
        a = np.ascontiguousarray(a, dtype=np.float32); b = np.ascontiguousarray(b, dtype=np.float32)
        K = a.shape[1]
        N = b.shape[1] if b_mn_major else b.shape[0]
        out = np.zeros((128, N), dtype=np.float32)
        _check(self.lib.lorakv_selftest_umma(self.h, a.ctypes.data_as(_pf), b.ctypes.data_as(_pf), N, K, int(b_mn_major),
                                             alpha, int(rescale), int(a_in_tmem), out.ctypes.data_as(_pf)))
        return out

    def last_kernel(self) -> str:
        return self.lib.lorakv_last_kernel(self.h).decode()

    def flush_l2(self):
        _check(self.lib.lorakv_flush_l2(self.h))

    # device timing on the ctx stream -----------------------------------------------------------
    def event(self) -> "Event":
        return Event(self)

    # raw buffers -----------------------------------------------------------------------------
    def dev_alloc(self, nbytes: int) -> int:
        p = _vp()
        _check(self.lib.lorakv_dev_alloc(self.h, nbytes, C.byref(p)))
        return p.value

    def dev_free(self, p: int):
        _check(self.lib.lorakv_dev_free(self.h, _vp(p)))

    def pinned_array(self, shape, dtype=np.float32):
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = _vp()
        _check(self.lib.lorakv_host_alloc(self.h, n, C.byref(p)))
        buf = (C.c_char * max(n, 1)).from_address(p.value)
        arr = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)
        self._pinned = getattr(self, "_pinned", []) + [p.value]   # freed with the process
        return arr

    def h2d(self, dst_dev: int, src: np.ndarray):
        src = np.ascontiguousarray(src)
        _check(self.lib.lorakv_copy_h2d(self.h, _vp(dst_dev), src.ctypes.data_as(_vp), src.nbytes))

    def d2h(self, dst: np.ndarray, src_dev: int):
        assert dst.flags.c_contiguous
        _check(self.lib.lorakv_copy_d2h(self.h, dst.ctypes.data_as(_vp), _vp(src_dev), dst.nbytes))

    # per-head operators over host arrays (float32 / float64) -----------------------------------
    def _attn(self, name, q, k, v, v_lr, b_up, lr_scale, query_offset, stats=False):
        if q.dtype == np.float32:
            suf, T = "f32", _f
        elif q.dtype == np.float64:
            suf, T = "f64", _d
        else:
            raise TypeError(q.dtype)
        for a in (k, v, v_lr, b_up):
            assert a.dtype == q.dtype
        L_c, d = q.shape
        L, r = k.shape[0], v_lr.shape[1]
        if k.shape[1] != d or v.shape != (L, d) or (r > 0 and (v_lr.shape[0] != L or b_up.shape != (r, d))) \
                or b_up.shape[0] != r:
            raise LorakvError("attention: operand shapes do not match")
        out = np.zeros((L_c, d), dtype=q.dtype)
        args = []
        for a in (q, k, v, v_lr, b_up):
            args.extend(_span(a, T))
        P = C.POINTER(T)
        tail = [out.ctypes.data_as(P)]
        rmax = rden = None
        if stats:
            rmax = np.zeros(L_c, dtype=q.dtype)
            rden = np.zeros(L_c, dtype=q.dtype)
            tail += [rmax.ctypes.data_as(P), rden.ctypes.data_as(P)]
        elif name == "fla_forward":
            tail += [P(), P()]
        _check(getattr(self.lib, f"lorakv_{name}_{suf}")(self.h, *args, T(lr_scale), L_c, L, d, r,
                                                        query_offset, *tail))
        return (out, rmax, rden) if stats else out

    def flash_lora_attention(self, q, k, v, v_lr, b_up, lr_scale, query_offset, stats=False):
        return self._attn("fla_forward", q, k, v, v_lr, b_up, lr_scale, query_offset, stats)

    def expand_first_attention(self, q, k, v, v_lr, b_up, lr_scale, query_offset):
        return self._attn("expand_first_forward", q, k, v, v_lr, b_up, lr_scale, query_offset)

    def naive_attention(self, q, k, v, v_lr, b_up, lr_scale, query_offset):
        return self._attn("naive_forward", q, k, v, v_lr, b_up, lr_scale, query_offset)

    def matmul(self, a, b):
        suf, T = ("f32", _f) if a.dtype == np.float32 else ("f64", _d)
        assert a.dtype == b.dtype and a.shape[1] == b.shape[0]
        out = np.zeros((a.shape[0], b.shape[1]), dtype=a.dtype)
        (pa, lda), (pb, ldb) = _span(a, T), _span(b, T)
        _check(getattr(self.lib, f"lorakv_matmul_{suf}")(self.h, pa, lda, pb, ldb, a.shape[0], a.shape[1],
                                                        b.shape[1], out.ctypes.data_as(C.POINTER(T))))
        return out

    def gqa_attention_keylr(self, q, k, v, v_lr, b_up, lr_scale, l_k, b_k, k_scale, query_offset, n_q, n_kv):
        """gqa_attention over K_eff = K_base + k_scale * L_k B_k without forming K_eff (extension, parity unpinned)."""
        T = np.float64 if q.dtype == np.float64 else np.float32
        arrs = [np.ascontiguousarray(a, dtype=T) for a in (q, k, v, v_lr, b_up, l_k, b_k)]
        q, k, v, v_lr, b_up, l_k, b_k = arrs
        P, fn = (_pd, self.lib.lorakv_gqa_forward_keylr_f64) if T == np.float64 else (_pf, self.lib.lorakv_gqa_forward_keylr_f32)
        d = q.shape[1] // n_q
        out = np.zeros((q.shape[0], q.shape[1]), dtype=T)
        ld = lambda a: max(a.shape[1], 1)
        ptr = lambda a: a.ctypes.data_as(P)
        _check(fn(self.h, ptr(q), ld(q), ptr(k), ld(k), ptr(v), ld(v), ptr(v_lr), ld(v_lr), ptr(b_up), ld(b_up), T(lr_scale),
                  ptr(l_k), ld(l_k), ptr(b_k), ld(b_k), T(k_scale), q.shape[0], k.shape[0], n_q, n_kv, d, v_lr.shape[1], l_k.shape[1],
                  query_offset, ptr(out)))
        return out

    def gqa_attention(self, q, k, v, v_lr, b_up, lr_scale, query_offset, n_q, n_kv):
        suf, T = ("f32", _f) if q.dtype == np.float32 else ("f64", _d)
        if n_q < 1 or n_kv < 1 or n_q % n_kv or q.shape[1] % n_q:
            raise LorakvError(f"gqa_attention: n_q_heads {n_q} not divisible by n_kv_heads {n_kv}")
        d = q.shape[1] // n_q
        L, r = k.shape[0], v_lr.shape[1]
        if k.shape[1] != n_kv * d or v.shape != k.shape:
            raise LorakvError("gqa_attention: k/v width does not match n_kv_heads * d_head")
        out = np.zeros(q.shape, dtype=q.dtype)
        args = []
        for a in (q, k, v, v_lr, b_up):
            args.extend(_span(a, T))
        _check(getattr(self.lib, f"lorakv_gqa_forward_{suf}")(
            self.h, *args, T(lr_scale), q.shape[0], L, n_q, n_kv, d, r, query_offset,
            out.ctypes.data_as(C.POINTER(T))))
        return out


class Event:
    """lorakv_event: a CUDA event recorded on the ctx stream (the stream the kernels launch on)."""

    def __init__(self, ctx: Context):
        self.ctx = ctx
        h = _vp()
        _check(ctx.lib.lorakv_event_create(ctx.h, C.byref(h)))
        self.h = h

    def record(self):
        _check(self.ctx.lib.lorakv_event_record(self.ctx.h, self.h))
        return self

    def elapsed_ms(self, stop: "Event") -> float:
        ms = C.c_float()
        _check(self.ctx.lib.lorakv_event_elapsed_ms(self.h, stop.h, C.byref(ms)))
        return float(ms.value)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.ctx.lib.lorakv_event_destroy(self.h)
                self.h = None
        except Exception:
            pass


def lr_mac_counts(L, L_c, r, d):
    a, b = C.c_uint64(), C.c_uint64()
    load_library().lorakv_lr_mac_counts(L, L_c, r, d, C.byref(a), C.byref(b))
    return a.value, b.value


def attn_macs(L_c, L, d, r, expand_first=False):
    out = (C.c_uint64 * 3)()
    load_library().lorakv_attn_macs(L_c, L, d, r, int(expand_first), out)
    return tuple(out)


def plan_core(scheme, length, seen, new_tokens, first_recompute=0):
    out = (_i64 * 9)()
    _check(load_library().lorakv_plan_core(SCHEMES[scheme] if isinstance(scheme, str) else scheme,
                                           first_recompute, length, seen, new_tokens, out))
    v = list(out)
    return {"hidden_pass": (v[0], v[1]), "kv_project": (v[2], v[3]), "lr_project": (v[4], v[5]),
            "kv_recompute": (v[6], v[7]), "skip_layers_below": v[8]}


class Adapters:
    """lorakv_adapters: shared A per layer, B and alpha per (layer, agent)."""

    def __init__(self, ctx: Context, n_layers, n_agents, d_model, rank, n_kv_heads, d_head,
                 kv_head_begin=0, n_kv_local=0, dtype=F32):
        self.ctx = ctx
        h = _vp()
        _check(ctx.lib.lorakv_adapters_create(ctx.h, n_layers, n_agents, d_model, rank, n_kv_heads,
                                              d_head, kv_head_begin, n_kv_local, dtype, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.lorakv_adapters_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_a(self, layer, a):
        a = np.ascontiguousarray(a, dtype=np.float32)
        _check(self.ctx.lib.lorakv_adapters_set_a(self.h, layer, a.ctypes.data_as(_pf)))

    def set_a_agent(self, layer, agent, a):
        a = np.ascontiguousarray(a, dtype=np.float32)
        _check(self.ctx.lib.lorakv_adapters_set_a_agent(self.h, layer, agent, a.ctypes.data_as(_pf)))

    def enable_key(self, rank_k):
        _check(self.ctx.lib.lorakv_adapters_enable_key(self.h, rank_k))

    def set_a_k(self, layer, a_k):
        a_k = np.ascontiguousarray(a_k, dtype=np.float32)
        _check(self.ctx.lib.lorakv_adapters_set_a_k(self.h, layer, a_k.ctypes.data_as(_pf)))

    def set_b_k(self, layer, agent, b_k, alpha_k):
        b_k = np.ascontiguousarray(b_k, dtype=np.float32)
        _check(self.ctx.lib.lorakv_adapters_set_b_k(self.h, layer, agent, b_k.ctypes.data_as(_pf), float(alpha_k)))

    def set_b(self, layer, agent, b, alpha):
        b = np.ascontiguousarray(b, dtype=np.float32)
        _check(self.ctx.lib.lorakv_adapters_set_b(self.h, layer, agent, b.ctypes.data_as(_pf), alpha))


class Gather:
    """lorakv_gather: the end-of-step output gather of a kv-head-sharded decode over peer memory."""
    HANDLE_BYTES = 64

    def __init__(self, ctx: Context, rank: int, world: int, full_elems: int):
        self.ctx, self.rank, self.world, self.full_elems = ctx, rank, world, int(full_elems)
        h = _vp()
        _check(ctx.lib.lorakv_gather_create(ctx.h, rank, world, self.full_elems, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.lorakv_gather_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def disconnect(self):
        """Unmap the peers' buffers; barrier across ranks before close()."""
        _check(self.ctx.lib.lorakv_gather_disconnect(self.h))

    def export(self) -> bytes:
        buf = (C.c_ubyte * self.HANDLE_BYTES)()
        _check(self.ctx.lib.lorakv_gather_export(self.h, buf))
        return bytes(buf)

    def connect(self, handles):
        """handles: the exported handles of ranks 0..world-1, in rank order (bytes each, or one joined blob)."""
        blob = handles if isinstance(handles, (bytes, bytearray)) else b"".join(handles)
        if len(blob) != self.world * self.HANDLE_BYTES:
            raise LorakvError(f"gather_connect: {len(blob)} handle bytes for world size {self.world}")
        buf = (C.c_ubyte * len(blob)).from_buffer_copy(blob)
        _check(self.ctx.lib.lorakv_gather_connect(self.h, buf))

    def set_overlap(self, enabled: bool):
        _check(self.ctx.lib.lorakv_gather_set_overlap(self.h, 1 if enabled else 0))

    def wait(self):
        _check(self.ctx.lib.lorakv_gather_wait(self.h))

    def set_timeout_ms(self, ms: int):
        _check(self.ctx.lib.lorakv_gather_set_timeout_ms(self.h, ms))

    def steps(self) -> int:
        n = _i64()
        _check(self.ctx.lib.lorakv_gather_steps(self.h, C.byref(n)))
        return n.value

    def check(self):
        _check(self.ctx.lib.lorakv_gather_check(self.h))


class Projection:
    """lorakv_proj: Wk / Wv per layer for the fused projection + RoPE + append (engine.hpp:376-403)."""

    def __init__(self, ctx: Context, n_layers, d_model, n_kv_heads, d_head, kv_head_begin=0, n_kv_local=0, dtype=F32):
        self.ctx = ctx
        h = _vp()
        _check(ctx.lib.lorakv_proj_create(ctx.h, n_layers, d_model, n_kv_heads, d_head, kv_head_begin, n_kv_local,
                                          dtype, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.lorakv_proj_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_kv(self, layer, wk, wv):
        wk = np.ascontiguousarray(wk, dtype=np.float32)
        wv = np.ascontiguousarray(wv, dtype=np.float32)
        _check(self.ctx.lib.lorakv_proj_set_kv(self.h, layer, wk.ctypes.data_as(_pf), wv.ctypes.data_as(_pf)))

    def set_q(self, layer, n_q_heads, wq):
        wq = np.ascontiguousarray(wq, dtype=np.float32)
        self._dq_full = wq.shape[1]
        _check(self.ctx.lib.lorakv_proj_set_q(self.h, layer, n_q_heads, wq.ctypes.data_as(_pf)))

    def set_q_lora(self, layer, agent, n_agents, a_q, b_q, alpha):
        a_q = np.ascontiguousarray(a_q, dtype=np.float32)
        b_q = np.ascontiguousarray(b_q, dtype=np.float32)
        _check(self.ctx.lib.lorakv_proj_set_q_lora(self.h, layer, agent, n_agents, a_q.shape[1], a_q.ctypes.data_as(_pf),
                                                   b_q.ctypes.data_as(_pf), alpha))

    def query(self, layer, agent, pos_begin, x, n_q_local_cols, rope=True):
        """q rows of the shard's heads for x (host arrays); agent < 0 skips the adapter."""
        x = np.asarray(x, dtype=np.float32)
        ptr, ld_ = _span(x, _f)
        out = np.empty((x.shape[0], n_q_local_cols), dtype=np.float32)
        _check(self.ctx.lib.lorakv_proj_query(self.h, layer, agent, pos_begin, C.cast(ptr, _vp), x.shape[0], ld_, int(rope),
                                              out.ctypes.data_as(_vp), HOST))
        return out

    def query_device(self, layer, agent, pos_begin, x_ptr, n_rows, ld, q_ptr, rope=True):
        _check(self.ctx.lib.lorakv_proj_query(self.h, layer, agent, pos_begin, _vp(x_ptr), n_rows, ld, int(rope), _vp(q_ptr), DEVICE))


class Pool:
    """lorakv_pool: the paged HBM cache of one trajectory with KvStore's interface (kvcache.hpp:213)."""

    def __init__(self, ctx: Context, scheme, n_layers, n_kv_heads, d_head, d_model, rank, n_agents,
                 max_tokens, dtype=F32, page_tokens=0, kv_head_begin=0, n_kv_local=0, rank_k=0):
        self.ctx = ctx
        dims = PoolDims(SCHEMES[scheme] if isinstance(scheme, str) else scheme, dtype, n_layers,
                        n_kv_heads, d_head, d_model, rank, n_agents, page_tokens, max_tokens,
                        kv_head_begin, n_kv_local, rank_k)
        h = _vp()
        _check(ctx.lib.lorakv_pool_create(ctx.h, C.byref(dims), C.byref(h)))
        self.h = h
        got = PoolDims()
        _check(ctx.lib.lorakv_pool_dims_get(h, C.byref(got)))
        self.dims = got

    @classmethod
    def load_snapshot(cls, ctx: Context, path, n_kv_heads, dtype=F32, page_tokens=0, max_tokens=0):
        """KvStore::load_snapshot (kvcache.hpp:472-521) into a new pool; returns (pool, token ids)."""
        self = cls.__new__(cls)
        self.ctx = ctx
        h, n = _vp(), _i64()
        cap = 1 << 20
        toks = (C.c_int32 * cap)()
        _check(ctx.lib.lorakv_pool_load_snapshot(ctx.h, str(path).encode(), dtype, n_kv_heads, page_tokens, max_tokens,
                                                 C.byref(h), toks, cap, C.byref(n)))
        self.h = h
        got = PoolDims()
        _check(ctx.lib.lorakv_pool_dims_get(h, C.byref(got)))
        self.dims = got
        return self, list(toks[:min(n.value, cap)])

    def save_snapshot(self, path, tokens):
        """KvStore::save_snapshot (kvcache.hpp:438-470); tokens = the trajectory's token ids."""
        arr = (C.c_int32 * len(tokens))(*tokens)
        _check(self.ctx.lib.lorakv_pool_save_snapshot(self.h, str(path).encode(), arr, len(tokens)))

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.lorakv_pool_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # KvStore surface --------------------------------------------------------------------------
    def append_tokens(self, n):
        _check(self.ctx.lib.lorakv_pool_append_tokens(self.h, n))

    def length(self):
        return self.ctx.lib.lorakv_pool_length(self.h)

    def seen(self, agent):
        out = _i64()
        _check(self.ctx.lib.lorakv_pool_seen(self.h, agent, C.byref(out)))
        return out.value

    def mark_seen(self, agent):
        _check(self.ctx.lib.lorakv_pool_mark_seen(self.h, agent))

    def plan_step(self, agent, new_tokens):
        out = (_i64 * 9)()
        _check(self.ctx.lib.lorakv_pool_plan_step(self.h, agent, new_tokens, out))
        v = list(out)
        return {"hidden_pass": (v[0], v[1]), "kv_project": (v[2], v[3]), "lr_project": (v[4], v[5]),
                "kv_recompute": (v[6], v[7]), "skip_layers_below": v[8]}

    def _append(self, which, layer, agent, row_begin, rows):
        rows = np.asarray(rows, dtype=np.float32)
        assert rows.ndim == 2
        ptr, ld = _span(rows, _f)
        added = _i64()
        _check(self.ctx.lib.lorakv_pool_append(self.h, which, layer, agent, row_begin,
                                               C.cast(ptr, _vp), rows.shape[0], ld, HOST, C.byref(added)))
        return added.value

    def append_key(self, layer, agent, row_begin, rows):
        return self._append(KEY, layer, agent, row_begin, rows)

    def append_value(self, layer, agent, row_begin, rows):
        return self._append(VALUE, layer, agent, row_begin, rows)

    def append_lk(self, layer, row_begin, rows):
        """key-side low-rank rows L_k (n x rank_k), the extension of lorakv_gqa_forward_keylr_*"""
        return self._append(4, layer, 0, row_begin, rows)

    def append_lk_project(self, adapters, layer, row_begin, x):
        x = np.ascontiguousarray(x, dtype=np.float32)
        n = _i64()
        _check(self.ctx.lib.lorakv_pool_append_lk_project(self.h, adapters.h, layer, row_begin, x.ctypes.data_as(_vp), x.shape[0],
                                                          x.shape[1], HOST, C.byref(n)))
        return n.value

    def lk_view(self, layer):
        return self._view(4, layer, 0)

    def append_lr(self, layer, agent, row_begin, rows):
        return self._append(LR, layer, agent, row_begin, rows)

    def append_device(self, which, layer, agent, row_begin, dev_ptr, n_rows, ld):
        added = _i64()
        _check(self.ctx.lib.lorakv_pool_append(self.h, which, layer, agent, row_begin, _vp(dev_ptr),
                                               n_rows, ld, DEVICE, C.byref(added)))
        return added.value

    def append_lr_project(self, adapters: Adapters, layer, agent, row_begin, x=None, dev_ptr=None,
                          n_rows=None, ld=None):
        added = _i64()
        if dev_ptr is None:
            x = np.asarray(x, dtype=np.float32)
            ptr, ld_ = _span(x, _f)
            _check(self.ctx.lib.lorakv_pool_append_lr_project(self.h, adapters.h, layer, agent, row_begin,
                                                              C.cast(ptr, _vp), x.shape[0], ld_, HOST,
                                                              C.byref(added)))
        else:
            _check(self.ctx.lib.lorakv_pool_append_lr_project(self.h, adapters.h, layer, agent, row_begin,
                                                              _vp(dev_ptr), n_rows, ld, DEVICE, C.byref(added)))
        return added.value

    def append_kv_project(self, proj: "Projection", layer, agent, row_begin, x=None, rope=True, dev_ptr=None,
                          n_rows=None, ld=None, merge: "Adapters" = None):
        added = _i64()
        if merge is not None:        # "full values": V rows carry the agent's LoRA contribution (engine.hpp:385-393)
            x = np.asarray(x, dtype=np.float32)
            ptr, ld_ = _span(x, _f)
            _check(self.ctx.lib.lorakv_pool_append_kv_project_full(self.h, proj.h, merge.h, layer, agent, row_begin,
                                                                   C.cast(ptr, _vp), x.shape[0], ld_, HOST, int(rope),
                                                                   C.byref(added)))
            return added.value
        if dev_ptr is None:
            x = np.asarray(x, dtype=np.float32)
            ptr, ld_ = _span(x, _f)
            _check(self.ctx.lib.lorakv_pool_append_kv_project(self.h, proj.h, layer, agent, row_begin,
                                                              C.cast(ptr, _vp), x.shape[0], ld_, HOST, int(rope),
                                                              C.byref(added)))
        else:
            _check(self.ctx.lib.lorakv_pool_append_kv_project(self.h, proj.h, layer, agent, row_begin, _vp(dev_ptr),
                                                              n_rows, ld, DEVICE, int(rope), C.byref(added)))
        return added.value

    def rows(self, which, layer, agent):
        out = _i64()
        _check(self.ctx.lib.lorakv_pool_rows(self.h, which, layer, agent, C.byref(out)))
        return out.value

    def _view(self, which, layer, agent):
        n = self.rows(which, layer, agent)
        cols = self.dims.rank if which == LR else self.dims.rank_k if which == 4 else self.dims.n_kv_local * self.dims.d_head
        if which == LR and self.dims.scheme not in (2, 3):
            cols = 0
        out = np.zeros((n, cols), dtype=np.float32)
        if out.size:
            _check(self.ctx.lib.lorakv_pool_read(self.h, which, layer, agent, 0, n, out.ctypes.data_as(_pf)))
        return out

    def key_view(self, layer, agent):
        return self._view(KEY, layer, agent)

    def value_view(self, layer, agent):
        return self._view(VALUE, layer, agent)

    def lr_view(self, layer, agent):
        return self._view(LR, layer, agent)

    def bytes(self):
        out = (C.c_uint64 * 4)()
        _check(self.ctx.lib.lorakv_pool_bytes(self.h, out))
        return {"key": out[0], "value": out[1], "lr": out[2], "hidden": out[3]}

    def allocated_elements(self):
        return self.ctx.lib.lorakv_pool_allocated_elements(self.h)

    def reserved_bytes(self):
        return self.ctx.lib.lorakv_pool_reserved_bytes(self.h)

    def page_table(self, which=KEY, agent=0):
        n = _i64()
        _check(self.ctx.lib.lorakv_pool_page_table(self.h, which, agent, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.int32)
        if n.value:
            _check(self.ctx.lib.lorakv_pool_page_table(self.h, which, agent,
                                                       out.ctypes.data_as(C.POINTER(C.c_int32)), n.value,
                                                       C.byref(n)))
        return out

    # fast paths --------------------------------------------------------------------------------
    def decode(self, adapters, layer_begin, layer_end, agent_ids, n_q_heads, q, out=None):
        """q: [layers][n_batch][n_q_local*d] float32 host array -> same-shaped output."""
        q = np.ascontiguousarray(q, dtype=np.float32)
        ids = np.ascontiguousarray(agent_ids, dtype=np.int32)
        if out is None:
            out = np.zeros_like(q)
        _check(self.ctx.lib.lorakv_fla_decode_batched(
            self.h, adapters.h if adapters else None, layer_begin, layer_end,
            ids.ctypes.data_as(C.POINTER(C.c_int32)), len(ids), n_q_heads, q.ctypes.data_as(_vp),
            out.ctypes.data_as(_vp), HOST))
        return out

    def decode_device(self, adapters, layer_begin, layer_end, agent_ids, n_q_heads, q_dev, out_dev):
        ids = np.ascontiguousarray(agent_ids, dtype=np.int32)
        _check(self.ctx.lib.lorakv_fla_decode_batched(
            self.h, adapters.h if adapters else None, layer_begin, layer_end,
            ids.ctypes.data_as(C.POINTER(C.c_int32)), len(ids), n_q_heads, _vp(q_dev), _vp(out_dev), DEVICE))

    def decode_gather(self, adapters, gather, layer_begin, layer_end, agent_ids, n_q_heads, q=None, q_dev=None, out=None,
                      want_host=True):
        """This rank's shard of a decode step ending in the peer-memory output gather.  Returns (full host array or
        None, device pointer of the gathered rows)."""
        ids = np.ascontiguousarray(agent_ids, dtype=np.int32)
        n_layers = layer_end - layer_begin
        if q is not None:
            q = np.ascontiguousarray(q, dtype=np.float32)
            qp, kind = q.ctypes.data_as(_vp), HOST
        else:
            qp, kind = _vp(q_dev), DEVICE
        if want_host and out is None:
            out = np.zeros((n_layers, len(ids), gather.full_elems // (n_layers * len(ids))), dtype=np.float32)
        dev = _vp()
        _check(self.ctx.lib.lorakv_fla_decode_batched_gather(
            self.h, adapters.h if adapters else None, gather.h, layer_begin, layer_end,
            ids.ctypes.data_as(C.POINTER(C.c_int32)), len(ids), n_q_heads, qp, kind,
            out.ctypes.data_as(_vp) if want_host else None, C.byref(dev)))
        return (out if want_host else None), dev.value

    def prefill(self, adapters, layer, agent, n_q_heads, q, query_offset):
        q = np.ascontiguousarray(q, dtype=np.float32)
        out = np.zeros_like(q)
        _check(self.ctx.lib.lorakv_fla_prefill(self.h, adapters.h if adapters else None, layer, agent,
                                               n_q_heads, q.ctypes.data_as(_vp), q.shape[0], query_offset,
                                               out.ctypes.data_as(_vp), HOST))
        return out

    def step_layer(self, proj, adapters, layer, agent, row_begin, x, n_q_heads, rope=True):
        """One decode layer-step (projections + appends + attention) on HOST rows x; returns (q rows, attention output)."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        group = n_q_heads // self.dims.n_kv_heads
        n_kv_local = self.dims.n_kv_local or self.dims.n_kv_heads
        dq = group * n_kv_local * self.dims.d_head
        q = np.zeros((x.shape[0], dq), dtype=np.float32)
        out = np.zeros_like(q)
        _check(self.ctx.lib.lorakv_step_layer(self.h, proj.h, adapters.h if adapters else None, layer, agent, row_begin,
                                              x.ctypes.data_as(_vp), x.shape[0], x.shape[1], 1 if rope else 0, n_q_heads,
                                              q.ctypes.data_as(_vp), out.ctypes.data_as(_vp), HOST))
        return q, out

    def step_layer_device(self, proj, adapters, layer, agent, row_begin, x_dev, n_rows, ld, n_q_heads, out_dev, q_dev=0, rope=True):
        _check(self.ctx.lib.lorakv_step_layer(self.h, proj.h, adapters.h if adapters else None, layer, agent, row_begin,
                                              _vp(x_dev), n_rows, ld, 1 if rope else 0, n_q_heads, _vp(q_dev) if q_dev else None,
                                              _vp(out_dev), DEVICE))

    def prefill_device(self, adapters, layer, agent, n_q_heads, q_dev, L_c, query_offset, out_dev):
        _check(self.ctx.lib.lorakv_fla_prefill(self.h, adapters.h if adapters else None, layer, agent,
                                               n_q_heads, _vp(q_dev), L_c, query_offset, _vp(out_dev), DEVICE))
