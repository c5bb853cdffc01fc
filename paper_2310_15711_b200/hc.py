"""Thin ctypes binding of libhc.so (the C-ABI of include/hc.h).

Argument marshalling only: every step of the search runs in the library's
CUDA kernels.  PyTorch supplies device memory and streams.  There is no CPU
fallback: if libhc.so is missing this module raises ImportError.

    from paper_2310_15711_b200 import hc
    h = hc.prepare(b"ACGTACGT", q=4, alpha=12)
    pos = hc.search(h, y)            # y: torch.uint8 CUDA tensor -> torch.int64 CUDA tensor
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# HC_LIB: another build of the same library (A/B experiments in tools/)
LIB_PATH = os.environ.get("HC_LIB") or os.path.join(_HERE, "libhc.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2310_15711_b200.build` "
                      "(or __graft_entry__.build()); there is no CPU fallback")

_lib = C.CDLL(LIB_PATH)

HC_OK, HC_EINVAL, HC_ETOOSHORT, HC_EALPHA, HC_ENOMEM, HC_ECUDA, HC_ETOOLONG, HC_ENODEV = (
    0, -1, -2, -3, -4, -5, -6, -7)
PATH_AUTO, PATH_STAGED, PATH_GATHER, PATH_STREAM, PATH_SHC, PATH_SCAN = 0, 1, 2, 3, 4, 5
WORD_BITS = 32

# the symbols include/hc.h declares (tests check every one is exported)
EXPORTS = ("hc_prepare", "hc_last_error", "hc_strerror", "hc_search", "hc_search_ex",
           "hc_search_batch", "hc_prepare_batch", "hc_search_host", "hc_search_batch_host", "hc_destroy", "hc_table", "hc_build_table",
           "hc_version")


class Opts(C.Structure):
    _fields_ = [("path", C.c_int), ("tile_bytes", C.c_int), ("stages", C.c_int),
                ("seg_per_lane", C.c_int), ("max_ctas", C.c_int), ("time_kernel", C.c_int),
                ("ctas_per_sm", C.c_int), ("debug", C.c_int), ("tma_chunk", C.c_int),
                ("trace", C.c_void_p), ("trace_tiles", C.c_int), ("surv_warps", C.c_int),
                ("block_warps", C.c_int), ("no_multi", C.c_int)]


class Stats(C.Structure):
    _fields_ = [("path", C.c_int), ("grid", C.c_int), ("block", C.c_int),
                ("smem_bytes", C.c_int), ("tiles", C.c_int64), ("launches", C.c_int),
                ("reruns", C.c_int), ("kernel_ms", C.c_float), ("dbg", C.c_uint32 * 2),
                ("search_ms", C.c_float)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_}
        d["dbg"] = list(self.dbg)
        return d


P8 = C.POINTER(C.c_uint8)
_lib.hc_prepare.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int]
_lib.hc_prepare.restype = C.c_void_p
_lib.hc_last_error.argtypes = []
_lib.hc_last_error.restype = C.c_int
_lib.hc_strerror.argtypes = [C.c_int]
_lib.hc_strerror.restype = C.c_char_p
_lib.hc_search.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_void_p]
_lib.hc_search.restype = C.c_int64
_lib.hc_search_ex.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t,
                              C.c_void_p, C.POINTER(Opts), C.POINTER(Stats)]
_lib.hc_search_ex.restype = C.c_int64
_lib.hc_search_batch.argtypes = [C.POINTER(C.c_void_p), C.c_size_t, C.c_void_p, C.c_size_t,
                                 C.POINTER(C.c_int64), C.POINTER(C.c_void_p),
                                 C.POINTER(C.c_size_t), C.c_void_p, C.POINTER(Opts),
                                 C.POINTER(Stats)]
_lib.hc_search_batch.restype = C.c_int
_lib.hc_prepare_batch.argtypes = [C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.c_size_t, C.c_int,
                                  C.c_int, C.POINTER(C.c_void_p)]
_lib.hc_prepare_batch.restype = C.c_int
_lib.hc_search_host.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t,
                                C.c_void_p]
_lib.hc_search_host.restype = C.c_int64
_lib.hc_search_batch_host.argtypes = [C.POINTER(C.c_void_p), C.c_size_t, C.c_void_p, C.c_size_t,
                                      C.POINTER(C.c_int64), C.POINTER(C.c_void_p),
                                      C.POINTER(C.c_size_t), C.c_void_p, C.POINTER(Opts),
                                      C.POINTER(Stats)]
_lib.hc_search_batch_host.restype = C.c_int
_lib.hc_destroy.argtypes = [C.c_void_p]
_lib.hc_destroy.restype = None
_lib.hc_table.argtypes = [C.c_void_p, C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_int),
                          C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_uint32)]
_lib.hc_table.restype = C.c_int
_lib.hc_build_table.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p,
                                C.POINTER(C.c_int), C.POINTER(C.c_uint32)]
_lib.hc_build_table.restype = C.c_int
_lib.hc_version.argtypes = []
_lib.hc_version.restype = C.c_char_p


class HCError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        super().__init__(f"{what}: {_lib.hc_strerror(code).decode()} ({code})")


def lib():
    return _lib


def version() -> str:
    return _lib.hc_version().decode()


def _bytes(x) -> np.ndarray:
    if isinstance(x, np.ndarray):
        return np.ascontiguousarray(x, dtype=np.uint8)
    if isinstance(x, str):
        x = x.encode("latin-1")
    return np.frombuffer(bytes(x), dtype=np.uint8)


def _stream_ptr(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


@dataclass
class Table:
    F: np.ndarray
    alpha: int
    s: int
    w: int
    hv: int


def build_table(x, q: int, alpha: int) -> Table:
    """Host-only Fig. 3 Preprocessing (no GPU needed): hc_build_table."""
    xa = _bytes(x)
    F = np.zeros(1 << alpha, dtype=np.uint32) if 1 <= alpha <= 15 else np.zeros(1, np.uint32)
    s = C.c_int(0)
    hv = C.c_uint32(0)
    rc = _lib.hc_build_table(xa.ctypes.data if len(xa) else None, len(xa), q, alpha,
                             F.ctypes.data, C.byref(s), C.byref(hv))
    if rc != HC_OK:
        raise HCError(rc, "hc_build_table")
    return Table(F=F, alpha=alpha, s=s.value, w=WORD_BITS, hv=hv.value)


class Handle:
    """Owns an hc_handle (Preprocessing of one pattern, resident on the device)."""

    def __init__(self, x, q: int, alpha: int):
        xa = _bytes(x)
        self.m, self.q, self.alpha = len(xa), q, alpha
        self.x = xa.tobytes()
        ptr = _lib.hc_prepare(xa.ctypes.data if len(xa) else None, len(xa), q, alpha)
        if not ptr:
            raise HCError(_lib.hc_last_error(), "hc_prepare")
        self._h = C.c_void_p(ptr)

    @property
    def ptr(self):
        return self._h

    def table(self) -> Table:
        Fp = C.POINTER(C.c_uint32)()
        a, s, w = C.c_int(), C.c_int(), C.c_int()
        hv = C.c_uint32()
        rc = _lib.hc_table(self._h, C.byref(Fp), C.byref(a), C.byref(s), C.byref(w), C.byref(hv))
        if rc != HC_OK:
            raise HCError(rc, "hc_table")
        F = np.ctypeslib.as_array(Fp, shape=(1 << a.value,)).copy()
        return Table(F=F, alpha=a.value, s=s.value, w=w.value, hv=hv.value)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.hc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def prepare(x, q: int, alpha: int) -> Handle:
    return Handle(x, q, alpha)


def prepare_batch(xs, q: int, alpha: int) -> list:
    """hc_prepare_batch: Preprocessing of every pattern in xs (same q, alpha) with one
    device allocation and one upload; returns one Handle per pattern."""
    arrs = [_bytes(x) for x in xs]
    P = len(arrs)
    if P == 0:
        return []
    ptrs = (C.c_void_p * P)(*[a.ctypes.data if len(a) else None for a in arrs])
    ms = (C.c_size_t * P)(*[len(a) for a in arrs])
    out = (C.c_void_p * P)()
    rc = _lib.hc_prepare_batch(ptrs, ms, P, q, alpha, out)
    if rc != HC_OK:
        raise HCError(int(rc), "hc_prepare_batch")
    hs = []
    for a, ptr in zip(arrs, out):
        h = Handle.__new__(Handle)
        h.m, h.q, h.alpha, h.x = len(a), q, alpha, a.tobytes()
        h._h = C.c_void_p(ptr)
        hs.append(h)
    return hs


def _opts(path=PATH_AUTO, tile_bytes=0, stages=0, seg_per_lane=0, max_ctas=0, time_kernel=0,
          ctas_per_sm=0, debug=0, tma_chunk=0, trace=0, trace_tiles=0, surv_warps=0,
          block_warps=0, no_multi=0):
    return Opts(path, tile_bytes, stages, seg_per_lane, max_ctas, int(time_kernel), ctas_per_sm,
                debug, tma_chunk, trace or None, trace_tiles, surv_warps, block_warps, int(no_multi))


def search_raw(h: Handle, y_ptr: int, n: int, pos_ptr: int | None, max_out: int,
               stream_ptr: int, opts: Opts | None = None, stats: Stats | None = None) -> int:
    """Direct hc_search_ex call on raw device pointers; returns the count (raises on error)."""
    cnt = _lib.hc_search_ex(h.ptr, C.c_void_p(y_ptr), n, C.c_void_p(pos_ptr) if pos_ptr else None,
                            max_out, C.c_void_p(stream_ptr),
                            C.byref(opts) if opts is not None else None,
                            C.byref(stats) if stats is not None else None)
    if cnt < 0:
        raise HCError(int(cnt), "hc_search_ex")
    return int(cnt)


def count(h: Handle, y, stream=None, **kw) -> int:
    """Number of occurrences only (pos_out = NULL)."""
    return search_raw(h, y.data_ptr(), y.numel(), None, 0, _stream_ptr(stream),
                      _opts(**kw) if kw else None)


def search(h: Handle, y, max_out: int | None = None, stream=None, stats: bool = False, **kw):
    """All (or the max_out smallest) occurrence positions of h's pattern in the uint8 CUDA
    tensor y, ascending, as an int64 CUDA tensor.  With max_out=None the result is exact:
    a first call with room for 2^16 positions is repeated with the exact count if needed."""
    import torch
    assert y.dtype == torch.uint8 and y.is_cuda and y.is_contiguous()
    n = y.numel()
    st = _stream_ptr(stream)
    o = _opts(**kw) if kw else None
    S = Stats() if stats else None
    if max_out is not None:
        out = torch.empty(max(int(max_out), 1), dtype=torch.int64, device=y.device)
        cnt = search_raw(h, y.data_ptr(), n, out.data_ptr(), int(max_out), st, o, S)
        res = out[:min(cnt, int(max_out))]
    else:
        guess = 1 << 16
        out = torch.empty(guess, dtype=torch.int64, device=y.device)
        cnt = search_raw(h, y.data_ptr(), n, out.data_ptr(), guess, st, o, S)
        if cnt > guess:
            out = torch.empty(cnt, dtype=torch.int64, device=y.device)
            cnt = search_raw(h, y.data_ptr(), n, out.data_ptr(), cnt, st, o, S)
        res = out[:cnt]
    return (res, S.as_dict()) if stats else res


def search_batch_raw(handles, y_ptr: int, n: int, pos_ptrs, max_outs, stream_ptr: int,
                     opts: Opts | None = None, stats: Stats | None = None) -> list[int]:
    """hc_search_batch on raw pointers: pos_ptrs / max_outs are per-pattern lists (or
    None for count only); returns the counts (raises on error)."""
    P = len(handles)
    hs = (C.c_void_p * P)(*[h.ptr.value for h in handles])
    counts = (C.c_int64 * P)()
    pp = (C.c_void_p * P)(*pos_ptrs) if pos_ptrs is not None else None
    mo = (C.c_size_t * P)(*max_outs) if max_outs is not None else None
    rc = _lib.hc_search_batch(hs, P, C.c_void_p(y_ptr), n, counts, pp, mo, C.c_void_p(stream_ptr),
                              C.byref(opts) if opts is not None else None,
                              C.byref(stats) if stats is not None else None)
    if rc != HC_OK:
        raise HCError(int(rc), "hc_search_batch")
    return list(counts)


def search_batch(handles, y, max_out: int | None = None, stream=None, stats: bool = False, **kw):
    """Searches every handle's pattern in the uint8 CUDA tensor y with one
    hc_search_batch call; returns a list of int64 CUDA tensors (as search() would).
    With max_out=None the results are exact (counts first, then the positions)."""
    import torch
    assert y.dtype == torch.uint8 and y.is_cuda and y.is_contiguous()
    n = y.numel()
    st = _stream_ptr(stream)
    o = _opts(**kw) if kw else None
    S = Stats() if stats else None
    if max_out is None:
        cnts = search_batch_raw(handles, y.data_ptr(), n, None, None, st, o, None)
        mos = [max(c, 1) for c in cnts]
    else:
        mos = [max(int(max_out), 1)] * len(handles)
    outs = [torch.empty(k, dtype=torch.int64, device=y.device) for k in mos]
    cnts = search_batch_raw(handles, y.data_ptr(), n, [t.data_ptr() for t in outs], mos, st, o, S)
    res = [t[:min(c, k)] for t, c, k in zip(outs, cnts, mos)]
    return (res, S.as_dict()) if stats else res


def search_host(h: Handle, y, max_out: int | None = None) -> np.ndarray:
    """hc_search_host: y is host memory (numpy uint8); returns numpy int64 positions."""
    ya = _bytes(y)
    n = len(ya)
    exact = max_out is None
    cap = max(0, min(n - h.m + 1, 1 << 20)) if exact else int(max_out)

    def call(cap):
        out = np.empty(max(cap, 1), dtype=np.int64)
        cnt = _lib.hc_search_host(h.ptr, ya.ctypes.data if n else None, n,
                                  out.ctypes.data if cap else None, cap, None)
        if cnt < 0:
            raise HCError(int(cnt), "hc_search_host")
        return int(cnt), out

    cnt, out = call(cap)
    if exact and cnt > cap:
        cap = cnt
        cnt, out = call(cap)
    return out[:min(cnt, cap)].copy()


def search_batch_host_raw(handles, y_ptr: int, n: int, pos_ptrs, max_outs, stream_ptr: int = 0,
                          opts: Opts | None = None, stats: Stats | None = None) -> list[int]:
    """hc_search_batch_host on raw HOST pointers (text and per-pattern int64 buffers)."""
    P = len(handles)
    hs = (C.c_void_p * P)(*[h.ptr.value for h in handles])
    counts = (C.c_int64 * P)()
    pp = (C.c_void_p * P)(*pos_ptrs) if pos_ptrs is not None else None
    mo = (C.c_size_t * P)(*max_outs) if max_outs is not None else None
    rc = _lib.hc_search_batch_host(hs, P, C.c_void_p(y_ptr) if n else None, n, counts, pp, mo,
                                   C.c_void_p(stream_ptr) if stream_ptr else None,
                                   C.byref(opts) if opts is not None else None,
                                   C.byref(stats) if stats is not None else None)
    if rc != HC_OK:
        raise HCError(int(rc), "hc_search_batch_host")
    return list(counts)


def search_batch_host(handles, y, max_out: int | None = None) -> list:
    """hc_search_batch_host: y is host memory (numpy uint8); returns numpy int64 positions
    per handle (exact when max_out is None: counts first, then the positions)."""
    ya = _bytes(y)
    n = len(ya)
    yp = ya.ctypes.data if n else 0
    if max_out is None:
        mos = [max(c, 1) for c in search_batch_host_raw(handles, yp, n, None, None)]
    else:
        mos = [max(int(max_out), 1)] * len(handles)
    outs = [np.empty(k, dtype=np.int64) for k in mos]
    cnts = search_batch_host_raw(handles, yp, n, [o.ctypes.data for o in outs], mos)
    return [o[:min(c, k)].copy() for o, c, k in zip(outs, cnts, mos)]
