"""ctypes wrapper of oracle/hc_oracle.c — TEST INFRASTRUCTURE ONLY.

Argument marshalling only; every step of the method is in the C file, which
follows PAPER.md Fig. 3 / Fig. 5 line by line.  Host threading helpers split
the text into disjoint ranges (brute force: ranges of start positions; HC:
ranges of window ends, SURVEY.md 8(a).2 / DESIGN.md R11) and run the plain C
routine on each range in a thread (ctypes releases the GIL).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

i64 = C.c_int64
u64 = C.c_uint64
P8 = C.POINTER(C.c_uint8)
P64 = C.POINTER(C.c_int64)
PU64 = C.POINTER(C.c_uint64)


def lib_path() -> str:
    return _LIB


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no fast-math: integer code)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-shared",
                               "-fPIC", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = C.CDLL(_LIB)
            lib.or_shift.argtypes = [C.c_int, C.c_int]
            lib.or_shift.restype = C.c_int
            lib.or_hash.argtypes = [P8, i64, C.c_int, C.c_int, u64]
            lib.or_hash.restype = u64
            lib.or_link_hash.argtypes = [u64, C.c_int]
            lib.or_link_hash.restype = u64
            lib.or_preprocess.argtypes = [P8, i64, C.c_int, C.c_int, C.c_int, PU64, PU64,
                                          P64, P64]
            lib.or_preprocess.restype = C.c_int
            lib.or_hc_search.argtypes = [P8, i64, P8, i64, C.c_int, C.c_int, C.c_int, PU64,
                                         u64, i64, i64, P64, i64, P64]
            lib.or_hc_search.restype = i64
            lib.or_shc_search.argtypes = [P8, i64, P8, i64, C.c_int, C.c_int, C.c_int, PU64,
                                          u64, P64, i64, P64]
            lib.or_shc_search.restype = i64
            lib.or_brute.argtypes = [P8, i64, P8, i64, i64, i64, P64, i64]
            lib.or_brute.restype = i64
            _lib = lib
    return _lib


def _u8(a) -> np.ndarray:
    if isinstance(a, np.ndarray):
        assert a.dtype == np.uint8
        return np.ascontiguousarray(a)
    if isinstance(a, str):
        a = a.encode("latin-1")
    return np.frombuffer(bytes(a), dtype=np.uint8)


def _p8(a: np.ndarray):
    return a.ctypes.data_as(P8)


def shift(alpha: int, q: int) -> int:
    return _load().or_shift(alpha, q)


def hash_qgram(x, p: int, q: int, s: int, mask: int) -> int:
    xa = _u8(x)
    assert q - 1 <= p < len(xa)
    return int(_load().or_hash(_p8(xa), p, q, s, mask))


def link_hash(v: int, w: int) -> int:
    return int(_load().or_link_hash(v, w))


@dataclass
class Table:
    F: np.ndarray          # uint64[2^alpha], low w bits used
    s: int
    mask: int
    hv: int
    q: int
    alpha: int
    w: int
    trace: list = field(default_factory=list)


def preprocess(x, q: int, alpha: int, w: int = 32, trace: bool = False) -> Table:
    """Fig. 3 Preprocessing."""
    xa = _u8(x)
    m = len(xa)
    F = np.zeros(1 << alpha, dtype=np.uint64)
    hv = u64(0)
    tr = np.zeros(m + q + 1, dtype=np.int64)
    nt = i64(0)
    rc = _load().or_preprocess(_p8(xa), m, q, alpha, w, F.ctypes.data_as(PU64), C.byref(hv),
                               tr.ctypes.data_as(P64) if trace else None, C.byref(nt))
    if rc != 0:
        raise ValueError(f"invalid parameters m={m} q={q} alpha={alpha} w={w}")
    return Table(F=F, s=alpha // q, mask=(1 << alpha) - 1, hv=int(hv.value), q=q,
                 alpha=alpha, w=w, trace=tr[:nt.value].tolist() if trace else [])


@dataclass
class Metrics:
    windows: int = 0
    qgram_hashes: int = 0
    link_checks: int = 0
    verifications: int = 0
    hv_rejections: int = 0
    completed_walks: int = 0
    min_shift: int = 0
    max_shift: int = 0

    @classmethod
    def from_array(cls, a):
        return cls(*[int(v) for v in a])


def _run_positions(call, cap_hint: int):
    """Call `call(out_ptr, max_out)` -> count; re-run with exact capacity if needed."""
    cap = max(1, cap_hint)
    out = np.empty(cap, dtype=np.int64)
    cnt = call(out, cap)
    if cnt > cap:
        out = np.empty(cnt, dtype=np.int64)
        cnt2 = call(out, cnt)
        assert cnt2 == cnt
    return out[:cnt].copy()


def hc_search(x, y, q: int, alpha: int, w: int = 32, table: Table | None = None,
              start: int | None = None, stop: int | None = None, metrics: bool = False,
              cap_hint: int = 1 << 16):
    """Fig. 5 HC searching phase; returns int64 positions ascending (and Metrics)."""
    xa, ya = _u8(x), _u8(y)
    m, n = len(xa), len(ya)
    t = table if table is not None else preprocess(xa, q, alpha, w)
    a = m - 1 if start is None else start
    b = n if stop is None else stop
    met = np.zeros(8, dtype=np.int64)
    lib = _load()

    def call(out, cap):
        met[:] = 0
        return lib.or_hc_search(_p8(xa), m, _p8(ya), n, q, alpha, w,
                                t.F.ctypes.data_as(PU64), t.hv, a, b,
                                out.ctypes.data_as(P64), cap,
                                met.ctypes.data_as(P64) if metrics else None)

    pos = _run_positions(call, cap_hint) if n >= m else np.zeros(0, dtype=np.int64)
    if metrics:
        return pos, Metrics.from_array(met)
    return pos


def hc_search_segmented(x, y, q: int, alpha: int, seg: int, w: int = 32):
    """HC run independently on segments of window ends [a_k, a_k + seg) with
    a_k = m-1 + k*seg, results concatenated (SURVEY.md 8(a).2 argument)."""
    xa, ya = _u8(x), _u8(y)
    m, n = len(xa), len(ya)
    if n < m:
        return np.zeros(0, dtype=np.int64)
    t = preprocess(xa, q, alpha, w)
    parts = []
    a = m - 1
    while a < n:
        b = min(a + seg, n)
        parts.append(hc_search(xa, ya, q, alpha, w, table=t, start=a, stop=b))
        a = b
    return np.concatenate(parts)


def shc_search(x, y, q: int, alpha: int, w: int = 32, metrics: bool = False,
               cap_hint: int = 1 << 16):
    """Fig. 5 SHC on a copy of y with m bytes of slack."""
    xa, ya = _u8(x), _u8(y)
    m, n = len(xa), len(ya)
    t = preprocess(xa, q, alpha, w)
    buf = np.zeros(n + m, dtype=np.uint8)
    buf[:n] = ya
    met = np.zeros(8, dtype=np.int64)
    lib = _load()

    def call(out, cap):
        met[:] = 0
        return lib.or_shc_search(_p8(xa), m, _p8(buf), n, q, alpha, w,
                                 t.F.ctypes.data_as(PU64), t.hv,
                                 out.ctypes.data_as(P64), cap,
                                 met.ctypes.data_as(P64) if metrics else None)

    pos = _run_positions(call, cap_hint) if n >= m else np.zeros(0, dtype=np.int64)
    assert np.array_equal(buf[:n], ya), "SHC must not modify y[0..n-1]"
    if metrics:
        return pos, Metrics.from_array(met)
    return pos


def brute(x, y, s0: int = 0, s1: int | None = None, cap_hint: int = 1 << 16):
    """O1: every s in [s0, s1) with y[s..s+m-1] == x."""
    xa, ya = _u8(x), _u8(y)
    m, n = len(xa), len(ya)
    if m < 1:
        raise ValueError("empty pattern")
    if n < m:
        return np.zeros(0, dtype=np.int64)
    hi = n - m + 1 if s1 is None else s1
    lib = _load()

    def call(out, cap):
        return lib.or_brute(_p8(xa), m, _p8(ya), n, s0, hi, out.ctypes.data_as(P64), cap)

    return _run_positions(call, cap_hint)


def brute_threaded(x, y, threads: int | None = None):
    """O1 over `threads` disjoint ranges of start positions."""
    xa, ya = _u8(x), _u8(y)
    m, n = len(xa), len(ya)
    if n < m:
        return np.zeros(0, dtype=np.int64)
    T = threads or os.cpu_count() or 1
    total = n - m + 1
    bounds = [total * k // T for k in range(T + 1)]
    with ThreadPoolExecutor(T) as ex:
        parts = list(ex.map(lambda k: brute(xa, ya, bounds[k], bounds[k + 1]), range(T)))
    return np.concatenate(parts)


def hc_threaded(x, y, q: int, alpha: int, w: int = 32, threads: int | None = None,
                table: Table | None = None):
    """O2 over `threads` disjoint ranges of window ends [m-1, n) (exact by the
    segment argument, R11)."""
    xa, ya = _u8(x), _u8(y)
    m, n = len(xa), len(ya)
    if n < m:
        return np.zeros(0, dtype=np.int64)
    t = table if table is not None else preprocess(xa, q, alpha, w)
    T = threads or os.cpu_count() or 1
    ends = n - (m - 1)
    bounds = [m - 1 + ends * k // T for k in range(T + 1)]
    with ThreadPoolExecutor(T) as ex:
        parts = list(ex.map(lambda k: hc_search(xa, ya, q, alpha, w, table=t,
                                                start=bounds[k], stop=bounds[k + 1]),
                            range(T)))
    return np.concatenate(parts)
