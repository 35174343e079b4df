"""TEST INFRASTRUCTURE ONLY -- the CPU oracle (see dm_oracle.c's header for what it computes).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2508_21287_b200``) never imports it and shares no code with it.

``match()`` is a ctypes binding over ``libdmoracle.so`` (plain C, built with gcc by
``__graft_entry__.build()`` or lazily here).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dm_oracle.c")
_LIB_PATH = os.path.join(_HERE, "libdmoracle.so")
_lib = None
_lock = threading.Lock()

ERRORS = {-1: "bad argument", -2: "vertex out of range", -3: "self-loop",
          -4: "pattern disconnected", -5: "out of memory"}


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle error {code}: {ERRORS.get(code, '?')}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile libdmoracle.so with gcc (plain C11 + pthreads)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", "-pthread",
                               _SRC, "-o", tmp])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB_PATH)
            lib.oracle_match.restype = ctypes.c_int
            lib.oracle_match.argtypes = [
                ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int32,
                ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64),
                ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_double),
                ctypes.POINTER(ctypes.c_int), ctypes.c_void_p]
            lib.oracle_free.argtypes = [ctypes.c_void_p]
            lib.oracle_free.restype = None
            _lib = lib
    return _lib


class OracleResult:
    __slots__ = ("count", "rows", "seconds", "threads", "order")

    def __init__(self, count, rows, seconds, threads, order):
        self.count, self.rows, self.seconds, self.threads, self.order = count, rows, seconds, threads, order


def match(n: int, edges, k: int, p_edges, *, induced: bool = False, table: bool = True,
          drop_self_loops: bool = False, roots: tuple[int, int] | None = None,
          threads: int | None = None) -> OracleResult:
    """All embeddings of pattern (k, p_edges) in data graph (n, edges).

    Returns OracleResult(count, rows[count, k] int32 sorted lexicographically (or None),
    seconds, threads, order) -- ``order`` is the oracle's pattern order pi; ``roots`` restricts
    f(order[0]) to [roots[0], roots[1]).
    """
    lib = _load()
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
    pe = np.ascontiguousarray(np.asarray(p_edges, dtype=np.int32).reshape(-1, 2))
    if threads is None:
        threads = os.cpu_count() or 1
    rb, re_ = (0, -1) if roots is None else roots
    cnt = ctypes.c_uint64(0)
    rows_p = ctypes.c_void_p(None)
    secs = ctypes.c_double(0.0)
    used = ctypes.c_int(0)
    order = np.zeros(max(k, 1), dtype=np.int32)
    rc = lib.oracle_match(n, e.ctypes.data if e.size else None, e.shape[0], int(drop_self_loops),
                          k, pe.ctypes.data if pe.size else None, pe.shape[0], int(induced),
                          rb, re_, int(threads), int(table), ctypes.byref(cnt),
                          ctypes.byref(rows_p), ctypes.byref(secs), ctypes.byref(used),
                          order.ctypes.data)
    if rc != 0:
        raise OracleError(rc)
    rows = None
    if table:
        c = int(cnt.value)
        if c and rows_p.value:
            buf = (ctypes.c_int32 * (c * k)).from_address(rows_p.value)
            rows = np.frombuffer(buf, dtype=np.int32).reshape(c, k).copy()
        else:
            rows = np.zeros((0, k), dtype=np.int32)
        if rows_p.value:
            lib.oracle_free(rows_p)
    return OracleResult(int(cnt.value), rows, float(secs.value), int(used.value), order[:k].copy())
