"""TEST/BASELINE INFRASTRUCTURE ONLY — ctypes wrapper of oracle/_ref/libsfref.so,
the unmodified reference library (/root/reference/proj/src) plus ref_shim.cpp.

Available only where the library was built (``make -C oracle ref`` here, where
/root/reference exists; the built .so travels to the GPU box with the repo
snapshot). Callers must handle ``available() == False``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libsfref.so")
KIND = {np.dtype(np.int32): 0, np.dtype(np.int64): 1, np.dtype(np.float64): 2, np.dtype(np.uint8): 3}
OPS = {"replace": 0, "sum": 1, "prod": 2, "max": 3, "min": 4, "land": 5, "lor": 6, "band": 7,
       "bor": 8}
OPKIND = {"bcast": 0, "reduce": 1, "fetch_and_op": 2, "gather": 3, "scatter": 4}

_lib = None


def available() -> bool:
    return os.path.exists(LIB)


def _load():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference library not built at {LIB} (make -C oracle ref)")
        lib = C.CDLL(LIB)
        V, I, I64 = C.c_void_p, C.c_int, C.c_int64
        G = [I, V, V, V, V, V]
        lib.sfref_run.argtypes = G + [I, I, I64, I, I, I, C.c_uint64, V, V, V]
        lib.sfref_two_sided.argtypes = G + [V, V]
        lib.sfref_time_bcast_reduce.argtypes = G + [I, I, V]
        lib.sfref_last_error.restype = C.c_char_p
        lib.sfref_rng.argtypes = [C.c_uint64, I64, V, C.c_uint64, V]
        lib.sfref_random_graph.argtypes = [C.c_uint64, I, I64, V, I64]
        lib.sfref_spmv.argtypes = [I, I64, V, V, V, I, I, V, V]
        _lib = lib
    return _lib


class _Graph:
    """Keeps the per-rank arrays alive and exposes pointer tables."""

    def __init__(self, specs):
        self.n = len(specs)
        self.nroots = np.array([int(s.nroots) for s in specs], np.int64)
        self.nleaves = np.array([int(s.nleaves) for s in specs], np.int64)
        self.keep = []
        self.local = (C.c_void_p * self.n)()
        self.rr = (C.c_void_p * self.n)()
        self.ro = (C.c_void_p * self.n)()
        for r, s in enumerate(specs):
            rr = np.ascontiguousarray(np.asarray(s.remote_rank, np.int32))
            ro = np.ascontiguousarray(np.asarray(s.remote_off, np.int64))
            self.keep += [rr, ro]
            self.rr[r] = rr.ctypes.data if rr.size else None
            self.ro[r] = ro.ctypes.data if ro.size else None
            if s.local is not None:
                lo = np.ascontiguousarray(np.asarray(s.local, np.int64))
                self.keep.append(lo)
                self.local[r] = lo.ctypes.data if lo.size else None
            else:
                self.local[r] = None

    def args(self):
        return [self.n, self.nroots.ctypes.data, self.nleaves.ctypes.data, self.local, self.rr,
                self.ro]


def _ptrs(arrs):
    t = (C.c_void_p * max(1, len(arrs)))()
    for i, a in enumerate(arrs):
        t[i] = a.ctypes.data if a is not None and a.size else None
    return t


def run(specs, opkind: str, a, b, c=None, op: str = "replace", blocklen: int = 1,
        deterministic: bool = True, force_remote: bool = False, seed: int = 1):
    """Run one op on the reference's distributed CPU path; returns the in/out arrays (copies)."""
    g = _Graph(specs)
    a = [np.array(x, copy=True) for x in a]
    b = [np.array(x, copy=True) for x in b]
    c = [np.array(x, copy=True) for x in c] if c is not None else None
    kind = KIND[np.dtype((a if opkind in ("bcast", "fetch_and_op", "scatter") else b)[0].dtype)]
    rc = _load().sfref_run(*g.args(), OPKIND[opkind], kind, blocklen, OPS[op],
                           int(deterministic), int(force_remote), seed, _ptrs(a), _ptrs(b),
                           _ptrs(c) if c is not None else None)
    if rc != 0:
        raise RuntimeError(_load().sfref_last_error().decode())
    return a, b, c


def two_sided(specs):
    g = _Graph(specs)
    outs = [np.zeros(8 + 4 * int(g.nleaves.sum() + g.nroots.sum()) + 64, np.int64) for _ in specs]
    cap = np.array([o.size for o in outs], np.int64)
    rc = _load().sfref_two_sided(*g.args(), _ptrs(outs), cap.ctypes.data)
    if rc != 0:
        raise RuntimeError(_load().sfref_last_error().decode())
    res = []
    for o in outs:
        p = 0
        parts = []
        for _ in range(2):
            ng = int(o[p]); p += 1
            gs = []
            for _ in range(ng):
                rank, n = int(o[p]), int(o[p + 1]); p += 2
                gs.append((rank, o[p:p + n].tolist())); p += n
            parts.append(gs)
        res.append(tuple(parts))
    return res


def time_bcast_reduce(specs, steps: int, warmup: int) -> dict:
    g = _Graph(specs)
    out = np.zeros(4, np.float64)
    rc = _load().sfref_time_bcast_reduce(*g.args(), steps, warmup, out.ctypes.data)
    if rc != 0:
        raise RuntimeError(_load().sfref_last_error().decode())
    return {"setup_s": float(out[0]), "us_per_step": float(out[1]), "bcast_us": float(out[2]),
            "reduce_us": float(out[3])}


def rng(seed: int, n: int, salt: int = 0):
    out = np.zeros(n, np.uint64)
    mixed = np.zeros(1, np.uint64)
    _load().sfref_rng(seed, n, out.ctypes.data, salt, mixed.ctypes.data)
    return out, int(mixed[0])


def random_graph(seed: int, nranks: int, max_vertices: int):
    """The reference's random_graph_specs as (nroots, nleaves, local|None, ranks, offs) per rank."""
    cap = nranks * (3 + 4 * (max_vertices + 1)) + 16
    out = np.zeros(cap, np.int64)
    n = _load().sfref_random_graph(seed, nranks, max_vertices, out.ctypes.data, cap)
    if n < 0:
        raise RuntimeError(_load().sfref_last_error().decode())
    res, p = [], 0
    for _ in range(nranks):
        nroots, nleaves, has_local = int(out[p]), int(out[p + 1]), int(out[p + 2]); p += 3
        local = None
        if has_local:
            local = out[p:p + nleaves].copy(); p += nleaves
        pairs = out[p:p + 2 * nleaves].reshape(-1, 2); p += 2 * nleaves
        res.append((nroots, nleaves, local, pairs[:, 0].astype(np.int32).copy(), pairs[:, 1].copy()))
    return res


def time_op(specs, opkind: str, dtype: str, op: str, steps: int, warmup: int = 1) -> dict:
    """Mean microseconds per call of one operation on the reference CPU path."""
    lib = _load()
    if not getattr(lib, "_time_op_typed", False):
        V, I = C.c_void_p, C.c_int
        lib.sfref_time_op.argtypes = [I, V, V, V, V, V, I, I, I, I, I, V]
        lib._time_op_typed = True
    g = _Graph(specs)
    out = np.zeros(2, np.float64)
    kind = {"int32": 0, "int64": 1, "float64": 2}[dtype]
    rc = lib.sfref_time_op(*g.args(), OPKIND[opkind], kind, OPS[op], steps, warmup, out.ctypes.data)
    if rc != 0:
        raise RuntimeError(lib.sfref_last_error().decode())
    return {"setup_s": float(out[0]), "us_per_call": float(out[1])}


def pingpong(min_bytes: int, max_bytes: int, iters: int = 50, warmup: int = 5) -> list[dict]:
    """The reference's own 2-rank ping-pong benchmark (bench.cpp:24-100):
    sizes x4 from min_bytes; half round trip median / min in microseconds."""
    lib = _load()
    if not getattr(lib, "_pingpong_typed", False):
        lib.sfref_pingpong.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_int]
        lib._pingpong_typed = True
    out = np.zeros(3 * 64, np.float64)
    k = lib.sfref_pingpong(min_bytes, max_bytes, iters, warmup, out.ctypes.data, 64)
    if k < 0:
        raise RuntimeError(lib.sfref_last_error().decode())
    return [{"bytes": int(out[3 * i]), "median_us": float(out[3 * i + 1]), "min_us": float(out[3 * i + 2])}
            for i in range(k)]


def spmv(nranks: int, rowptr, colind, vals, x, transpose: bool = False) -> np.ndarray:
    """The reference's distributed spmv / spmv_transpose (spmv.hpp:147-169)
    over `nranks` rank threads with contiguous layouts, as selfcheck.cpp's
    spmv_trial runs it; returns the concatenated y."""
    lib = _load()
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    colind = np.ascontiguousarray(colind, np.int64)
    vals = np.ascontiguousarray(vals)
    x = np.ascontiguousarray(x, vals.dtype)
    n = len(rowptr) - 1
    y = np.zeros(n, vals.dtype)
    rc = lib.sfref_spmv(nranks, n, rowptr.ctypes.data, colind.ctypes.data, vals.ctypes.data,
                        KIND[vals.dtype], int(transpose), x.ctypes.data, y.ctypes.data)
    if rc != 0:
        raise RuntimeError(lib.sfref_last_error().decode())
    return y
