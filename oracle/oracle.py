"""TEST INFRASTRUCTURE ONLY — Python wrapper of the C oracle (sf_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module; the product package never does. Every function takes the
global graph as a list of per-rank GraphSpec-like objects (nroots, nleaves,
local, remote_rank, remote_off) and per-rank numpy arrays, and returns fresh
per-rank arrays — the restated semantics of /root/reference/proj/src/oracle.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "sf_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

KIND = {np.dtype(np.int32): 0, np.dtype(np.int64): 1, np.dtype(np.float64): 2, np.dtype(np.uint8): 3}
OPS = {"replace": 0, "sum": 1, "prod": 2, "max": 3, "min": 4, "land": 5, "lor": 6, "band": 7,
       "bor": 8}

_lib = None


def build() -> str:
    if (not os.path.exists(LIB)) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-Wall", "-o", LIB + ".tmp", SRC],
                       check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(LIB)
        V, I64, I = C.c_void_p, C.c_int64, C.c_int
        E = [I64, V, V, V, V]
        lib.oracle_bcast.argtypes = E + [I, I64, I, V, V]
        lib.oracle_reduce.argtypes = E + [I, I64, I, V, V]
        lib.oracle_fetch_and_op.argtypes = E + [I, I64, I, V, V, V]
        lib.oracle_degrees.argtypes = [I64, V, V, V]
        lib.oracle_gather.argtypes = E + [I, V, I, I64, V, V]
        lib.oracle_scatter.argtypes = E + [I, V, I, I64, V, V]
        _lib = lib
    return _lib


def edges(specs) -> tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
    """GlobalGraph::from_specs (oracle.cpp:12-26): leaf-rank major, ordinal order."""
    rr, ro, lr, li = [], [], [], []
    for rank, s in enumerate(specs):
        n = int(s.nleaves)
        local = np.arange(n, dtype=np.int64) if s.local is None else np.asarray(s.local, np.int64)
        rr.append(np.asarray(s.remote_rank, np.int32)[:n])
        ro.append(np.asarray(s.remote_off, np.int64)[:n])
        lr.append(np.full(n, rank, np.int32))
        li.append(local[:n])
    cat = lambda xs, dt: np.ascontiguousarray(np.concatenate(xs).astype(dt)) if xs else np.zeros(0, dt)
    return cat(rr, np.int32), cat(ro, np.int64), cat(lr, np.int32), cat(li, np.int64)


def _ptrs(arrays) -> C.Array:
    arr = (C.c_void_p * max(1, len(arrays)))()
    for i, a in enumerate(arrays):
        arr[i] = a.ctypes.data if a.size else None
    return arr


def _e(specs):
    rr, ro, lr, li = edges(specs)
    return (rr, ro, lr, li), [rr.size, rr.ctypes.data, ro.ctypes.data, lr.ctypes.data,
                              li.ctypes.data]


def _copy(xs):
    return [np.ascontiguousarray(np.array(x, copy=True)) for x in xs]


def _kind(arrs, bl):
    dt = arrs[0].dtype
    return KIND[np.dtype(dt)]


def bcast(specs, rootdata, leafdata, op="replace", blocklen=1):
    keep, e = _e(specs)
    roots, leaves = _copy(rootdata), _copy(leafdata)
    k = _kind(roots, blocklen)
    _load().oracle_bcast(*e, k, blocklen, OPS[op], _ptrs(roots), _ptrs(leaves))
    return leaves


def reduce(specs, leafdata, rootdata, op="sum", blocklen=1):
    keep, e = _e(specs)
    leaves, roots = _copy(leafdata), _copy(rootdata)
    k = _kind(roots, blocklen)
    _load().oracle_reduce(*e, k, blocklen, OPS[op], _ptrs(leaves), _ptrs(roots))
    return roots


def fetch_and_op(specs, rootdata, leafdata, leafupdate, op="sum", blocklen=1):
    keep, e = _e(specs)
    roots, leaves, upd = _copy(rootdata), _copy(leafdata), _copy(leafupdate)
    k = _kind(roots, blocklen)
    rc = _load().oracle_fetch_and_op(*e, k, blocklen, OPS[op], _ptrs(roots),
                                     _ptrs(leaves), _ptrs(upd))
    if rc != 0:
        raise ValueError("oracle fetch_and_op: replace/bytes have no fetch semantics")
    return roots, upd


def degrees(specs):
    keep, e = _e(specs)
    deg = [np.zeros(int(s.nroots), np.int64) for s in specs]
    _load().oracle_degrees(e[0], e[1], e[2], _ptrs(deg))
    return deg


def gather(specs, leafdata, blocklen=1, fill=None):
    keep, e = _e(specs)
    deg = degrees(specs)
    leaves = _copy(leafdata)
    dt = leaves[0].dtype
    multi = [np.full(int(d.sum()) * blocklen, fill if fill is not None else 0, dtype=dt) for d in deg]
    nroots = np.array([int(s.nroots) for s in specs], np.int64)
    _load().oracle_gather(*e, len(specs), nroots.ctypes.data, KIND[np.dtype(dt)],
                          blocklen, _ptrs(leaves), _ptrs(multi))
    return multi


def scatter(specs, multiroot, leafdata, blocklen=1):
    keep, e = _e(specs)
    multi, leaves = _copy(multiroot), _copy(leafdata)
    nroots = np.array([int(s.nroots) for s in specs], np.int64)
    _load().oracle_scatter(*e, len(specs), nroots.ctypes.data,
                           KIND[np.dtype(leaves[0].dtype)], blocklen, _ptrs(multi),
                           _ptrs(leaves))
    return leaves


# ------------------------------------------------------------------ SpMV
def spmv(glob, layout, x, transpose: bool = False):
    """The reference's distributed SpMV (spmv.hpp:149-169) restated
    sequentially: split_matrix per rank, then the Csr loops in the reference
    order (diag product, then += off-diagonal product; for the transpose
    A^T x into zeros, B^T x into zeros, Reduce(SUM) into the owners in
    ascending rank order, ops.cpp:364,372-376). Pure-Python loops: test-sized
    matrices only. `glob` is a paper_2102_13018_b200.spmv.Csr."""
    import numpy as np

    from paper_2102_13018_b200 import spmv as S

    P = layout.nranks()
    ms = [S.split_matrix(glob, layout, layout, r) for r in range(P)]
    ys = []
    if not transpose:
        for r, m in enumerate(ms):
            xo = x[layout.begin(r):layout.end(r)]
            y = m.diag.multiply(xo)
            m.offdiag.multiply_add(x[m.garray], y)
            ys.append(y)
        return np.concatenate(ys)
    lvecs = []
    for r, m in enumerate(ms):
        xo = x[layout.begin(r):layout.end(r)]
        y = np.zeros(layout.local_size(r), dtype=glob.vals.dtype)
        m.diag.multiply_transpose_add(xo, y)
        lv = np.zeros(len(m.garray), dtype=glob.vals.dtype)
        m.offdiag.multiply_transpose_add(xo, lv)
        ys.append(y)
        lvecs.append(lv)
    with np.errstate(over="ignore"):
        for r in range(P):  # owners fold remote contributions rank by rank
            for s in range(P):
                if s == r:
                    continue
                g = ms[s].garray
                mine = (g >= layout.begin(r)) & (g < layout.end(r))
                for gi, v in zip(g[mine], lvecs[s][mine]):
                    ys[r][gi - layout.begin(r)] = ys[r][gi - layout.begin(r)] + v
    return np.concatenate(ys)
