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


def bcast_edges(edge_arrays, rootdata, leafdata, op="replace", blocklen=1):
    """oracle::bcast over an arbitrary edge list (rr, ro, lr, li) — e.g. a
    transposed graph where a leaf may have several roots (selfcheck.cpp:
    165-197 duality: GlobalGraph::transposed)."""
    rr, ro, lr, li = (np.ascontiguousarray(a) for a in edge_arrays)
    rr, lr = rr.astype(np.int32), lr.astype(np.int32)
    ro, li = ro.astype(np.int64), li.astype(np.int64)
    roots, leaves = _copy(rootdata), _copy(leafdata)
    k = _kind(roots, blocklen)
    _load().oracle_bcast(rr.size, rr.ctypes.data, ro.ctypes.data, lr.ctypes.data, li.ctypes.data,
                         k, blocklen, OPS[op], _ptrs(roots), _ptrs(leaves))
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
def _split(rowptr, colind, vals, starts, r):
    """split_matrix (spmv.hpp:95-127) restated: the diagonal block's rows as
    (local col, val) lists in stored order, the off-diagonal block's rows as
    (reduced col, val) lists in ascending global column order (Csr::
    from_triplets sorts each row by column, spmv.hpp:44-56), and garray."""
    r0, r1 = int(starts[r]), int(starts[r + 1])
    diag, off, ghost = [], [], set()
    for row in range(r0, r1):
        d, o = [], []
        for i in range(int(rowptr[row]), int(rowptr[row + 1])):
            c = int(colind[i])
            if r0 <= c < r1:
                d.append((c - r0, vals[i]))
            else:
                o.append((c, vals[i]))
                ghost.add(c)
        diag.append(sorted(d, key=lambda t: t[0]))
        off.append(sorted(o, key=lambda t: t[0]))
    garray = sorted(ghost)
    pos = {g: k for k, g in enumerate(garray)}
    off = [[(pos[c], v) for c, v in row] for row in off]
    return diag, off, np.array(garray, np.int64)


def spmv(glob, layout, x, transpose: bool = False):
    """The reference's distributed SpMV (spmv.hpp:149-169) restated
    sequentially from the global CSR (``glob.rowptr/colind/vals``) and the
    row layout (``layout.starts``): per rank the diagonal product, then +=
    the off-diagonal product over the gathered ghosts; for the transpose
    A^T x and B^T x into zeros, then Reduce(SUM) of the ghost partial sums
    into their owners in ascending rank order (ops.cpp:364,372-376).
    Pure-Python loops: test-sized matrices only. Shares no code with the
    product package."""
    starts = np.asarray(layout.starts, np.int64)
    P = len(starts) - 1
    dt = np.asarray(glob.vals).dtype
    parts = [_split(glob.rowptr, glob.colind, glob.vals, starts, r) for r in range(P)]
    ys = []
    with np.errstate(over="ignore"):
        if not transpose:
            for r, (diag, off, garray) in enumerate(parts):
                xo = x[starts[r]:starts[r + 1]]
                xg = x[garray]
                y = np.zeros(len(diag), dtype=dt)
                for i, row in enumerate(diag):
                    acc = dt.type(0)
                    for c, v in row:
                        acc = acc + v * xo[c]
                    y[i] = acc
                for i, row in enumerate(off):
                    acc = dt.type(0)
                    for c, v in row:
                        acc = acc + v * xg[c]
                    y[i] = y[i] + acc
                ys.append(y)
            return np.concatenate(ys)
        lvecs = []
        for r, (diag, off, garray) in enumerate(parts):
            xo = x[starts[r]:starts[r + 1]]
            y = np.zeros(len(diag), dtype=dt)
            lv = np.zeros(len(garray), dtype=dt)
            for i, row in enumerate(diag):
                for c, v in row:
                    y[c] = y[c] + v * xo[i]
            for i, row in enumerate(off):
                for c, v in row:
                    lv[c] = lv[c] + v * xo[i]
            ys.append(y)
            lvecs.append(lv)
        for r in range(P):  # owners fold remote contributions rank by rank
            for s in range(P):
                if s == r:
                    continue
                g = parts[s][2]
                for gi, v in zip(g, lvecs[s]):
                    if starts[r] <= gi < starts[r + 1]:
                        ys[r][gi - starts[r]] = ys[r][gi - starts[r]] + v
    return np.concatenate(ys)
