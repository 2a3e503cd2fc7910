"""Distributed SpMV over the star forest — Python mirror of the reference's
``sf/spmv.hpp`` (the path's consumer).

Host-side structures follow the reference one to one:
  Layout           spmv.hpp:19-29, spmv.cpp:10-27
  Csr              spmv.hpp:31-78 (host CSR; ``multiply*`` are the reference's
                   sequential loops, used by tests as the oracle)
  SplitMatrix /    spmv.hpp:84-127 (diagonal block with local columns,
  split_matrix     off-diagonal block with reduced columns + garray)
  build_column_sf  spmv.cpp:29-43
The device side is the C ABI: ``Matrix`` uploads a block (SELL-32 + its
transpose), ``spmv`` / ``spmv_transpose`` run spmv.hpp:149-169 on the GPU with
the ghost Bcast overlapped with the diagonal product.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import sf as _sf
from .graphs import GraphSpec, Rng
from .sf import Kind, StarForest, _check, _lib, _ptr, _stream


@dataclass
class Layout:
    """Contiguous per-rank ranges of a global index space (spmv.hpp:19-29)."""

    starts: np.ndarray

    @staticmethod
    def contiguous(n: int, nranks: int) -> "Layout":
        base, extra = divmod(n, nranks)
        sizes = [base + (1 if r < extra else 0) for r in range(nranks)]
        return Layout(np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64))

    def nranks(self) -> int:
        return len(self.starts) - 1

    def total(self) -> int:
        return int(self.starts[-1])

    def begin(self, r: int) -> int:
        return int(self.starts[r])

    def end(self, r: int) -> int:
        return int(self.starts[r + 1])

    def local_size(self, r: int) -> int:
        return self.end(r) - self.begin(r)

    def owner(self, g):
        """spmv.cpp:22-27 (vectorised over an array of global indices)."""
        g = np.asarray(g, dtype=np.int64)
        if g.size and (g.min() < 0 or g.max() >= self.total()):
            raise _sf.Error("global index outside the layout range")
        return np.searchsorted(self.starts, g, side="right").astype(np.int32) - 1


@dataclass
class Csr:
    """Host CSR (spmv.hpp:31-78). ``multiply*`` are the reference's sequential
    loops (pure Python over rows, vectorised inside a row only where the order
    is kept), the CPU oracle of the GPU SpMV for test-sized matrices."""

    rows: int
    cols: int
    rowptr: np.ndarray
    colind: np.ndarray
    vals: np.ndarray

    @staticmethod
    def from_triplets(rows: int, cols: int, r, c, v) -> "Csr":
        r = np.asarray(r, dtype=np.int64)
        c = np.asarray(c, dtype=np.int64)
        v = np.asarray(v)
        order = np.lexsort((c, r))
        r, c, v = r[order], c[order], v[order]
        rowptr = np.zeros(rows + 1, dtype=np.int64)
        np.add.at(rowptr, r + 1, 1)
        return Csr(rows, cols, np.cumsum(rowptr), c, v)

    def _row_dot(self, r: int, x) -> object:
        acc = self.vals.dtype.type(0)
        for i in range(int(self.rowptr[r]), int(self.rowptr[r + 1])):
            acc = acc + self.vals[i] * x[self.colind[i]]
        return acc

    def multiply(self, x) -> np.ndarray:  # y = A x
        with np.errstate(over="ignore"):
            return np.array([self._row_dot(r, x) for r in range(self.rows)], dtype=self.vals.dtype)

    def multiply_add(self, x, y) -> None:  # y += A x
        with np.errstate(over="ignore"):
            for r in range(self.rows):
                y[r] = y[r] + self._row_dot(r, x)

    def multiply_transpose_add(self, x, y) -> None:  # y += A^T x
        with np.errstate(over="ignore"):
            for r in range(self.rows):
                for i in range(int(self.rowptr[r]), int(self.rowptr[r + 1])):
                    c = self.colind[i]
                    y[c] = y[c] + self.vals[i] * x[r]


@dataclass
class SplitMatrix:
    """spmv.hpp:84-92."""

    row_layout: Layout
    col_layout: Layout
    rank: int
    diag: Csr
    offdiag: Csr
    garray: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))


def split_matrix(glob: Csr, rows: Layout, cols: Layout, rank: int) -> SplitMatrix:
    """spmv.hpp:95-127: diagonal block (local columns), off-diagonal block
    with columns renumbered densely in ascending global order (garray)."""
    r0, r1 = rows.begin(rank), rows.end(rank)
    c0, c1 = cols.begin(rank), cols.end(rank)
    lo, hi = int(glob.rowptr[r0]), int(glob.rowptr[r1])
    rr = np.repeat(np.arange(r0, r1, dtype=np.int64), np.diff(glob.rowptr[r0:r1 + 1])) - r0
    cc = glob.colind[lo:hi]
    vv = glob.vals[lo:hi]
    own = (cc >= c0) & (cc < c1)
    diag = Csr.from_triplets(r1 - r0, c1 - c0, rr[own], cc[own] - c0, vv[own])
    garray = np.unique(cc[~own])
    red = np.searchsorted(garray, cc[~own])
    off = Csr.from_triplets(r1 - r0, len(garray), rr[~own], red, vv[~own])
    return SplitMatrix(rows, cols, rank, diag, off, garray.astype(np.int64))


def column_sf_spec(col_layout: Layout, rank: int, global_cols) -> GraphSpec:
    """The graph build_column_sf sets (spmv.cpp:29-43): roots = my owned
    columns, leaf i = global column global_cols[i] at its owner."""
    g = np.asarray(global_cols, dtype=np.int64)
    owner = col_layout.owner(g)
    off = g - col_layout.starts[owner]
    return GraphSpec(col_layout.local_size(rank), len(g), None, owner.astype(np.int32), off.astype(np.int64))


def build_column_sf(comm, col_layout: Layout, global_cols) -> StarForest:
    """spmv.cpp:29-43 (collective)."""
    f = StarForest(comm)
    f.set_graph_spec(column_sf_spec(col_layout, comm.rank(), global_cols))
    f.setup()
    return f


def select_submatrix_columns(sf_a: StarForest, sf_b: StarForest, selected_global_columns,
                             stream=None):
    """spmv.cpp:45-73 (collective): the new column index, in the
    submatrix's column layout (my selected columns take [prefix, prefix +
    count), ranks in order), of every leaf of `sf_a` (the matrix's column SF,
    e.g. build_column_sf over its garray), or -1 for a column nobody
    selected. `sf_b` = build_column_sf over the selection. Two device
    operations: Reduce REPLACE of the new indices onto the column owners, then
    Bcast REPLACE of the owners' tags into sf_a's leaves. Returns an int64
    CUDA tensor of sf_a.leaf_index_bound() entries."""
    import torch

    comm = sf_a.comm
    sel = np.asarray(selected_global_columns, dtype=np.int64)
    counts = comm.allgather_int64([sel.size])[:, 0]
    prefix = int(counts[:comm.rank()].sum())
    new_index = torch.arange(prefix, prefix + sel.size, dtype=torch.int64, device="cuda")
    tags = torch.full((sf_b.nroots(),), -1, dtype=torch.int64, device="cuda")
    u = _sf.Unit(Kind.int64)
    _sf.reduce(sf_b, u, new_index, tags, _sf.ReduceOp.replace, stream)
    out = torch.full((sf_a.leaf_index_bound(),), -1, dtype=torch.int64, device="cuda")
    _sf.bcast(sf_a, u, tags, out, _sf.ReduceOp.replace, stream)
    return out


def build_ghost_sf(comm, m: SplitMatrix) -> StarForest:
    """spmv.hpp:140-143."""
    return build_column_sf(comm, m.col_layout, m.garray)


_KIND = {np.dtype(np.float64): Kind.float64, np.dtype(np.int64): Kind.int64}


class Matrix:
    """A matrix block on the communicator's GPU (SELL-32 + transpose)."""

    def __init__(self, comm, a: Csr):
        kind = _KIND.get(np.dtype(a.vals.dtype))
        if kind is None:
            raise _sf.Error("SpMV supports float64 and int64 matrices")
        rp = np.ascontiguousarray(a.rowptr, dtype=np.int64)
        ci = np.ascontiguousarray(a.colind, dtype=np.int64)
        vv = np.ascontiguousarray(a.vals)
        h = C.c_void_p()
        _check(_lib().sfg_mat_create(comm._h, a.rows, a.cols, rp.ctypes.data, ci.ctypes.data,
                                     vv.ctypes.data, int(kind), C.byref(h)))
        self._h = h
        self.rows, self.cols, self.nnz, self.kind = a.rows, a.cols, int(a.rowptr[-1]), kind

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _lib().sfg_mat_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass


def spmv(ghost_sf: StarForest, diag: Matrix, offdiag: Matrix, x_owned, lvec, y, stream=None) -> None:
    """spmv.hpp:149-157 on the GPU: y = A x_owned + B lvec; the ghost Bcast
    (x_owned -> lvec) is overlapped with A x_owned. Stream-ordered."""
    _check(_lib().sfg_spmv(ghost_sf._h, diag._h, offdiag._h, _ptr(x_owned), _ptr(lvec), _ptr(y),
                           _stream(stream)))


def spmv_transpose(ghost_sf: StarForest, diag: Matrix, offdiag: Matrix, x_owned, lvec, y,
                   stream=None) -> None:
    """spmv.hpp:161-169 on the GPU: y = A^T x_owned; lvec = B^T x_owned;
    Reduce(SUM) lvec into the owners of y."""
    _check(_lib().sfg_spmv_transpose(ghost_sf._h, diag._h, offdiag._h, _ptr(x_owned), _ptr(lvec),
                                     _ptr(y), _stream(stream)))


# ------------------------------------------------------------ generators
def random_sparse(rng: Rng, n: int, nnz_per_row: int, dtype=np.float64) -> Csr:
    """spmv.hpp:186-214 (duplicate coordinates summed)."""
    r, c, v = [], [], []
    for i in range(n):
        for _ in range(nnz_per_row):
            r.append(i)
            c.append(rng.range(0, n - 1))
            v.append(rng.range(-50, 50) if np.dtype(dtype) == np.int64 else rng.uniform01() * 2.0 - 1.0)
    r, c, v = np.array(r, np.int64), np.array(c, np.int64), np.array(v, dtype=dtype)
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    keep = np.ones(len(r), bool)
    keep[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    starts = np.flatnonzero(keep)
    vs = np.array([v[a:b].sum() if b - a > 1 else v[a] for a, b in zip(starts, list(starts[1:]) + [len(v)])],
                  dtype=dtype)
    return Csr.from_triplets(n, n, r[keep], c[keep], vs)


def laplacian_5pt(nx: int, ny: int) -> Csr:
    """spmv.cpp:75-89."""
    j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    rid = (j * nx + i).ravel()
    rr, cc, vv = [rid], [rid], [np.full(rid.size, 4.0)]
    for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        ii, jj = i + di, j + dj
        ok = ((ii >= 0) & (ii < nx) & (jj >= 0) & (jj < ny)).ravel()
        rr.append(rid[ok])
        cc.append((jj * nx + ii).ravel()[ok])
        vv.append(np.full(int(ok.sum()), -1.0))
    return Csr.from_triplets(nx * ny, nx * ny, np.concatenate(rr), np.concatenate(cc), np.concatenate(vv))


def laplacian27_block(N: int, dims, rank: int):
    """Rank `rank`'s rows of the 27-point Laplacian on an N^3 grid numbered
    block-by-block (BASELINE config 3: 2x2x2 blocks, rank-major global
    numbering, so Layout.contiguous gives the row/column distribution).
    Returns (global CSR rows of this rank as (rowptr, colind, vals), layout)."""
    px, py, pz = dims
    P = px * py * pz

    def split(n, p):
        base, extra = divmod(n, p)
        sz = [base + (1 if k < extra else 0) for k in range(p)]
        return np.concatenate([[0], np.cumsum(sz)]).astype(np.int64)

    xs, ys, zs = split(N, px), split(N, py), split(N, pz)
    sizes = [int((xs[b % px + 1] - xs[b % px]) * (ys[(b // px) % py + 1] - ys[(b // px) % py]) *
                 (zs[b // (px * py) + 1] - zs[b // (px * py)])) for b in range(P)]
    starts = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    layout = Layout(starts)

    def gid(x, y, z):
        bx = np.searchsorted(xs, x, side="right") - 1
        by = np.searchsorted(ys, y, side="right") - 1
        bz = np.searchsorted(zs, z, side="right") - 1
        b = bx + px * (by + py * bz)
        lx, ly, lz = x - xs[bx], y - ys[by], z - zs[bz]
        nx_, ny_ = xs[bx + 1] - xs[bx], ys[by + 1] - ys[by]
        return starts[b] + lx + nx_ * (ly + ny_ * lz)

    bx, by, bz = rank % px, (rank // px) % py, rank // (px * py)
    z, y, x = np.meshgrid(np.arange(zs[bz], zs[bz + 1]), np.arange(ys[by], ys[by + 1]),
                          np.arange(xs[bx], xs[bx + 1]), indexing="ij")
    x, y, z = x.ravel(), y.ravel(), z.ravel()
    rows = x.size
    cols_l, vals_l, cnt = [], [], np.zeros(rows, np.int64)
    offs = [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    for dx, dy, dz in offs:
        xx, yy, zz = x + dx, y + dy, z + dz
        ok = (xx >= 0) & (xx < N) & (yy >= 0) & (yy < N) & (zz >= 0) & (zz < N)
        c = np.where(ok, gid(np.clip(xx, 0, N - 1), np.clip(yy, 0, N - 1), np.clip(zz, 0, N - 1)), -1)
        cols_l.append(c)
        vals_l.append(np.where((dx, dy, dz) == (0, 0, 0), 26.0, -1.0) * np.ones(rows))
        cnt += ok
    C_ = np.stack(cols_l, axis=1)
    V = np.stack(vals_l, axis=1)
    order = np.argsort(np.where(C_ < 0, np.iinfo(np.int64).max, C_), axis=1, kind="stable")
    C_ = np.take_along_axis(C_, order, axis=1)
    V = np.take_along_axis(V, order, axis=1)
    mask = C_ >= 0
    rowptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    return (rowptr, C_[mask].astype(np.int64), V[mask].astype(np.float64)), layout


def split_rows(rowptr, colind, vals, layout: Layout, rank: int) -> SplitMatrix:
    """split_matrix for a rank that only holds its own rows (global column
    indices), as laplacian27_block produces them."""
    n = len(rowptr) - 1
    c0, c1 = layout.begin(rank), layout.end(rank)
    rr = np.repeat(np.arange(n, dtype=np.int64), np.diff(rowptr))
    own = (colind >= c0) & (colind < c1)
    # rows are in order and columns ascend within a row, so the two masked
    # subsets are already in CSR order (same as from_triplets, without a sort)
    def csr(mask, cols, ncols):
        rp = np.zeros(n + 1, dtype=np.int64)
        rp[1:] = np.cumsum(np.bincount(rr[mask], minlength=n))
        return Csr(n, ncols, rp, cols, vals[mask])
    diag = csr(own, colind[own] - c0, c1 - c0)
    ghost = colind[~own]
    garray = np.unique(ghost)
    off = csr(~own, np.searchsorted(garray, ghost), len(garray))
    return SplitMatrix(layout, layout, rank, diag, off, garray.astype(np.int64))
