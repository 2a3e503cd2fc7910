"""Graph and data generators for the BASELINE configurations and the tests.

Every generator returns per-rank ``GraphSpec`` objects (host numpy arrays) so
the GPU path and the reference CPU path are fed identical graphs and data.

* ``Rng`` / ``mix_seed`` — the reference's splitmix64 generator
  (/root/reference/proj/include/sf/rng.hpp:14-51). ``Rng.stream`` draws n
  consecutive ``next()`` values vectorised (state advances by a constant).
* ``random_graph_specs`` — port of the reference's random forest generator
  (/root/reference/proj/src/harness.cpp:148-193), call-for-call identical.
* ``g2l_halo`` — config 2: PETSc DMDA global->local SF of a 3-D grid with a
  7-point (star) stencil, block-partitioned (ghost faces + the interior
  3-D subblock), in the leaf numbering of the ghosted local box.
* ``random_leaf_root`` — configs 1 and 4: contiguous leaves, root = bounded(R).
* ``laplacian27_ghosts`` — config 3: ghost-column SF of a 27-point
  Laplacian (build_column_sf shape, /root/reference/proj/src/spmv.cpp:29-43).
* ``pingpong`` — config 5 (/root/reference/proj/src/bench.cpp:43-53).
"""
from __future__ import annotations

from typing import Optional

import numpy as np

from .sf import GraphSpec

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def _mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class Rng:
    """splitmix64 exactly as rng.hpp:14-45."""

    def __init__(self, seed: int):
        self.state = (seed + GOLDEN) & M64

    def next(self) -> int:
        self.state = (self.state + GOLDEN) & M64
        return _mix(self.state)

    def bounded(self, n: int) -> int:
        return self.next() % n

    def range(self, lo: int, hi: int) -> int:
        return lo + self.bounded(hi - lo + 1)

    def uniform01(self) -> float:
        return float(self.next() >> 11) * (2.0 ** -53)

    def chance(self, p: float) -> bool:
        return self.uniform01() < p

    def shuffle(self, v: list) -> None:
        for i in range(len(v), 1, -1):
            j = self.bounded(i)
            v[i - 1], v[j] = v[j], v[i - 1]

    def stream(self, n: int) -> np.ndarray:
        """The next n values of next(), vectorised (uint64)."""
        k = np.arange(1, n + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = np.uint64(self.state) + k * np.uint64(GOLDEN)
            self.state = (self.state + n * GOLDEN) & M64
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        return z

    def bounded_array(self, n: int, bound: int) -> np.ndarray:
        return (self.stream(n) % np.uint64(bound)).astype(np.int64)

    def uniform01_array(self, n: int) -> np.ndarray:
        return (self.stream(n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def range_array(self, n: int, lo: int, hi: int) -> np.ndarray:
        return lo + self.bounded_array(n, hi - lo + 1)


def mix_seed(seed: int, salt: int) -> int:
    """rng.hpp:48-51."""
    return Rng((seed ^ ((salt * 0xD1342543DE82EF95 + 0x2545F4914F6CDD1D) & M64)) & M64).next()


# ------------------------------------------------------------ random forests
def random_graph_specs(seed: int, nranks: int, max_vertices: int) -> list[GraphSpec]:
    """harness.cpp:148-193, identical draw sequence."""
    rng = Rng(mix_seed(seed, 0x5F0C))
    nroots = [rng.range(0, max_vertices) for _ in range(nranks)]
    total = sum(nroots)
    owners = [r for r in range(nranks) if nroots[r] > 0]
    specs = []
    for r in range(nranks):
        if total == 0:
            specs.append(GraphSpec(nroots[r], 0, None, np.zeros(0, np.int32), np.zeros(0, np.int64)))
            continue
        leaf_space = rng.range(0, max_vertices)
        nleaves = rng.range(0, leaf_space)
        contiguous = rng.chance(0.25)
        local = None
        if not contiguous:
            allv = list(range(leaf_space))
            rng.shuffle(allv)
            local = np.array(sorted(allv[:nleaves]), np.int64)
        rr, ro = [], []
        for _ in range(nleaves):
            if rng.chance(0.2) and nroots[r] > 0:
                owner = r
            else:
                owner = owners[rng.bounded(len(owners))]
            off = rng.range(0, nroots[owner] - 1)
            rr.append(owner)
            ro.append(off)
        specs.append(GraphSpec(nroots[r], nleaves, local, np.array(rr, np.int32),
                               np.array(ro, np.int64)))
    return specs


def gen_ints(seed: int, salt: int, n: int, lo: int = -1000, hi: int = 1000) -> np.ndarray:
    """selfcheck.cpp:25-30 (vectorised: identical values)."""
    return Rng(mix_seed(seed, salt)).range_array(n, lo, hi)


def gen_f64(seed: int, salt: int, n: int) -> np.ndarray:
    return Rng(mix_seed(seed, salt)).uniform01_array(n)


# ------------------------------------------------------------ configs 1 and 4
def random_leaf_root(nleaves: int, nroots: int, nranks: int = 1, seed: int = 1,
                     salt: int = 1) -> list[GraphSpec]:
    """Contiguous leaves; global root g = bounded(nroots) drawn in global leaf
    order; rank r owns leaves [r*L/P, (r+1)*L/P) and roots [r*R/P, ...)."""
    rng = Rng(mix_seed(seed, salt))
    g = rng.bounded_array(nleaves, nroots)
    rpr = nroots // nranks
    lpr = nleaves // nranks
    specs = []
    for r in range(nranks):
        gg = g[r * lpr:(r + 1) * lpr] if r < nranks - 1 else g[r * lpr:]
        owner = np.minimum(gg // rpr, nranks - 1).astype(np.int32)
        off = gg - owner.astype(np.int64) * rpr
        nr = rpr if r < nranks - 1 else nroots - rpr * (nranks - 1)
        specs.append(GraphSpec(nr, gg.size, None, owner, off))
    return specs


# ------------------------------------------------------------------- config 2
def proc_grid(p: int) -> tuple[int, int, int]:
    """P=2 -> 1x1x2, 4 -> 1x2x2, 8 -> 2x2x2, general: factor into z, y, x."""
    dims = [1, 1, 1]
    axis = 2
    n = p
    f = 2
    while n > 1:
        while n % f:
            f += 1
        dims[axis] *= f
        n //= f
        axis = (axis - 1) % 3
    return dims[0], dims[1], dims[2]


def _split(n: int, parts: int) -> list[tuple[int, int]]:
    base, extra = divmod(n, parts)
    out, s = [], 0
    for i in range(parts):
        sz = base + (1 if i < extra else 0)
        out.append((s, sz))
        s += sz
    return out


class G2L:
    """Geometry of config 2 for one rank."""

    def __init__(self, N, P: int, rank: int, dims: Optional[tuple[int, int, int]] = None):
        """N: grid edge (int) or (NX, NY, NZ)."""
        NX, NY, NZ = (N, N, N) if isinstance(N, int) else tuple(N)
        self.N = N
        self.P = P
        self.rank = rank
        self.px, self.py, self.pz = dims or proc_grid(P)
        assert self.px * self.py * self.pz == P
        self.bx = rank % self.px
        self.by = (rank // self.px) % self.py
        self.bz = rank // (self.px * self.py)
        self.xs, self.ys, self.zs = _split(NX, self.px), _split(NY, self.py), _split(NZ, self.pz)
        self.nx, self.ny, self.nz = self.xs[self.bx][1], self.ys[self.by][1], self.zs[self.bz][1]
        self.X, self.Y, self.Z = self.nx + 2, self.ny + 2, self.nz + 2

    def rank_of(self, bx, by, bz) -> int:
        return bx + self.px * (by + self.py * bz)

    @property
    def n_owned(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def n_local(self) -> int:
        return self.X * self.Y * self.Z


def g2l_halo(N, P: int, rank: int, dims=None, ghosts: bool = True,
             interior: bool = True) -> GraphSpec:
    """PETSc DMDA global->local SF, star stencil width 1, non-periodic.

    Roots: the rank's owned block (natural order). Leaves: points of the
    ghosted local box (nx+2)(ny+2)(nz+2) in natural order; owned points map to
    the rank's own roots (the interior 3-D subblock), face ghosts map to the
    neighbour's boundary plane, edge/corner ghosts and ghosts beyond the
    domain boundary stay unconnected. ``interior=False`` gives the halo-only SF.
    Leaves are generated in ascending local index.
    """
    g = G2L(N, P, rank, dims)
    nx, ny, nz, X, Y = g.nx, g.ny, g.nz, g.X, g.Y
    XY = X * Y
    has = {
        "xl": g.bx > 0, "xh": g.bx < g.px - 1,
        "yl": g.by > 0, "yh": g.by < g.py - 1,
        "zl": g.bz > 0, "zh": g.bz < g.pz - 1,
    }
    has = {k: v and ghosts for k, v in has.items()}
    nbr = {
        "xl": g.rank_of(g.bx - 1, g.by, g.bz), "xh": g.rank_of(g.bx + 1, g.by, g.bz),
        "yl": g.rank_of(g.bx, g.by - 1, g.bz), "yh": g.rank_of(g.bx, g.by + 1, g.bz),
        "zl": g.rank_of(g.bx, g.by, g.bz - 1), "zh": g.rank_of(g.bx, g.by, g.bz + 1),
    }
    nxl = g.xs[g.bx - 1][1] if has["xl"] else 0
    nyl = g.ys[g.by - 1][1] if has["yl"] else 0
    nzl = g.zs[g.bz - 1][1] if has["zl"] else 0
    nyh = g.ys[g.by + 1][1] if has["yh"] else 0
    nxh = g.xs[g.bx + 1][1] if has["xh"] else 0

    i1 = np.arange(1, nx + 1, dtype=np.int64)

    # ---- template of one interior plane (k in 1..nz), in ascending order
    t_off, t_rank, t_root = [], [], []  # root = f(k) affine: root_base + k_coef*(k-1)
    t_kcoef = []

    def add(off, rank, base, kcoef):
        t_off.append(off)
        t_rank.append(np.full(off.size, rank, np.int32))
        t_root.append(base)
        t_kcoef.append(np.full(off.size, kcoef, np.int64))

    if has["yl"]:  # row j = 0, i = 1..nx -> neighbour (by-1) top row y = nyl-1
        add(i1.copy(), nbr["yl"], (i1 - 1) + nx * (nyl - 1), nx * nyl)
    for j in range(1, ny + 1):
        if has["xl"]:
            add(np.array([X * j]), nbr["xl"], np.array([(nxl - 1) + nxl * (j - 1)]), nxl * ny)
        if interior:
            add(X * j + i1, g.rank, (i1 - 1) + nx * (j - 1), nx * ny)
        if has["xh"]:
            add(np.array([X * j + nx + 1]), nbr["xh"], np.array([nxh * (j - 1)]), nxh * ny)
    if has["yh"]:
        add(X * (ny + 1) + i1, nbr["yh"], (i1 - 1), nx * nyh)

    parts_off, parts_rank, parts_root = [], [], []
    jj, ii = np.meshgrid(np.arange(1, ny + 1, dtype=np.int64), i1, indexing="ij")
    face_off = (X * jj + ii).ravel()
    face_root_in = ((ii - 1) + nx * (jj - 1)).ravel()
    if has["zl"]:
        parts_off.append(face_off)
        parts_rank.append(np.full(face_off.size, nbr["zl"], np.int32))
        parts_root.append(face_root_in + nx * ny * (nzl - 1))
    if t_off:
        to = np.concatenate(t_off)
        tr = np.concatenate(t_rank)
        tb = np.concatenate(t_root).astype(np.int64)
        tk = np.concatenate(t_kcoef)
        ks = np.arange(1, nz + 1, dtype=np.int64)
        parts_off.append((ks[:, None] * XY + to[None, :]).ravel())
        parts_rank.append(np.broadcast_to(tr[None, :], (nz, tr.size)).ravel())
        parts_root.append((tb[None, :] + (ks[:, None] - 1) * tk[None, :]).ravel())
    if has["zh"]:
        parts_off.append(face_off + (nz + 1) * XY)
        parts_rank.append(np.full(face_off.size, nbr["zh"], np.int32))
        parts_root.append(face_root_in.copy())
    if parts_off:
        local = np.ascontiguousarray(np.concatenate(parts_off))
        rr = np.ascontiguousarray(np.concatenate(parts_rank).astype(np.int32))
        ro = np.ascontiguousarray(np.concatenate(parts_root).astype(np.int64))
    else:
        local, rr, ro = np.zeros(0, np.int64), np.zeros(0, np.int32), np.zeros(0, np.int64)
    return GraphSpec(g.n_owned, local.size, local, rr, ro)


def g2l_ghost_copies(g: G2L):
    """Per-axis counts of how many neighbours ghost an owned point (star
    stencil: a point on a block face with a neighbour across it is one ghost
    leaf there). copies(x, y, z) = cx[x] + cy[y] + cz[z]."""
    def axis(n, lo, hi):
        c = np.zeros(n, np.int64)
        c[0] += int(lo)
        c[n - 1] += int(hi)
        return c

    return (axis(g.nx, g.bx > 0, g.bx < g.px - 1), axis(g.ny, g.by > 0, g.by < g.py - 1),
            axis(g.nz, g.bz > 0, g.bz < g.pz - 1))


def g2l_check(g: G2L, leaf, root_after) -> dict:
    """Closed-form check of one Bcast(REPLACE) + Reduce(SUM) of the G2L forest
    (``g2l_halo(..., interior=True)``) whose roots started as their local ids
    0..n_owned-1 (float64), any P, every rank independently (torch tensors on
    the device; no oracle, so it runs at the full 512^3 size):

    * leaf box: interior = own ids; a face ghost = the id the neighbour gave
      its boundary point; edges, corners and domain-boundary ghosts keep the
      -1 the leaf array was filled with;
    * roots: id + id (own interior leaf) + id per neighbour ghosting it =
      id * (2 + copies), exact in float64 for ids < 2^50.
    """
    import torch

    dev = leaf.device
    f64 = torch.float64
    nx, ny, nz = g.nx, g.ny, g.nz
    ar = lambda n: torch.arange(n, dtype=f64, device=dev)  # noqa: E731
    x, y, z = ar(nx), ar(ny), ar(nz)
    want = torch.full((g.Z, g.Y, g.X), -1.0, dtype=f64, device=dev)
    want[1:-1, 1:-1, 1:-1] = x[None, None, :] + nx * (y[None, :, None] + ny * z[:, None, None])
    if g.bx > 0:  # neighbour's x = nxl-1 column
        n = g.xs[g.bx - 1][1]
        want[1:-1, 1:-1, 0] = (n - 1) + n * (y[None, :] + ny * z[:, None])
    if g.bx < g.px - 1:
        n = g.xs[g.bx + 1][1]
        want[1:-1, 1:-1, -1] = n * (y[None, :] + ny * z[:, None])
    if g.by > 0:
        n = g.ys[g.by - 1][1]
        want[1:-1, 0, 1:-1] = x[None, :] + nx * (n - 1) + nx * n * z[:, None]
    if g.by < g.py - 1:
        n = g.ys[g.by + 1][1]
        want[1:-1, -1, 1:-1] = x[None, :] + nx * n * z[:, None]
    if g.bz > 0:
        n = g.zs[g.bz - 1][1]
        want[0, 1:-1, 1:-1] = x[None, :] + nx * y[:, None] + nx * ny * (n - 1)
    if g.bz < g.pz - 1:
        want[-1, 1:-1, 1:-1] = x[None, :] + nx * y[:, None]
    leaf_ok = bool(torch.equal(leaf.view(g.Z, g.Y, g.X), want))
    del want
    cx, cy, cz = (torch.from_numpy(c).to(dev) for c in g2l_ghost_copies(g))
    copies = (cx[None, None, :] + cy[None, :, None] + cz[:, None, None]).reshape(-1)
    ids = ar(g.n_owned)
    root_ok = bool(torch.equal(root_after, ids * (2 + copies).to(f64)))
    return {"leaf_ok": leaf_ok, "root_ok": root_ok}


def g2l_reduce_expect(g: G2L, r):
    """Roots after Bcast(REPLACE) + Reduce(SUM) of the G2L forest for ANY
    float64 root values r: the fold r + r (own interior leaf) + r per ghost
    copy, rounded after every addition in the reference order (all addends
    are equal, so the order among ranks does not matter)."""
    import torch

    cx, cy, cz = (torch.from_numpy(c).to(r.device) for c in g2l_ghost_copies(g))
    copies = (cx[None, None, :] + cy[None, :, None] + cz[:, None, None]).reshape(-1)
    e = r + r
    for t in range(1, 4):
        e = torch.where(copies >= t, e + r, e)
    return e


# ------------------------------------------------------------------- config 3
def laplacian27_ghosts(N: int, dims=(2, 2, 2), rank: int = 0, permute_seed: Optional[int] = None):
    """Ghost-column SF of a 27-point Laplacian on an N^3 grid partitioned in
    blocks; rows numbered block by block (each rank's block contiguous,
    natural order inside). Leaves = ghost columns in ascending global order
    (contiguous, like lvec); roots = owned rows. With ``permute_seed`` every
    rank's local numbering is a random permutation (irregular root indices)."""
    px, py, pz = dims
    P = px * py * pz
    xs, ys, zs = _split(N, px), _split(N, py), _split(N, pz)
    bx, by, bz = rank % px, (rank // px) % py, rank // (px * py)

    def block(r):
        return r % px, (r // px) % py, r // (px * py)

    starts = [0]
    for r in range(P):
        a, b, c = block(r)
        starts.append(starts[-1] + xs[a][1] * ys[b][1] * zs[c][1])

    def perm_of(r):
        a, b, c = block(r)
        n = xs[a][1] * ys[b][1] * zs[c][1]
        if permute_seed is None:
            return None
        return np.random.default_rng(mix_seed(permute_seed, r) & 0xFFFFFFFF).permutation(n)

    x0, nx = xs[bx]
    y0, ny = ys[by]
    z0, nz = zs[bz]
    # ghost points: the shell of the (nx+2)(ny+2)(nz+2) box inside the domain
    gx = np.arange(x0 - 1, x0 + nx + 1)
    gy = np.arange(y0 - 1, y0 + ny + 1)
    gz = np.arange(z0 - 1, z0 + nz + 1)
    pts = []
    for z in gz:
        if z < 0 or z >= N:
            continue
        zin = z0 <= z < z0 + nz
        if zin:
            # only the ring of this plane
            ring = [(x, y) for y in (y0 - 1, y0 + ny) for x in gx] + \
                   [(x, y) for y in range(y0, y0 + ny) for x in (x0 - 1, x0 + nx)]
            arr = np.array(ring, np.int64).reshape(-1, 2)
            xx, yy = arr[:, 0], arr[:, 1]
        else:
            yy, xx = np.meshgrid(gy, gx, indexing="ij")
            xx, yy = xx.ravel(), yy.ravel()
        ok = (xx >= 0) & (xx < N) & (yy >= 0) & (yy < N)
        pts.append(np.stack([xx[ok], yy[ok], np.full(ok.sum(), z)], 1))
    pts = np.concatenate(pts) if pts else np.zeros((0, 3), np.int64)
    # owner + local natural index
    def locate(p, parts):
        idx = np.searchsorted(np.array([s for s, _ in parts]), p, side="right") - 1
        return idx
    ox, oy, oz = locate(pts[:, 0], xs), locate(pts[:, 1], ys), locate(pts[:, 2], zs)
    owner = (ox + px * (oy + py * oz)).astype(np.int32)
    lx = pts[:, 0] - np.array([s for s, _ in xs])[ox]
    ly = pts[:, 1] - np.array([s for s, _ in ys])[oy]
    lz = pts[:, 2] - np.array([s for s, _ in zs])[oz]
    nxo = np.array([n for _, n in xs])[ox]
    nyo = np.array([n for _, n in ys])[oy]
    loc = lx + nxo * (ly + nyo * lz)
    if permute_seed is not None:
        for r in np.unique(owner):
            pm = perm_of(int(r))
            sel = owner == r
            loc[sel] = pm[loc[sel]]
    glob = np.array(starts[:-1], np.int64)[owner] + loc
    order = np.argsort(glob, kind="stable")
    owner, loc = owner[order], loc[order]
    a, b, c = block(rank)
    nroots = xs[a][1] * ys[b][1] * zs[c][1]
    return GraphSpec(nroots, owner.size, None, np.ascontiguousarray(owner), np.ascontiguousarray(loc))


# ------------------------------------------------------------------- config 5
def pingpong(nbytes: int) -> list[GraphSpec]:
    """bench.cpp:43-53: rank 0 owns n roots, rank 1 has n contiguous leaves."""
    n = nbytes // 8
    return [GraphSpec(n, 0, None, np.zeros(0, np.int32), np.zeros(0, np.int64)),
            GraphSpec(0, n, None, np.zeros(n, np.int32), np.arange(n, dtype=np.int64))]
