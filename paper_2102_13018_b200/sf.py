"""Python mirror of the reference's ``sf::`` API over the C ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/sf/{unit,errors,comm,starforest,ops}.hpp, so the
parity tests read like the reference's own tests (tests/test_sfops.cpp,
test_sfgraph.cpp). Data buffers are CUDA tensors (or raw device pointers);
``*_end`` is stream-ordered, the blocking one-shot forms (``bcast``,
``reduce``, ...) synchronise the stream like the reference's End returns
with data ready.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field
from typing import Any, Callable, Optional, Sequence

import numpy as np

from . import _lib as L


# ----------------------------------------------------------------- vocabulary
class Kind(enum.IntEnum):  # unit.hpp:14
    int32 = 0
    int64 = 1
    float64 = 2
    bytes = 3


class ReduceOp(enum.IntEnum):  # unit.hpp:46
    replace = 0
    sum = 1
    prod = 2
    max = 3
    min = 4
    land = 5
    lor = 6
    band = 7
    bor = 8


class SetupAlg(enum.IntEnum):  # starforest.hpp:41
    automatic = 0
    dense = 1
    consensus = 2


class SfState(enum.IntEnum):  # starforest.hpp:38
    created = 0
    graph_set = 1
    set_up = 2


class OpKind(enum.IntEnum):  # ops.hpp:14
    bcast = 0
    reduce = 1
    fetch_and_op = 2
    gather = 3
    scatter = 4


_KIND_SIZE = {Kind.int32: 4, Kind.int64: 8, Kind.float64: 8, Kind.bytes: 1}


@dataclass(frozen=True)
class Unit:  # unit.hpp:37-44
    kind: Kind = Kind.int64
    blocklen: int = 1

    def elem_size(self) -> int:
        return _KIND_SIZE[Kind(self.kind)]

    def bytes(self) -> int:
        return self.elem_size() * self.blocklen


def unit_of(dtype: Any, blocklen: int = 1) -> Unit:
    """unit.hpp:88-91; accepts numpy/torch dtypes or names."""
    name = str(dtype).replace("torch.", "")
    table = {"int32": Kind.int32, "int64": Kind.int64, "float64": Kind.float64,
             "double": Kind.float64, "uint8": Kind.bytes}
    if name not in table:
        raise Error(f"no unit kind for dtype {dtype}")
    return Unit(table[name], blocklen)


# --------------------------------------------------------------------- errors
class Error(RuntimeError):  # errors.hpp:11
    pass


class TimeoutError(Error):  # noqa: A001  (errors.hpp:18, the reference's name)
    pass


class CudaError(Error):
    pass


@dataclass
class RankReport:  # harness.hpp:35-39
    rank: int
    state: str = "ok"  # ok | failed | stalled
    message: str = ""


class HarnessError(Error):  # harness.hpp:41-49
    def __init__(self, msg: str, report: list[RankReport]):
        super().__init__(msg)
        self.report = report


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = L.last_error()
    if rc == 2:
        raise TimeoutError(msg)
    if rc == 3:
        raise CudaError(msg)
    raise Error(msg)


def _lib():
    return L.load()


# ------------------------------------------------------------------- config
@dataclass
class CommConfig:  # comm.hpp:54-66
    nranks: int = 1
    backend: str = "threads"  # threads | nccl | p2p
    deterministic: bool = True
    debug_checksum: bool = False
    force_remote: bool = False
    dense_discovery_threshold: int = 64
    seed: int = 1
    timeout_s: float = 30.0

    def _c(self) -> L.sfg_config:
        c = L.sfg_config()
        c.deterministic = int(self.deterministic)
        c.debug_checksum = int(self.debug_checksum)
        c.force_remote = int(self.force_remote)
        c.dense_discovery_threshold = int(self.dense_discovery_threshold)
        c.seed = int(self.seed)
        c.timeout_s = float(self.timeout_s)
        return c


class World:
    """In-process world of thread ranks (harness.cpp:51-101)."""

    def __init__(self, nranks: int, timeout_s: float = 30.0):
        h = C.c_void_p()
        _check(_lib().sfg_world_create(nranks, timeout_s, C.byref(h)))
        self._h = h
        self.nranks = nranks

    def abort(self) -> None:
        _lib().sfg_world_abort(self._h)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _lib().sfg_world_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib().sfg_nccl_unique_id(buf, 128))
    return buf.raw


class Comm:
    """One rank of a communicator (comm.hpp:97-146)."""

    def __init__(self, nranks: int = 1, rank: int = 0, device: int = -1,
                 config: Optional[CommConfig] = None, world: Optional[World] = None,
                 nccl_id: Optional[bytes] = None):
        cfg = config or CommConfig(nranks=nranks)
        h = C.c_void_p()
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        _check(_lib().sfg_comm_create(world._h if world else None, nranks, rank, device,
                                      cfg.backend.encode(), idbuf, C.byref(cfg._c()),
                                      C.byref(h)))
        self._h = h
        self._world = world  # keep alive
        self.config = cfg
        self.device = device
        self._rank, self._size = rank, nranks

    @classmethod
    def from_torch_distributed(cls, device: int = -1, config: Optional[CommConfig] = None,
                               nccl_id: Optional[bytes] = None, group=None) -> "Comm":
        """One rank per process; SetUp's host collectives run over an
        initialised torch.distributed process group (gloo or nccl); the data
        plane is the library's NCCL communicator (config.backend 'nccl',
        nccl_id shared by the caller) or none for host-only use."""
        import torch
        import torch.distributed as dist

        nranks, rank = dist.get_world_size(group), dist.get_rank(group)
        tdev = torch.device("cuda", torch.cuda.current_device()) \
            if dist.get_backend(group) == "nccl" else torch.device("cpu")

        def allgather(ctx, inp, nbytes, out):
            try:
                t = torch.frombuffer(bytearray(C.string_at(inp, nbytes)), dtype=torch.uint8).to(tdev)
                outs = [torch.empty(nbytes, dtype=torch.uint8, device=tdev) for _ in range(nranks)]
                dist.all_gather(outs, t, group=group)
                host = torch.cat(outs).cpu().numpy()
                C.memmove(out, host.ctypes.data, nbytes * nranks)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        def alltoallv(ctx, send, send_bytes, recv, recv_bytes):
            try:
                sb = [int(send_bytes[i]) for i in range(nranks)]
                rb = [int(recv_bytes[i]) for i in range(nranks)]
                st = torch.frombuffer(bytearray(C.string_at(send, sum(sb)) if sum(sb) else b"\0"),
                                      dtype=torch.uint8)[:sum(sb)].to(tdev)
                rt = torch.empty(sum(rb), dtype=torch.uint8, device=tdev)
                dist.all_to_all_single(rt, st, output_split_sizes=rb, input_split_sizes=sb, group=group)
                if sum(rb):
                    host = rt.cpu().numpy()
                    C.memmove(recv, host.ctypes.data, sum(rb))
                return 0
            except Exception:  # noqa: BLE001
                return 1

        def barrier(ctx):
            try:
                dist.barrier(group=group)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        cfg = config or CommConfig(nranks=nranks, backend="nccl" if device >= 0 else "threads")
        cfg.nranks = nranks
        ops = L.sfg_ctrl_ops(None, L.ALLGATHER_FN(allgather), L.ALLTOALLV_FN(alltoallv),
                             L.BARRIER_FN(barrier))
        self = cls.__new__(cls)
        h = C.c_void_p()
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        _check(_lib().sfg_comm_create_ext(nranks, rank, device, cfg.backend.encode(), idbuf,
                                          C.byref(cfg._c()), C.byref(ops), C.byref(h)))
        self._h, self._world, self.config, self.device = h, None, cfg, device
        self._rank, self._size = rank, nranks
        self._ops = ops  # callbacks must outlive the communicator
        return self

    def rank(self) -> int:
        return self._rank

    def allgather_int64(self, values) -> np.ndarray:
        """Every rank's int64 vector (same length on every rank), stacked
        (size x n) — the control plane's allgather. Collective."""
        v = np.ascontiguousarray(np.asarray(values, dtype=np.int64).reshape(-1))
        out = np.zeros((self._size, v.size), np.int64)
        _check(_lib().sfg_comm_allgather(self._h, v.ctypes.data if v.size else None, v.nbytes,
                                         out.ctypes.data if out.size else None))
        return out

    def size(self) -> int:
        return self._size

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib().sfg_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass


# --------------------------------------------------------------- star forest
@dataclass
class Pattern:
    kind: str
    count: int
    start: int
    dx: int = 0
    dy: int = 0
    dz: int = 0
    s1: int = 0
    s2: int = 0
    bound: int = 0
    has_duplicates: bool = False

    @staticmethod
    def _from(p: L.sfg_pattern) -> "Pattern":
        return Pattern(("contiguous", "affine", "indexed")[p.kind], p.count, p.start, p.dx,
                       p.dy, p.dz, p.s1, p.s2, p.bound, bool(p.has_duplicates))


def analyze(indices: Sequence[int], infer_affine: bool = True,
            extents: Optional[tuple[int, int]] = None) -> Pattern:
    """IndexPattern::analyze (pattern.hpp:52-53) + Affine3D inference."""
    a = np.ascontiguousarray(np.asarray(indices, dtype=np.int64))
    out = L.sfg_pattern()
    ex, exy = extents if extents else (0, 0)
    _check(_lib().sfg_pattern_analyze(a.ctypes.data if a.size else None, a.size,
                                      int(infer_affine), ex, exy, C.byref(out)))
    return Pattern._from(out)


@dataclass
class Group:
    rank: int
    items: np.ndarray
    pattern: Pattern


@dataclass
class TwoSidedInfo:  # starforest.hpp:47-55
    root_ranks: list[tuple[int, list[int]]]
    leaf_ranks: list[tuple[int, list[int]]]
    self_first: bool


@dataclass
class GraphSpec:  # starforest.hpp:29-34
    nroots: int = 0
    nleaves: int = 0
    local: Optional[np.ndarray] = None
    remote_rank: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    remote_off: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))

    def leaf_indices(self) -> np.ndarray:
        return np.arange(self.nleaves, dtype=np.int64) if self.local is None else self.local

    def leaf_bound(self) -> int:
        li = self.leaf_indices()
        return int(li.max()) + 1 if li.size else 0


def _arr(x, dtype) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=dtype))


class StarForest:
    """starforest.hpp:61-148."""

    def __init__(self, comm: Comm, _borrowed: Optional[C.c_void_p] = None):
        self.comm = comm
        self._owned = _borrowed is None
        if _borrowed is None:
            h = C.c_void_p()
            _check(_lib().sfg_sf_create(comm._h, C.byref(h)))
            self._h = h
        else:
            self._h = _borrowed
        self._multi: Optional[StarForest] = None

    def __del__(self):
        try:
            if getattr(self, "_owned", False) and getattr(self, "_h", None):
                _lib().sfg_sf_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass

    # -- graph
    def set_graph(self, nroots: int, nleaves: int, local=None, remote=None, *,
                  remote_rank=None, remote_off=None) -> None:
        """remote: list of (rank, offset) RootRefs, or pass remote_rank/remote_off arrays."""
        if remote is not None:
            rr = _arr([r for r, _ in remote], np.int32) if len(remote) else np.zeros(0, np.int32)
            ro = _arr([o for _, o in remote], np.int64) if len(remote) else np.zeros(0, np.int64)
        else:
            rr = _arr(remote_rank if remote_rank is not None else [], np.int32)
            ro = _arr(remote_off if remote_off is not None else [], np.int64)
        if rr.size != nleaves or ro.size != nleaves:
            raise Error("set_graph: leaf_remote length does not match nleaves")
        loc = None
        if local is not None:
            loc = _arr(local, np.int64)
            if loc.size != nleaves:
                raise Error("set_graph: leaf_local length does not match nleaves")
        _check(_lib().sfg_sf_set_graph(self._h, int(nroots), int(nleaves),
                                       loc.ctypes.data if loc is not None and loc.size else
                                       (C.c_void_p(1) if loc is not None else None),
                                       rr.ctypes.data if rr.size else None,
                                       ro.ctypes.data if ro.size else None))
        self._multi = None

    def set_graph_device(self, nroots: int, nleaves: int, local, remote_rank, remote_off) -> None:
        """set_graph with the arrays already in the communicator's device memory
        (torch CUDA tensors: int64 leaf indices or None, int32 root ranks,
        int64 root offsets); setup() then plans on the GPU."""
        import torch

        def ptr(t, dtype, name):
            if t is None:
                return None
            if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dtype and t.is_contiguous()):
                raise Error(f"set_graph_device: {name} must be a contiguous CUDA {dtype} tensor")
            if t.numel() != nleaves:
                raise Error("set_graph: leaf_remote length does not match nleaves")
            return t.data_ptr() if t.numel() else None
        lp = ptr(local, torch.int64, "local")
        if local is not None and lp is None:
            lp = C.c_void_p(1)  # empty but present
        _check(_lib().sfg_sf_set_graph_device(self._h, int(nroots), int(nleaves), lp,
                                              ptr(remote_rank, torch.int32, "remote_rank"),
                                              ptr(remote_off, torch.int64, "remote_off")))
        self._multi = None

    def set_graph_spec(self, spec: GraphSpec) -> None:
        self.set_graph(spec.nroots, spec.nleaves, spec.local, remote_rank=spec.remote_rank,
                       remote_off=spec.remote_off)

    def setup(self, alg: SetupAlg = SetupAlg.automatic) -> None:
        _check(_lib().sfg_sf_setup(self._h, int(alg)))

    def prepare(self, unit: "Unit") -> None:
        """Device plans + a staging slot for `unit`, built before a CUDA-graph
        capture (SetUp does it for 8-byte units). Collective on p2p."""
        _check(_lib().sfg_sf_prepare(self._h, int(unit.kind), unit.blocklen))

    def _info(self) -> L.sfg_sf_info:
        i = L.sfg_sf_info()
        _check(_lib().sfg_sf_get_info(self._h, C.byref(i)))
        return i

    def state(self) -> SfState:
        return SfState(self._info().state)

    def nroots(self) -> int:
        return self._info().nroots

    def nleaves(self) -> int:
        return self._info().nleaves

    def leaf_index_bound(self) -> int:
        return self._info().leaf_index_bound

    def contiguous_leaves(self) -> bool:
        return bool(self._info().contiguous_leaves)

    def has_self_edges(self) -> bool:
        return bool(self._info().self_first)

    def _groups(self, which: int) -> list[Group]:
        i = self._info()
        if i.state != SfState.set_up:
            _check(_lib().sfg_sf_group(self._h, which, 0, None, None, None))
        n = i.n_root_groups if which == 0 else i.n_leaf_groups
        out = []
        for g in range(n):
            rank, cnt, pat = C.c_int(), C.c_int64(), L.sfg_pattern()
            _check(_lib().sfg_sf_group(self._h, which, g, C.byref(rank), C.byref(cnt), C.byref(pat)))
            items = np.zeros(cnt.value, np.int64)
            _check(_lib().sfg_sf_group_items(self._h, which, g, items.ctypes.data if cnt.value else None))
            out.append(Group(rank.value, items, Pattern._from(pat)))
        return out

    def group_plans(self, which: int) -> list[tuple[int, int, Pattern]]:
        """(rank, count, pattern) per group without copying the item lists
        (which = 0 root groups, 1 leaf groups)."""
        i = self._info()
        n = i.n_root_groups if which == 0 else i.n_leaf_groups
        out = []
        for g in range(n):
            rank, cnt, pat = C.c_int(), C.c_int64(), L.sfg_pattern()
            _check(_lib().sfg_sf_group(self._h, which, g, C.byref(rank), C.byref(cnt), C.byref(pat)))
            out.append((rank.value, cnt.value, Pattern._from(pat)))
        return out

    def root_groups(self) -> list[Group]:
        """Per root-owning rank: leaf ordinals + leaf-index pattern (starforest.hpp:114-118)."""
        return self._groups(0)

    def leaf_groups(self) -> list[Group]:
        """Per leaf-owning rank: root offsets + root pattern (starforest.hpp:119-123)."""
        return self._groups(1)

    def two_sided(self) -> TwoSidedInfo:
        rg, lg = self.root_groups(), self.leaf_groups()
        return TwoSidedInfo([(g.rank, g.items.tolist()) for g in rg],
                            [(g.rank, g.items.tolist()) for g in lg],
                            self.has_self_edges())

    def compute_degrees(self) -> np.ndarray:
        n = self.nroots()
        out = np.zeros(n, np.int64)
        _check(_lib().sfg_sf_compute_degrees(self._h, out.ctypes.data if n else None))
        return out

    def multi_sf(self) -> "StarForest":
        if self._multi is None:
            h = C.c_void_p()
            _check(_lib().sfg_sf_multi_sf(self._h, C.byref(h)))
            m = StarForest(self.comm, _borrowed=h)
            m._parent = self  # keep the owner alive
            self._multi = m
        return self._multi

    def graph_spec(self) -> GraphSpec:
        n = self.nleaves()
        li, rr, ro = np.zeros(n, np.int64), np.zeros(n, np.int32), np.zeros(n, np.int64)
        if n:
            _check(_lib().sfg_sf_graph(self._h, li.ctypes.data, rr.ctypes.data, ro.ctypes.data))
        return GraphSpec(self.nroots(), n, None if self.contiguous_leaves() else li, rr, ro)


# ---------------------------------------------------------------- operations
def _ptr(x) -> Optional[int]:
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        if x.numel() == 0:
            return None
        if not x.is_cuda:
            raise Error("data buffers must be CUDA tensors (device pointers)")
        if not x.is_contiguous():
            raise Error("data buffers must be contiguous")
        return x.data_ptr()
    raise Error(f"unsupported buffer type {type(x)}")


def _stream(s) -> Optional[int]:
    if s is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    if isinstance(s, int):
        return s
    return s.cuda_stream


class OpHandle:
    """ops.hpp:31-51. End must be called exactly once."""

    def __init__(self, h: C.c_void_p, sf: StarForest, stream: int, keep: tuple):
        self._h = h
        self._sf = sf
        self.stream = stream
        self._keep = keep  # buffers stay referenced until the handle is ended

    def _q(self):
        k, o, e = C.c_int(), C.c_int(), C.c_int()
        _check(_lib().sfg_handle_info(self._h, C.byref(k), C.byref(o), C.byref(e)))
        return k.value, o.value, e.value

    def kind(self) -> OpKind:
        return OpKind(self._q()[0])

    def op(self) -> ReduceOp:
        return ReduceOp(self._q()[1])

    def ended(self) -> bool:
        return bool(self._q()[2])

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _lib().sfg_handle_free(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass


def _begin(fn, sf: StarForest, args: list, stream, keep) -> OpHandle:
    s = _stream(stream)
    h = C.c_void_p()
    _check(fn(sf._h, *args, s, C.byref(h)))
    return OpHandle(h, sf, s, keep)


def bcast_begin(sf: StarForest, unit: Unit, rootdata, leafdata, op: ReduceOp, stream=None) -> OpHandle:
    """ops.hpp:57-63: leafdata[leaf] (op)= rootdata[root] per edge."""
    return _begin(_lib().sfg_bcast_begin, sf,
                  [int(unit.kind), unit.blocklen, _ptr(rootdata), _ptr(leafdata), int(op)],
                  stream, (rootdata, leafdata))


def bcast_end(h: OpHandle) -> None:
    _check(_lib().sfg_bcast_end(h._h))


def reduce_begin(sf: StarForest, unit: Unit, leafdata, rootdata, op: ReduceOp, stream=None) -> OpHandle:
    """ops.hpp:65-71: rootdata[root] (op)= fold of its leaves."""
    return _begin(_lib().sfg_reduce_begin, sf,
                  [int(unit.kind), unit.blocklen, _ptr(leafdata), _ptr(rootdata), int(op)],
                  stream, (leafdata, rootdata))


def reduce_end(h: OpHandle) -> None:
    _check(_lib().sfg_reduce_end(h._h))


def fetch_and_op_begin(sf: StarForest, unit: Unit, rootdata, leafdata, leafupdate,
                       op: ReduceOp, stream=None) -> OpHandle:
    """ops.hpp:73-83."""
    return _begin(_lib().sfg_fetch_and_op_begin, sf,
                  [int(unit.kind), unit.blocklen, _ptr(rootdata), _ptr(leafdata),
                   _ptr(leafupdate), int(op)], stream, (rootdata, leafdata, leafupdate))


def fetch_and_op_end(h: OpHandle) -> None:
    _check(_lib().sfg_fetch_and_op_end(h._h))


def gather_begin(sf: StarForest, unit: Unit, leafdata, multirootdata, stream=None) -> OpHandle:
    """ops.hpp:85-89 (over the multi-SF)."""
    return _begin(_lib().sfg_gather_begin, sf,
                  [int(unit.kind), unit.blocklen, _ptr(leafdata), _ptr(multirootdata)],
                  stream, (leafdata, multirootdata))


def gather_end(h: OpHandle) -> None:
    _check(_lib().sfg_gather_end(h._h))


def scatter_begin(sf: StarForest, unit: Unit, multirootdata, leafdata, stream=None) -> OpHandle:
    """ops.hpp:91-94."""
    return _begin(_lib().sfg_scatter_begin, sf,
                  [int(unit.kind), unit.blocklen, _ptr(multirootdata), _ptr(leafdata)],
                  stream, (multirootdata, leafdata))


def scatter_end(h: OpHandle) -> None:
    _check(_lib().sfg_scatter_end(h._h))


def _one_shot(fn, args: list, stream, sync: bool) -> None:
    s = _stream(stream)
    _check(fn(*args, s))
    if sync:
        import torch

        torch.cuda.ExternalStream(s).synchronize()


# One-shot forms (ops.hpp:60, 68, 79, 88, 94): Begin + End back to back on
# `stream`. sync=True blocks like the reference's; sync=False leaves them
# stream-ordered (CUDA-graph capturable). With nothing of the caller's between
# the halves, the p2p exchange runs on the stream itself (no fork / join).
def bcast(sf, unit, rootdata, leafdata, op, stream=None, sync: bool = True) -> None:
    _one_shot(_lib().sfg_bcast, [sf._h, int(unit.kind), unit.blocklen, _ptr(rootdata), _ptr(leafdata),
                                 int(op)], stream, sync)


def reduce(sf, unit, leafdata, rootdata, op, stream=None, sync: bool = True) -> None:
    _one_shot(_lib().sfg_reduce, [sf._h, int(unit.kind), unit.blocklen, _ptr(leafdata), _ptr(rootdata),
                                  int(op)], stream, sync)


def fetch_and_op(sf, unit, rootdata, leafdata, leafupdate, op, stream=None, sync: bool = True) -> None:
    _one_shot(_lib().sfg_fetch_and_op, [sf._h, int(unit.kind), unit.blocklen, _ptr(rootdata), _ptr(leafdata),
                                        _ptr(leafupdate), int(op)], stream, sync)


def gather(sf, unit, leafdata, multirootdata, stream=None, sync: bool = True) -> None:
    _one_shot(_lib().sfg_gather, [sf._h, int(unit.kind), unit.blocklen, _ptr(leafdata), _ptr(multirootdata)],
              stream, sync)


def scatter(sf, unit, multirootdata, leafdata, stream=None, sync: bool = True) -> None:
    _one_shot(_lib().sfg_scatter, [sf._h, int(unit.kind), unit.blocklen, _ptr(multirootdata), _ptr(leafdata)],
              stream, sync)


# --------------------------------------------------------------- counters
def counters() -> dict:
    c = L.sfg_counters()
    _check(_lib().sfg_counters_get(C.byref(c)))
    return {n: getattr(c, n) for n, _ in L.sfg_counters._fields_}


def counters_reset() -> None:
    _check(_lib().sfg_counters_reset())


def timing_enable(on: bool = True) -> None:
    """Record CUDA events around every library kernel (on its launch stream)."""
    _check(_lib().sfg_timing_enable(int(on)))


def timing_collect() -> dict:
    """{tag: {"launches", "total_ms", "bytes", "link_bytes"}} for launches since the last collect."""
    cap = 64
    arr = (L.sfg_timing * cap)()
    n = C.c_int()
    _check(_lib().sfg_timing_collect(arr, cap, C.byref(n)))
    return {arr[i].tag.decode(): {"launches": arr[i].launches, "total_ms": arr[i].total_ms,
                                  "bytes": arr[i].bytes, "link_bytes": arr[i].link_bytes}
            for i in range(n.value)}


# ------------------------------------------------------------ graph algebra
def _new_forest(comm: Comm, h: C.c_void_p) -> StarForest:
    f = StarForest.__new__(StarForest)
    f.comm, f._owned, f._h, f._multi = comm, True, h, None
    return f


def compose(a: StarForest, b: StarForest) -> StarForest:
    """starforest.hpp:150-154 (collective): roots of A, leaves of B, an edge
    where an A leaf and a B root coincide on (rank, index)."""
    h = C.c_void_p()
    _check(_lib().sfg_sf_compose(a._h, b._h, 0, C.byref(h)))
    return _new_forest(a.comm, h)


def compose_inverse(a: StarForest, b: StarForest) -> StarForest:
    """starforest.hpp:156-159 (collective): roots of A, leaves = B's roots."""
    h = C.c_void_p()
    _check(_lib().sfg_sf_compose(a._h, b._h, 1, C.byref(h)))
    return _new_forest(a.comm, h)


def _embed(f: StarForest, which: int, selected) -> StarForest:
    sel = np.ascontiguousarray(np.asarray(selected, dtype=np.int64))
    h = C.c_void_p()
    _check(_lib().sfg_sf_embed(f._h, which, sel.ctypes.data if sel.size else None, sel.size, C.byref(h)))
    return _new_forest(f.comm, h)


def embed_root(f: StarForest, selected_roots) -> StarForest:
    """starforest.hpp:161-166: keep the edges whose root is selected."""
    return _embed(f, 0, selected_roots)


def embed_leaf(f: StarForest, selected_leaves) -> StarForest:
    """starforest.hpp:161-167: keep the edges whose leaf index is selected."""
    return _embed(f, 1, selected_leaves)


def identity_sf(comm: Comm, n: int) -> StarForest:
    """starforest.hpp:169-171: leaf i -> root i on this rank (graph set)."""
    h = C.c_void_p()
    _check(_lib().sfg_sf_identity(comm._h, n, C.byref(h)))
    return _new_forest(comm, h)


# ----------------------------------------------------------------- harness
def run_ranks(cfg: CommConfig, body: Callable[[Comm], Any], devices: Optional[Sequence[int]] = None) -> list:
    """harness.hpp:58-72: one thread per rank, results per rank; a failing or
    stalled rank aborts the others and raises HarnessError with a report.

    devices[r] is the CUDA device of rank r (default: every rank on device 0
    when CUDA is available, host-only otherwise)."""
    n = cfg.nranks
    if devices is None:
        try:
            import torch

            dev = 0 if torch.cuda.is_available() else -1
        except Exception:
            dev = -1
        devices = [dev] * n
    world = World(n, cfg.timeout_s)
    nccl_id = nccl_unique_id() if cfg.backend == "nccl" else None
    results: list = [None] * n
    errors: list = [None] * n

    def worker(r: int) -> None:
        try:
            if devices[r] >= 0:
                import torch

                torch.cuda.set_device(devices[r])
            comm = Comm(n, r, devices[r], cfg, world=world, nccl_id=nccl_id)
            try:
                results[r] = body(comm)
            finally:
                if devices[r] >= 0:
                    import torch

                    torch.cuda.synchronize(devices[r])
                del comm
        except BaseException as e:  # noqa: BLE001
            errors[r] = e
            world.abort()

    threads = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(n)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(cfg.timeout_s * 4 + 30)
    report = []
    first = None
    stalled = False
    for r in range(n):
        e = errors[r]
        if e is None and threads[r].is_alive():
            report.append(RankReport(r, "stalled", "did not finish"))
            stalled = True
        elif e is None:
            report.append(RankReport(r))
        elif isinstance(e, TimeoutError):
            report.append(RankReport(r, "stalled", str(e)))
            stalled = True
        else:
            report.append(RankReport(r, "failed", str(e)))
            first = first or e
    if first is None and not stalled:
        return results
    head = f"rank failure: {first}" if first is not None else f"harness timeout after {cfg.timeout_s} s"
    detail = "; ".join(f"rank {x.rank} {'failed' if x.state == 'failed' else 'stalled'}: {x.message}"
                       for x in report if x.state != "ok")
    raise HarnessError(f"{head} [{detail}]", report)


# ------------------------------------------------------------- graph text
def graph_text_parse(text: str) -> list[GraphSpec]:
    """graph_text::parse (starforest.cpp:485-511): per line
    'nroots nleaves [local:rank.offset ...]'."""
    out = []
    for line in text.splitlines():
        if not line.strip():
            continue
        tok = line.split()
        nroots, nleaves = int(tok[0]), int(tok[1])
        local, rr, ro = [], [], []
        for t in tok[2:2 + nleaves]:
            idx, rest = t.split(":")
            rank, off = rest.split(".")
            local.append(int(idx))
            rr.append(int(rank))
            ro.append(int(off))
        out.append(GraphSpec(nroots, nleaves, np.array(local, np.int64),
                             np.array(rr, np.int32), np.array(ro, np.int64)))
    return out


def graph_text_format(specs: Sequence[GraphSpec]) -> str:
    lines = []
    for s in specs:
        li = s.leaf_indices()
        parts = [str(s.nroots), str(s.nleaves)]
        parts += [f"{int(li[o])}:{int(s.remote_rank[o])}.{int(s.remote_off[o])}" for o in range(s.nleaves)]
        lines.append(" ".join(parts))
    return "\n".join(lines) + "\n"
