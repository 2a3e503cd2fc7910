"""Shared test helpers: run one star-forest operation on the GPU through the
C ABI (ranks = threads, every rank on cuda:0 unless devices are given) and
compare against the oracle."""
from __future__ import annotations

import numpy as np

from paper_2102_13018_b200 import sf

DT_KIND = {np.dtype(np.int32): sf.Kind.int32, np.dtype(np.int64): sf.Kind.int64,
           np.dtype(np.float64): sf.Kind.float64, np.dtype(np.uint8): sf.Kind.bytes}

FP_RTOL = 1e-12  # north_star / selfcheck.cpp:735-738: |a-b| <= 1e-12*max(1,|a|,|b|)


def to_dev(a: np.ndarray):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def set_graph_device(f, spec):
    """set_graph_device of a GraphSpec through CUDA copies of its arrays."""
    loc = None if spec.local is None else to_dev(np.asarray(spec.local, np.int64))
    f.set_graph_device(spec.nroots, spec.nleaves, loc, to_dev(np.asarray(spec.remote_rank, np.int32)),
                       to_dev(np.asarray(spec.remote_off, np.int64)))


def to_host(t) -> np.ndarray:
    return t.cpu().numpy()


def run_gpu(specs, opkind: str, data: list[list[np.ndarray]], op: str = "replace",
            blocklen: int = 1, config: sf.CommConfig | None = None, devices=None,
            setup_alg=sf.SetupAlg.automatic, two_phase: bool = False,
            device_graph: bool = False, one_shot: bool = False):
    """data: per-buffer list of per-rank arrays, in the op's argument order:
    bcast (root, leaf) reduce (leaf, root) fetch_and_op (root, leaf, update)
    gather (leaf, multiroot) scatter (multiroot, leaf). Returns the same
    structure after the op (host copies)."""
    n = len(specs)
    cfg = config or sf.CommConfig(nranks=n)
    cfg.nranks = n
    kind = DT_KIND[np.dtype(data[0][0].dtype)]
    unit = sf.Unit(kind, blocklen)
    rop = sf.ReduceOp[op]

    def body(comm):
        import torch

        r = comm.rank()
        f = sf.StarForest(comm)
        if device_graph:
            set_graph_device(f, specs[r])
        else:
            f.set_graph_spec(specs[r])
        f.setup(setup_alg)
        bufs = [to_dev(d[r]) for d in data]
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            if one_shot:  # sfg_bcast & co: Begin + End back to back (no p2p stream fork)
                one = {"bcast": lambda: sf.bcast(f, unit, bufs[0], bufs[1], rop, stream, sync=False),
                       "reduce": lambda: sf.reduce(f, unit, bufs[0], bufs[1], rop, stream, sync=False),
                       "fetch_and_op": lambda: sf.fetch_and_op(f, unit, bufs[0], bufs[1], bufs[2], rop, stream,
                                                               sync=False),
                       "gather": lambda: sf.gather(f, unit, bufs[0], bufs[1], stream, sync=False),
                       "scatter": lambda: sf.scatter(f, unit, bufs[0], bufs[1], stream, sync=False)}
                one[opkind]()
            elif opkind == "bcast":
                h = sf.bcast_begin(f, unit, bufs[0], bufs[1], rop, stream)
                sf.bcast_end(h)
            elif opkind == "reduce":
                h = sf.reduce_begin(f, unit, bufs[0], bufs[1], rop, stream)
                sf.reduce_end(h)
            elif opkind == "fetch_and_op":
                h = sf.fetch_and_op_begin(f, unit, bufs[0], bufs[1], bufs[2], rop, stream)
                sf.fetch_and_op_end(h)
            elif opkind == "gather":
                h = sf.gather_begin(f, unit, bufs[0], bufs[1], stream)
                sf.gather_end(h)
            elif opkind == "scatter":
                h = sf.scatter_begin(f, unit, bufs[0], bufs[1], stream)
                sf.scatter_end(h)
            else:
                raise ValueError(opkind)
        stream.synchronize()
        return [to_host(b) for b in bufs]

    per_rank = sf.run_ranks(cfg, body, devices=devices)
    return [[per_rank[r][i] for r in range(n)] for i in range(len(data))]


def assert_same(got, want, fp_tol: bool = False, what: str = ""):
    for r, (g, w) in enumerate(zip(got, want)):
        g = np.asarray(g)
        w = np.asarray(w)
        assert g.shape == w.shape, f"{what} rank {r}: shape {g.shape} vs {w.shape}"
        if fp_tol and g.dtype == np.float64:
            tol = FP_RTOL * np.maximum(1.0, np.maximum(np.abs(g), np.abs(w)))
            bad = np.abs(g - w) > tol
            assert not bad.any(), f"{what} rank {r}: {bad.sum()} values outside 1e-12 tolerance"
        else:
            if g.dtype == np.float64:
                eq = (g.view(np.int64) == w.view(np.int64))
            else:
                eq = g == w
            if not eq.all():
                i = int(np.argmin(eq))
                raise AssertionError(f"{what} rank {r}: {int((~eq).sum())} mismatches, first at "
                                     f"{i}: got {g.ravel()[i]} want {w.ravel()[i]}")


def rank_data(specs, seed: int, dtype, blocklen: int = 1, salt0: int = 100, which: str = "root",
              lo: int = -1000, hi: int = 1000):
    """Per-rank arrays sized nroots (which='root') or leaf bound ('leaf')."""
    from paper_2102_13018_b200 import graphs

    out = []
    for r, s in enumerate(specs):
        n = (int(s.nroots) if which == "root" else s.leaf_bound()) * blocklen
        if np.dtype(dtype) == np.float64:
            out.append(graphs.gen_f64(seed, salt0 + r, n))
        elif np.dtype(dtype) == np.uint8:
            out.append((graphs.gen_ints(seed, salt0 + r, n, 0, 255)).astype(np.uint8))
        else:
            out.append(graphs.gen_ints(seed, salt0 + r, n, lo, hi).astype(dtype))
    return out


def load_golden_cases(path=None):
    """Cases of tests/golden/ref_random.npz (reference-library outputs)."""
    import os

    path = path or os.path.join(os.path.dirname(__file__), "golden", "ref_random.npz")
    z = np.load(path)
    cases = []
    for ci in range(int(z["ncases"][0])):
        k = f"c{ci}"
        opk, dt, op, bl, nranks, seed = [str(x) for x in z[f"{k}/meta"]]
        nranks, bl = int(nranks), int(bl)
        specs, ins, outs = [], [], []
        nin = sum(1 for key in z.files if key.startswith(f"{k}/r0/in"))
        nout = sum(1 for key in z.files if key.startswith(f"{k}/r0/out"))
        for r in range(nranks):
            nroots, nleaves, has_local = (int(x) for x in z[f"{k}/r{r}/shape"])
            specs.append(sf.GraphSpec(nroots, nleaves, z[f"{k}/r{r}/local"] if has_local else None,
                                      z[f"{k}/r{r}/rr"], z[f"{k}/r{r}/ro"]))
        ins = [[z[f"{k}/r{r}/in{i}"] for r in range(nranks)] for i in range(nin)]
        outs = [[z[f"{k}/r{r}/out{i}"] for r in range(nranks)] for i in range(nout)]
        cases.append((opk, dt, op, bl, specs, ins, outs))
    return cases
