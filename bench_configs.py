#!/usr/bin/env python
"""Secondary benchmarks for the BASELINE configurations other than the
headline (bench.py runs config 2). One JSON line per measurement.

  config 1  single rank, 4,194,304 leaves -> 1,048,576 random roots, f64:
            Bcast REPLACE and Reduce SUM (deterministic and free-order)
  config 3  27-point Laplacian ghost-column SF, 400^3, 8 ranks (2x2x2),
            natural and locally permuted numbering: Bcast REPLACE, Reduce SUM
  config 4  16,777,216 leaves -> 65,536 roots (degree 256): Reduce SUM and
            FetchAndOp SUM, f64 and i64, deterministic and free-order
  config 5  2-rank ping-pong (bench.cpp:24-100 shape): Bcast REPLACE +
            Reduce REPLACE per iteration, half round trip, 8 B .. 256 MB

Run on one GPU: `python bench_configs.py --config 1`; multi-GPU with
torch.distributed.run (one process per GPU, NCCL). `--cpu` also times the
reference library (oracle/_ref) on the same graph (rank 0, single process).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


class Ctx:
    def __init__(self, deterministic=True, transport="p2p"):
        self.transport = transport
        import torch

        from paper_2102_13018_b200 import sf

        self.sf = sf
        self.torch = torch
        self.rank, self.world, self.local = env()
        torch.cuda.set_device(self.local)
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist

            if not dist.is_initialized():
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.dist = dist
        self.stream = torch.cuda.Stream()
        self.comms = {}

    def comm(self, deterministic=True):
        sf = self.sf
        if deterministic in self.comms:
            return self.comms[deterministic]
        if self.world > 1:
            obj = [sf.nccl_unique_id() if self.rank == 0 else None]
            self.dist.broadcast_object_list(obj, src=0)
            c = sf.Comm(self.world, self.rank, self.local,
                        sf.CommConfig(nranks=self.world, backend=self.transport,
                                      deterministic=deterministic),
                        nccl_id=obj[0])
        else:
            c = sf.Comm(1, 0, self.local, sf.CommConfig(nranks=1, deterministic=deterministic))
        self.comms[deterministic] = c
        return c

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def vmax(self, x):
        if not self.dist:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def vsum(self, x):
        if not self.dist:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t)
        return float(t.item())

    def timed(self, fn, steps, warmup, flush=True):
        torch, sf = self.torch, self.sf
        with torch.cuda.stream(self.stream):
            for _ in range(warmup):
                fn()
        torch.cuda.synchronize()
        self.barrier()
        sf.timing_collect()
        # Flush L2 before every timed call: the config-1/4 working sets fit in
        # the 126 MB L2 and would otherwise be timed hot. The flush READS a
        # 256 MB buffer (L2 left full of clean lines): a write-based flush
        # leaves ~126 MB of dirty lines whose write-back would be charged to
        # the timed kernel.
        flush_buf = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
        flush_out = torch.empty((), dtype=torch.int64, device="cuda")
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        sf.timing_enable(True)
        with torch.cuda.stream(self.stream):
            for e0, e1 in evs:
                if flush:
                    torch.sum(flush_buf, dim=0, dtype=torch.int64, out=flush_out)
                e0.record(self.stream)
                fn()
                e1.record(self.stream)
        torch.cuda.synchronize()
        sf.timing_enable(False)
        rec = sf.timing_collect()
        ms = self.vmax(sum(a.elapsed_time(b) for a, b in evs) / steps)
        byts = self.vsum(sum(v["bytes"] for v in rec.values()) / steps)
        self.barrier()
        return ms, byts, rec


def timed_graph(ctx, fn, steps, warmup, reps=5):
    """Device-side time per call: `steps` calls captured into one CUDA graph
    (the library's work is all stream-ordered kernels / NCCL calls, no host
    synchronisation), replayed `reps` times; median per call, max over ranks.
    Removes the Python/ctypes launch overhead that bounds latency-size
    operations when they are issued eagerly."""
    torch = ctx.torch
    with torch.cuda.stream(ctx.stream):
        for _ in range(warmup):
            fn()
    torch.cuda.synchronize()
    ctx.barrier()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=ctx.stream):
        for _ in range(steps):
            fn()
    torch.cuda.synchronize()
    ctx.barrier()
    g.replay()
    torch.cuda.synchronize()
    ctx.barrier()
    per = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.barrier()
        with torch.cuda.stream(ctx.stream):
            # the first replay absorbs the ranks' start skew after the
            # barrier (their exchanges couple them); the second, issued right
            # behind it, is timed: the steady-state period per call
            g.replay()
            e0.record(ctx.stream)
            g.replay()
            e1.record(ctx.stream)
        torch.cuda.synchronize()
        per.append(e0.elapsed_time(e1) / steps)
    ctx.barrier()
    del g
    return ctx.vmax(statistics.median(per))


def timed_graph_flushed(ctx, fn, steps=10, reps=5):
    """Device time per call with a cold L2: a CUDA graph of `steps` x
    [L2 read-flush, call] minus a graph of `steps` x [flush] (same stream),
    median over `reps` replays, max over ranks. No host launch gap inside the
    measurement (the eager per-call events include the Python/ctypes time it
    takes to issue Begin/End after the flush)."""
    torch = ctx.torch
    flush_buf = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
    flush_out = torch.empty((), dtype=torch.int64, device="cuda")

    def flush():
        torch.sum(flush_buf, dim=0, dtype=torch.int64, out=flush_out)

    with torch.cuda.stream(ctx.stream):
        for _ in range(2):
            flush()
            fn()
    torch.cuda.synchronize()
    ctx.barrier()
    gs = []
    for with_op in (True, False):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=ctx.stream):
            for _ in range(steps):
                flush()
                if with_op:
                    fn()
        gs.append(g)
    torch.cuda.synchronize()
    ctx.barrier()
    t = {}
    for name, g in zip(("op", "flush"), gs):
        g.replay()
        torch.cuda.synchronize()
        per = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ctx.barrier()
            with torch.cuda.stream(ctx.stream):
                e0.record(ctx.stream)
                g.replay()
                e1.record(ctx.stream)
            torch.cuda.synchronize()
            per.append(e0.elapsed_time(e1) / steps)
        t[name] = statistics.median(per)
    ctx.barrier()
    del gs
    return ctx.vmax(t["op"] - t["flush"])


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def emit(ctx, d):
    if ctx.rank == 0:
        print(json.dumps(d), flush=True)


def op_line(ctx, config, name, ms, byts, rec, extra=None):
    gbs = byts / (ms * 1e-3) / 1e9
    dom = max(rec.items(), key=lambda kv: kv[1]["total_ms"]) if rec else (None, None)
    d = {"config": config, "op": name, "n_gpus": ctx.world, "us_per_op": ms * 1e3,
         "GBps": gbs, "frac_hbm": gbs / peak() if ctx.world == 1 else None,
         "kernels": {k: {"launches": v["launches"], "us": 1e3 * v["total_ms"] / v["launches"],
                         "GBps": v["bytes"] / max(1e-12, v["total_ms"] * 1e-3) / 1e9,
                         "link_GBps": v.get("link_bytes", 0) / max(1e-12, v["total_ms"] * 1e-3) / 1e9}
                     for k, v in rec.items()},
         "dominant": dom[0]}
    lrec = [v for v in rec.values() if v.get("link_bytes", 0) > 0]
    if ctx.world > 1:
        lb = sum(v["link_bytes"] for v in lrec)
        lms = sum(v["total_ms"] for v in lrec)
        g = lb / (lms * 1e-3) / 1e9 if lms > 0 else 0.0
        d["transport"] = ctx.transport
        d["nvlink"] = {"GBps_min_rank": -ctx.vmax(-g), "frac_of_900": -ctx.vmax(-g) / 900.0,
                       "bytes_per_op_rank0": lb / max(1, sum(v["launches"] for v in lrec)),
                       "us_exchange_max_rank": ctx.vmax(1e3 * lms / max(1, sum(v["launches"] for v in lrec)))}
    d.update(extra or {})
    emit(ctx, d)


def setup_forest(ctx, spec, deterministic=True):
    f = ctx.sf.StarForest(ctx.comm(deterministic))
    f.set_graph_spec(spec)
    t0 = time.perf_counter()
    f.setup()
    return f, time.perf_counter() - t0


# ------------------------------------------------------------------ config 1
def config1(ctx, args):
    from paper_2102_13018_b200 import graphs

    torch, sf = ctx.torch, ctx.sf
    L, R = 4194304, 1048576
    specs = graphs.random_leaf_root(L, R, ctx.world, seed=1)
    spec = specs[ctx.rank]
    u = sf.Unit(sf.Kind.float64)
    root = torch.from_numpy(graphs.gen_f64(1, 100 + ctx.rank, int(spec.nroots))).cuda()
    leaf = torch.from_numpy(graphs.gen_f64(1, 200 + ctx.rank, spec.leaf_bound())).cuda()
    for det in (True, False):
        f, setup_s = setup_forest(ctx, spec, det)

        def bc():
            h = sf.bcast_begin(f, u, root, leaf, sf.ReduceOp.replace, ctx.stream)
            sf.bcast_end(h)

        def rd():
            h = sf.reduce_begin(f, u, leaf, root, sf.ReduceOp.sum, ctx.stream)
            sf.reduce_end(h)

        for name, fn in (("bcast_replace", bc), ("reduce_sum", rd)):
            ms, byts, rec = ctx.timed(fn, args.steps, args.warmup)
            gms = timed_graph_flushed(ctx, fn)
            op_line(ctx, 1, name, ms, byts, rec, {"deterministic": det, "setup_s": setup_s,
                                                   "L": L, "R": R, "dtype": "f64",
                                                   "graph_us_per_op": gms * 1e3,
                                                   "graph_GBps": byts / (gms * 1e-3) / 1e9,
                                                   "graph_frac_hbm": byts / (gms * 1e-3) / 1e9 / peak()})
    if args.cpu and ctx.world == 1 and ctx.rank == 0:
        from oracle import ref

        if ref.available():
            for opk, op in (("bcast", "replace"), ("reduce", "sum")):
                t = ref.time_op(specs, opk, "float64", op, 3, 1)
                emit(ctx, {"config": 1, "op": f"{opk}_{op}", "impl": "reference_cpu", "cores": 1,
                           "us_per_op": t["us_per_call"], "setup_s": t["setup_s"]})


# ------------------------------------------------------------------ config 2
def config2(ctx, args):
    """Halo-only variant (ii) of config 2: the ghost-face
    SF of the 512^3 grid without the interior self edges, so Bcast/Reduce are
    pure remote exchanges (pack -> NVLink -> unpack). Latency-reported."""
    from paper_2102_13018_b200 import graphs

    torch, sf = ctx.torch, ctx.sf
    N = args.n2
    spec = graphs.g2l_halo(N, ctx.world, ctx.rank, interior=False)
    geo = graphs.G2L(N, ctx.world, ctx.rank)
    f, setup_s = setup_forest(ctx, spec)
    u = sf.Unit(sf.Kind.float64)
    root = torch.rand(geo.n_owned, dtype=torch.float64, device="cuda")
    leaf = torch.zeros(geo.n_local, dtype=torch.float64, device="cuda")

    def bc():
        h = sf.bcast_begin(f, u, root, leaf, sf.ReduceOp.replace, ctx.stream)
        sf.bcast_end(h)

    def rd():
        h = sf.reduce_begin(f, u, leaf, root, sf.ReduceOp.sum, ctx.stream)
        sf.reduce_end(h)

    if os.environ.get("SFG_TRACE_LAUNCHES"):
        # debug: in-kernel timestamps of 20 captured Bcasts, replayed once
        g = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=ctx.stream):
            for _ in range(20):
                bc()
        torch.cuda.synchronize()
        ctx.barrier()
        g.replay()
        torch.cuda.synchronize()
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        sf._lib().sfg_trace_dump(os.path.join(ROOT, "gpurun_out", f"trace_cfg2_r{ctx.rank}.jsonl").encode())
        del g
    def bc1():  # one-shot forms (ops.hpp:60, 68): no caller work between the halves
        sf.bcast(f, u, root, leaf, sf.ReduceOp.replace, ctx.stream, sync=False)

    def rd1():
        sf.reduce(f, u, leaf, root, sf.ReduceOp.sum, ctx.stream, sync=False)

    for name, fn, fn1 in (("bcast_replace", bc, bc1), ("reduce_sum", rd, rd1)):
        ms, byts, rec = ctx.timed(fn, args.steps, args.warmup, flush=False)
        gms = timed_graph(ctx, fn, args.steps, args.warmup)
        gms1 = timed_graph(ctx, fn1, args.steps, args.warmup)
        nbytes = ctx.vmax(float(sum(v.get("link_bytes", 0) for v in rec.values()) / args.steps))
        op_line(ctx, 2, name, ms, byts, rec, {"variant": "halo-only", "grid": [N] * 3,
                                               "nleaves_rank0": int(spec.nleaves), "setup_s": setup_s,
                                               "graph_us_per_op": gms * 1e3,
                                               "graph_link_GBps_max_rank_egress": nbytes / (gms * 1e-3) / 1e9,
                                               "graph_us_per_op_one_shot": gms1 * 1e3,
                                               "graph_link_GBps_one_shot": nbytes / (gms1 * 1e-3) / 1e9})


# ------------------------------------------------------------------ config 4
def config4(ctx, args):
    from paper_2102_13018_b200 import graphs

    torch, sf = ctx.torch, ctx.sf
    L, R = 16777216, 65536
    specs = graphs.random_leaf_root(L, R, ctx.world, seed=4)
    spec = specs[ctx.rank]
    for det in (True, False):
        f, setup_s = setup_forest(ctx, spec, det)
        for dt, kind in (("f64", sf.Kind.float64), ("i64", sf.Kind.int64)):
            u = sf.Unit(kind)
            tdt = torch.float64 if dt == "f64" else torch.int64
            root = torch.ones(int(spec.nroots), dtype=tdt, device="cuda")
            leaf = torch.ones(spec.leaf_bound(), dtype=tdt, device="cuda")
            upd = torch.zeros_like(leaf)

            def rd():
                h = sf.reduce_begin(f, u, leaf, root, sf.ReduceOp.sum, ctx.stream)
                sf.reduce_end(h)

            def fo():
                h = sf.fetch_and_op_begin(f, u, root, leaf, upd, sf.ReduceOp.sum, ctx.stream)
                sf.fetch_and_op_end(h)

            for name, fn in (("reduce_sum", rd), ("fetch_and_op_sum", fo)):
                ms, byts, rec = ctx.timed(fn, args.steps, args.warmup)
                gms = timed_graph_flushed(ctx, fn)
                op_line(ctx, 4, name, ms, byts, rec, {"deterministic": det, "dtype": dt,
                                                       "setup_s": setup_s, "L": L, "R": R,
                                                       "graph_us_per_op": gms * 1e3,
                                                       "graph_GBps": byts / (gms * 1e-3) / 1e9,
                                                       "graph_frac_hbm": byts / (gms * 1e-3) / 1e9 / peak()})
    if args.cpu and ctx.world == 1 and ctx.rank == 0:
        from oracle import ref

        if ref.available():
            for opk in ("reduce", "fetch_and_op"):
                for dt in ("float64", "int64"):
                    t = ref.time_op(specs, opk, dt, "sum", 3, 1)
                    emit(ctx, {"config": 4, "op": f"{opk}_sum", "dtype": dt, "impl": "reference_cpu",
                               "cores": 1, "us_per_op": t["us_per_call"], "setup_s": t["setup_s"]})


# ------------------------------------------------------------------ config 5
def config5(ctx, args):
    from paper_2102_13018_b200 import graphs

    torch, sf = ctx.torch, ctx.sf
    assert ctx.world == 2, "config 5 needs exactly 2 ranks"
    u = sf.Unit(sf.Kind.int64)
    size = 8
    rows = []
    while size <= args.max_bytes:
        specs = graphs.pingpong(size)
        n = size // 8
        f, _ = setup_forest(ctx, specs[ctx.rank])
        root = torch.arange(n if ctx.rank == 0 else 0, dtype=torch.int64, device="cuda")
        leaf = torch.zeros(n if ctx.rank == 1 else 0, dtype=torch.int64, device="cuda")
        iters = 50 if size <= (1 << 20) else 10
        dev_us, host_us = [], []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for it in range(5 + iters):
            torch.cuda.synchronize()
            ctx.barrier()
            t0 = time.perf_counter()
            with torch.cuda.stream(ctx.stream):
                e0.record(ctx.stream)
                # the one-shot forms, as the reference's ping-pong (bench.cpp:65-66)
                sf.bcast(f, u, root, leaf, sf.ReduceOp.replace, ctx.stream, sync=False)
                sf.reduce(f, u, leaf, root, sf.ReduceOp.replace, ctx.stream, sync=False)
                e1.record(ctx.stream)
            ctx.stream.synchronize()
            t1 = time.perf_counter()
            if it >= 5:
                dev_us.append(e0.elapsed_time(e1) * 1e3 / 2)
                host_us.append((t1 - t0) * 1e6 / 2)
        ok = True
        if ctx.rank == 1:
            ok = bool((leaf.cpu() == torch.arange(n)).all()) if n else True

        def rt():
            sf.bcast(f, u, root, leaf, sf.ReduceOp.replace, ctx.stream, sync=False)
            sf.reduce(f, u, leaf, root, sf.ReduceOp.replace, ctx.stream, sync=False)

        def rt_split():  # split-phase Begin/End (exchange on a forked stream)
            h = sf.bcast_begin(f, u, root, leaf, sf.ReduceOp.replace, ctx.stream)
            sf.bcast_end(h)
            h = sf.reduce_begin(f, u, leaf, root, sf.ReduceOp.replace, ctx.stream)
            sf.reduce_end(h)

        reps = 20 if size <= (1 << 22) else 4
        graph_half = timed_graph(ctx, rt, reps, 2) * 1e3 / 2
        graph_half_split = timed_graph(ctx, rt_split, reps, 2) * 1e3 / 2
        if ctx.rank == 1:
            ok = ok and (bool((leaf.cpu() == torch.arange(n)).all()) if n else True)
        dmed = ctx.vmax(statistics.median(dev_us))
        dmin = ctx.vmax(min(dev_us))
        hmed = ctx.vmax(statistics.median(host_us))
        rows.append({"bytes": size, "half_rtt_us_median": dmed, "half_rtt_us_min": dmin,
                     "host_half_rtt_us_median": hmed, "GBps": size / (dmed * 1e-6) / 1e9,
                     "graph_half_rtt_us": graph_half, "graph_GBps": size / (graph_half * 1e-6) / 1e9,
                     "graph_half_rtt_us_split_phase": graph_half_split,
                     "payload_ok": ok})
        del f
        size *= 2
    emit(ctx, {"config": 5, "op": "pingpong_bcast+reduce_replace", "n_gpus": 2,
               "transport": ctx.transport, "rows": rows})
    if args.cpu and ctx.rank == 0:
        # the reference's own ping-pong (bench.cpp:24-100) on this box's host,
        # 2 rank threads, sizes x4 from 8 B (its sweep step)
        from oracle import ref

        if ref.available():
            import os as _os
            cores = len(_os.sched_getaffinity(0)) if hasattr(_os, "sched_getaffinity") else _os.cpu_count()
            rrows = ref.pingpong(8, min(args.max_bytes, 64 << 20), iters=20, warmup=3)
            emit(ctx, {"config": 5, "op": "pingpong_bcast+reduce_replace", "impl": "reference_cpu",
                       "cores": 2, "host_cores": cores, "rows": rrows,
                       "what": "sf::pingpong (bench.cpp:24-100), threads backend, median/min half RTT"})


# ------------------------------------------------------- config 3 consumer
def config3_spmv(ctx, args):
    """The ghost exchange inside its caller: y = A x with the
    27-point Laplacian on an N^3 grid, one block of rows per GPU
    (proc_grid(world)), spmv.hpp:149-157 on the device — the ghost Bcast is
    overlapped with the diagonal-block product. Reported beside the same
    product run without overlap (Bcast completed before the diagonal
    product); graph-replay device time, eager (instrumented) period and the
    per-kernel times of the eager run beside it."""
    from paper_2102_13018_b200 import graphs
    from paper_2102_13018_b200 import spmv as S

    torch, sf = ctx.torch, ctx.sf
    N = args.n3_spmv
    dims = graphs.proc_grid(ctx.world)
    t0 = time.perf_counter()
    (rp, ci, vals), layout = S.laplacian27_block(N, dims, ctx.rank)
    m = S.split_rows(rp, ci, vals, layout, ctx.rank)
    gen_s = time.perf_counter() - t0
    comm = ctx.comm(True)
    f = S.build_ghost_sf(comm, m)
    D, B = S.Matrix(comm, m.diag), S.Matrix(comm, m.offdiag)
    n = layout.local_size(ctx.rank)
    x = torch.cos(torch.arange(n, dtype=torch.float64, device="cuda") * 0.37)
    lvec = torch.zeros(len(m.garray), dtype=torch.float64, device="cuda")
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    u = sf.Unit(sf.Kind.float64)

    def overlapped():
        S.spmv(f, D, B, x, lvec, y, ctx.stream)

    def serial():  # exchange first, then both products (no overlap)
        h = sf.bcast_begin(f, u, x, lvec, sf.ReduceOp.replace, ctx.stream)
        sf.bcast_end(h)
        S.spmv(f, D, B, x, lvec, y, ctx.stream)

    nnz = ctx.vsum(float(m.diag.rowptr[-1] + m.offdiag.rowptr[-1]))
    res = {}
    for name, fn in (("spmv_overlapped", overlapped), ("exchange_then_spmv", serial)):
        ms, byts, rec = ctx.timed(fn, args.steps, args.warmup, flush=False)
        res[name] = (ms, byts, rec)
    e_o, byts, rec = res["spmv_overlapped"]
    e_s = res["exchange_then_spmv"][0]
    # Headline: the same two sequences captured into a CUDA graph and
    # replayed warm (the working set is ~10x the L2): device time without the
    # eager, instrumented issue path (per-kernel events, ctypes), which bounds
    # the eager period at N>1 where the ranks' exchanges couple them.
    ms_o = timed_graph(ctx, overlapped, 20, 3)
    ms_s = timed_graph(ctx, serial, 20, 3)

    def transpose():  # spmv.hpp:161-169: y = A^T x; lvec = B^T x; Reduce SUM lvec -> y
        S.spmv_transpose(f, D, B, x, lvec, y, ctx.stream)

    ms_t = timed_graph(ctx, transpose, 20, 3)
    kern = {k: 1e3 * v["total_ms"] / v["launches"] for k, v in rec.items()}
    emit(ctx, {"config": 3, "op": "spmv_27pt", "n_gpus": ctx.world, "grid": [N] * 3,
               "dims": list(dims), "rows": layout.total(), "nnz": nnz,
               "us_per_spmv": ms_o * 1e3, "us_exchange_then_spmv": ms_s * 1e3,
               "us_per_spmv_eager": e_o * 1e3, "us_exchange_then_spmv_eager": e_s * 1e3,
               "us_per_spmv_transpose": ms_t * 1e3,
               "GFLOPs": 2 * nnz / (ms_o * 1e-3) / 1e9,
               "GBps_algorithmic": byts / (ms_o * 1e-3) / 1e9,
               "frac_hbm_per_gpu": byts / ctx.world / (ms_o * 1e-3) / 1e9 / peak(),
               "kernels_us_rank0": kern, "transport": ctx.transport, "gen_s": gen_s,
               "ghosts_rank0": len(m.garray)})


# ------------------------------------------------------------------ config 3
def config3(ctx, args):
    """The ghost-column SF of the 27-point Laplacian. Under torchrun (world
    > 1): one process per GPU over proc_grid(world) blocks (BASELINE config 3
    is 8 ranks = 2x2x2; with fewer GPUs the same grid is cut into world
    blocks), transport --transport, eager and CUDA-graph timings. Single
    process: 8 thread ranks spread over the visible GPUs with the in-process
    transport (peer copies), reported as such."""
    import threading

    from paper_2102_13018_b200 import graphs

    torch, sf = ctx.torch, ctx.sf
    N = args.n3
    dims = graphs.proc_grid(ctx.world) if ctx.world > 1 else (2, 2, 2)
    nr = dims[0] * dims[1] * dims[2]
    for permute in (None, 3):
        specs = [graphs.laplacian27_ghosts(N, dims, r, permute) for r in range(nr)]
        if ctx.world > 1:
            f, setup_s = setup_forest(ctx, specs[ctx.rank])
            u = sf.Unit(sf.Kind.float64)
            root = torch.rand(int(specs[ctx.rank].nroots), dtype=torch.float64, device="cuda")
            leaf = torch.zeros(specs[ctx.rank].leaf_bound(), dtype=torch.float64, device="cuda")

            def bc():
                h = sf.bcast_begin(f, u, root, leaf, sf.ReduceOp.replace, ctx.stream)
                sf.bcast_end(h)

            def rd():
                h = sf.reduce_begin(f, u, leaf, root, sf.ReduceOp.sum, ctx.stream)
                sf.reduce_end(h)

            def bc1():  # one-shot forms (the ghost update of a VecScatter)
                sf.bcast(f, u, root, leaf, sf.ReduceOp.replace, ctx.stream, sync=False)

            def rd1():
                sf.reduce(f, u, leaf, root, sf.ReduceOp.sum, ctx.stream, sync=False)

            for name, fn, fn1 in (("bcast_replace", bc, bc1), ("reduce_sum", rd, rd1)):
                ms, byts, rec = ctx.timed(fn, args.steps, args.warmup, flush=False)
                gms = timed_graph(ctx, fn, args.steps, args.warmup)
                gms1 = timed_graph(ctx, fn1, args.steps, args.warmup)
                op_line(ctx, 3, name, ms, byts, rec, {"permuted": permute is not None, "N": N,
                                                       "dims": list(dims), "setup_s": setup_s,
                                                       "ghosts_rank0": int(specs[0].nleaves),
                                                       "graph_us_per_op": gms * 1e3,
                                                       "graph_us_per_op_one_shot": gms1 * 1e3})
            continue
        if ctx.rank != 0:
            continue
        ng = torch.cuda.device_count()
        devices = [r * ng // 8 for r in range(8)]
        res = {}

        def body(comm):
            r = comm.rank()
            f = sf.StarForest(comm)
            f.set_graph_spec(specs[r])
            f.setup()
            u = sf.Unit(sf.Kind.float64)
            root = torch.rand(int(specs[r].nroots), dtype=torch.float64, device="cuda")
            leaf = torch.zeros(specs[r].leaf_bound(), dtype=torch.float64, device="cuda")
            st = torch.cuda.Stream()
            out = {}
            for name, opf in (("bcast_replace", lambda: sf.bcast_end(sf.bcast_begin(
                    f, u, root, leaf, sf.ReduceOp.replace, st))),
                              ("reduce_sum", lambda: sf.reduce_end(sf.reduce_begin(
                                  f, u, leaf, root, sf.ReduceOp.sum, st)))):
                with torch.cuda.stream(st):
                    for _ in range(3):
                        opf()
                st.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(st):
                    e0.record(st)
                    for _ in range(args.steps):
                        opf()
                    e1.record(st)
                st.synchronize()
                out[name] = e0.elapsed_time(e1) * 1e3 / args.steps
            return out

        got = sf.run_ranks(sf.CommConfig(nranks=8, timeout_s=120), body, devices=devices)
        for name in ("bcast_replace", "reduce_sum"):
            emit(ctx, {"config": 3, "op": name, "permuted": permute is not None, "N": N,
                       "ranks": 8, "gpus": ng, "transport": "threads (peer copies)",
                       "us_per_op_max_rank": max(g[name] for g in got)})


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, required=True)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--cpu", action="store_true")
    p.add_argument("--max-bytes", type=int, default=256 << 20)
    p.add_argument("--n3", type=int, default=400)
    p.add_argument("--n2", type=int, default=512)
    p.add_argument("--n3-spmv", type=int, default=160)
    p.add_argument("--spmv", action="store_true", help="config 3: the SpMV consumer")
    p.add_argument("--transport", default="p2p", choices=["p2p", "nccl"])
    args = p.parse_args()
    ctx = Ctx(transport=args.transport)
    if args.config == 3 and args.spmv:
        config3_spmv(ctx, args)
    else:
        {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}[args.config](ctx, args)
    if ctx.dist:
        ctx.dist.barrier()
        ctx.dist.destroy_process_group()


if __name__ == "__main__":
    main()
