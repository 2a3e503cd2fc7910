#!/usr/bin/env python
"""Benchmark of the star-forest Bcast+Reduce path on B200 (BASELINE config 2).

Workload: the PETSc DMDA global->local star forest of a 512^3 float64 grid
with a 7-point (star) stencil, block-partitioned over the N ranks of the run
(1x1x1, 1x1x2, 1x2x2, 2x2x2): every rank's interior 3-D subblock (self
edges, Affine3D pattern) plus ghost faces from its neighbours (remote edges,
NCCL). One step = Bcast(REPLACE) global->local + Reduce(SUM) local->global
through the C ABI, all ranks, stream-ordered. Total grid fixed as N grows
("strong" scaling). Arrays are 1+ GB per rank, far above the 126 MB L2, so no
flush is needed between iterations.

value   = algorithmic bytes of all ranks' launches per step / max-over-ranks
          device time per step (GB/s); ms_per_step, us_per_op beside it.
e2e     = same metric through the public API with the root vector copied in
          from pinned host memory and read back every step.
roofline: dominant kernel's algorithmic bytes per launch / its CUDA-event
          duration on the launching stream, against MEASURED_PEAKS.json.
cpu_baseline: the unmodified reference library (oracle/_ref) timed on the
          box's host on a bounded slab of the same workload.

`--impl reference` runs the reference arm instead (rank 0 only under torchrun).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SF Bcast+Reduce GB/s and µs/op on 3D 7-pt halo SF at 1/2/4/8 B200"
HBM_FALLBACK = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--N", type=int, default=512)
    p.add_argument("--e2e-steps", type=int, default=32)
    p.add_argument("--sample-nz", type=int, default=64, help="reference sample: z planes per rank")
    p.add_argument("--sample-steps", type=int, default=10)
    p.add_argument("--ref-threads", type=int, default=0,
                   help="reference arm: rank threads (the reference parallelises by ranks only); "
                        "0 = every host core (max 32), at least one per GPU")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-device-setup", action="store_true")
    p.add_argument("--graph", action="store_true",
                   help="timed steps replay one CUDA graph of a step (captured after warm-up)")
    p.add_argument("--dims", type=lambda v: tuple(int(x) for x in v.split(",")), default=None,
                   help="process grid px,py,pz (default: 1x1x2 / 1x2x2 / 2x2x2 for 2 / 4 / 8 GPUs)")
    p.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                   help="remote exchange at N>1: one-sided NVLink puts (p2p) or grouped NCCL send/recv")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.lines: list[str] = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu_id}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def wait_first(self, timeout=5.0):
        """Block until nvidia-smi is producing samples (its start-up takes
        longer than a short timed region)."""
        t0 = time.perf_counter()
        while self.proc is not None and not self.lines and time.perf_counter() - t0 < timeout:
            time.sleep(0.01)

    def mark(self):
        return time.perf_counter()

    def stop(self, window=None) -> dict:
        """Samples taken inside `window` = (t0, t1) (host perf_counter around
        the timed region), plus the one just before and after it when the
        region is shorter than the sampling period."""
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if window is not None:
            t0, t1 = window
            inside = [x for x in lines if t0 <= x[0] <= t1]
            before = [x for x in lines if x[0] < t0][-1:]
            after = [x for x in lines if x[0] > t1][:1]
            lines = before + inside + after
        for _, ln in lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def g2l_step_bytes(geo) -> float:
    """Algorithmic bytes per Bcast(REPLACE)+Reduce(SUM) of one rank, f64:
    interior self edges 8+8 (bcast) + 8+16 (reduce) per point; ghost faces
    are packed/unpacked from HBM on both ends (counted by the library)."""
    return 40.0 * geo.n_owned


# ------------------------------------------------------------- reference arm
def reference_arm(args, rank, world):
    if rank != 0:
        return
    from oracle import ref
    from paper_2102_13018_b200 import graphs

    # The reference is single-threaded per rank; its only host parallelism is
    # more rank threads (run_ranks, threads backend). Use every host core: the
    # sample grid is decomposed over P rank threads, sample_nz planes each.
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    P = args.ref_threads if args.ref_threads > 0 else max(world, min(cores, 32))
    sample = (args.N, args.N, min(args.N, args.sample_nz * P))
    line = {"impl": "reference", "metric": METRIC, "unit": "GB/s", "higher_is_better": True,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup}
    if not ref.available():
        line["unavailable"] = "oracle/_ref/libsfref.so not built (needs /root/reference at build time)"
        print(json.dumps(line))
        return
    specs = [graphs.g2l_halo(sample, P, r) for r in range(P)]
    geo = [graphs.G2L(sample, P, r) for r in range(P)]
    steps = max(1, min(args.steps, args.sample_steps))
    t = ref.time_bcast_reduce(specs, steps, 1)
    byts = sum(g2l_step_bytes(g) for g in geo)
    gbs = byts / (t["us_per_step"] * 1e-6) / 1e9
    line.update({
        "value": gbs, "ms_per_step": t["us_per_step"] / 1e3,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "g2l_halo_7pt", "grid": [args.N] * 3, "parallelism": f"sf{P}",
                   "sample_grid": list(sample), "setup_s": t["setup_s"],
                   "bcast_us": t["bcast_us"], "reduce_us": t["reduce_us"]},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": P, "kind": "reference",
                         "sample": f"G2L {sample[0]}x{sample[1]}x{sample[2]} over {P} rank thread(s), "
                                   f"{steps} timed steps; host has {cores} cores"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })
    print(json.dumps(line))


# ------------------------------------------------------------------ our arm
def cpu_baseline(args):
    from oracle import ref
    from paper_2102_13018_b200 import graphs

    if not ref.available():
        return None
    sample = (args.N, args.N, min(args.N, args.sample_nz))
    spec = [graphs.g2l_halo(sample, 1, 0)]
    geo = graphs.G2L(sample, 1, 0)
    t = ref.time_bcast_reduce(spec, args.sample_steps, 1)
    gbs = g2l_step_bytes(geo) / (t["us_per_step"] * 1e-6) / 1e9
    return {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "reference",
            "sample": f"G2L {sample[0]}x{sample[1]}x{sample[2]} slab, 1 rank thread, "
                      f"{args.sample_steps} timed Bcast+Reduce steps (reference is single-threaded "
                      f"per rank); SetUp {t['setup_s']:.2f} s",
            "ms_per_step": t["us_per_step"] / 1e3}


def halo_exchange(args, sf, comm, graphs, torch, rank, world, allreduce, barrier) -> dict:
    """The remote phase alone: the halo-only forest of the same grid (ghost
    faces, no interior self edges), Bcast REPLACE captured 50x in a CUDA
    graph and replayed (device time; no Python launch overhead). achieved =
    bytes this GPU sends per exchange / time per exchange, slowest rank.
    Headline: the one-shot form (sf.bcast, ops.hpp:60 — the reference's own
    ping-pong benchmark calls it); the split-phase Begin/End pair, which keeps
    the exchange on a forked stream so caller work can overlap it, beside it."""
    spec = graphs.g2l_halo(args.N, world, rank, dims=args.dims, interior=False)
    geo = graphs.G2L(args.N, world, rank, dims=args.dims)
    f = sf.StarForest(comm)
    f.set_graph_spec(spec)
    f.setup()
    del spec
    unit = sf.Unit(sf.Kind.float64)
    root = torch.rand(geo.n_owned, dtype=torch.float64, device="cuda")
    leaf = torch.zeros(geo.n_local, dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()

    def one_shot():
        sf.bcast(f, unit, root, leaf, sf.ReduceOp.replace, st, sync=False)

    def split_phase():
        sf.bcast_end(sf.bcast_begin(f, unit, root, leaf, sf.ReduceOp.replace, st))

    c0 = sf.counters()["bytes_sent"]
    with torch.cuda.stream(st):
        one_shot()
    torch.cuda.synchronize()
    sent = sf.counters()["bytes_sent"] - c0
    K = 50

    def per_exchange_ms(fn):
        for _ in range(2):
            with torch.cuda.stream(st):
                fn()
        torch.cuda.synchronize()
        barrier()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(K):
                fn()
        torch.cuda.synchronize()
        barrier()
        g.replay()
        torch.cuda.synchronize()
        best = []
        for _ in range(5):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                g.replay()  # absorbs the ranks' start skew after the barrier
                e0.record(st)
                g.replay()  # timed: steady-state period of coupled exchanges
                e1.record(st)
            torch.cuda.synchronize()
            best.append(e0.elapsed_time(e1) / K)
        del g
        return statistics.median(best)

    mine = per_exchange_ms(one_shot)
    mine_split = per_exchange_ms(split_phase)
    ms = allreduce(mine, "max")
    ms_split = allreduce(mine_split, "max")
    gbs = -allreduce(-(sent / (mine * 1e-3) / 1e9), "max")
    del f
    return {"achieved": gbs, "peak": 900.0, "peak_kind": "nominal per direction per GPU",
            "measured_peer_copy": 770.0, "unit": "GB/s", "frac": gbs / 900.0,
            "us_per_exchange": ms * 1e3, "us_per_exchange_split_phase": ms_split * 1e3,
            "bytes_per_exchange_rank0": sent,
            "what": "halo-only Bcast (ghost faces of the same grid), one-shot sf.bcast, CUDA-graph replay, "
                    "puts+receives per exchange, slowest rank; split-phase Begin/End beside it"}


def ours(args, rank, world, local):
    import torch

    from paper_2102_13018_b200 import graphs, sf

    torch.cuda.set_device(local)
    dev = local
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [sf.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = sf.Comm(world, rank, dev, sf.CommConfig(nranks=world, backend=args.transport),
                       nccl_id=obj[0])
    else:
        dist = None
        comm = sf.Comm(1, 0, dev, sf.CommConfig(nranks=1, backend="threads"))

    def barrier():
        if dist is not None:
            dist.barrier()

    def allreduce(x: float, op: str) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return float(t.item())

    t0 = time.perf_counter()
    spec = graphs.g2l_halo(args.N, world, rank, dims=args.dims)
    geo = graphs.G2L(args.N, world, rank, dims=args.dims)
    gen_s = time.perf_counter() - t0
    f = sf.StarForest(comm)
    t0 = time.perf_counter()
    f.set_graph_spec(spec)
    set_graph_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    f.setup()
    setup_s = time.perf_counter() - t0
    # The same forest planned on the device: the graph arrays
    # are uploaded first (not timed), then set_graph_device + setup are timed.
    dsetup = None
    if not args.no_device_setup:
        dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
        loc = dev(spec.local) if spec.local is not None else None
        rr, ro = dev(spec.remote_rank), dev(spec.remote_off)
        # one tiny device SetUp first: loads the planner's kernels (lazy module loading)
        fw = sf.StarForest(comm)
        fw.set_graph_device(1, 1, None, torch.tensor([rank], dtype=torch.int32, device="cuda"),
                            torch.zeros(1, dtype=torch.int64, device="cuda"))
        fw.setup()
        del fw
        runs = []
        for _ in range(2):  # first: the planner's memory pool grows; second: steady state
            fd = sf.StarForest(comm)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fd.set_graph_device(spec.nroots, spec.nleaves, loc, rr, ro)
            t1 = time.perf_counter()
            fd.setup()
            t2 = time.perf_counter()
            same = all(fd.group_plans(w) == f.group_plans(w) for w in (0, 1))
            runs.append({"set_graph_s": allreduce(t1 - t0, "max"), "setup_s": allreduce(t2 - t1, "max"),
                         "plan_equal": bool(allreduce(0.0 if same else 1.0, "sum") == 0.0)})
            del fd
        dsetup = {"first": runs[0], "steady": runs[1],
                  "note": "same forest from device arrays; max over ranks; first = the planner's "
                          "memory pool grows, steady = second SetUp in the process"}
        del loc, rr, ro
    del spec

    unit = sf.Unit(sf.Kind.float64)
    root = (1.0 + (torch.arange(geo.n_owned, device="cuda", dtype=torch.float64) % 97) * 1e-3)
    leaf = torch.zeros(geo.n_local, dtype=torch.float64, device="cuda")
    stream = torch.cuda.Stream()

    def step_on(r):
        h = sf.bcast_begin(f, unit, r, leaf, sf.ReduceOp.replace, stream)
        sf.bcast_end(h)
        h = sf.reduce_begin(f, unit, leaf, r, sf.ReduceOp.sum, stream)
        sf.reduce_end(h)

    def step():
        step_on(root)

    with torch.cuda.stream(stream):
        for _ in range(max(3, args.warmup)):
            step()
    torch.cuda.synchronize()
    barrier()

    sampler = None
    if rank == 0:
        uuid = str(torch.cuda.get_device_properties(dev).uuid)
        sampler = ClockSampler(uuid if uuid.startswith("GPU-") else f"GPU-{uuid}")
        sampler.start()
        sampler.wait_first()
    timed_step = step
    graph_launches = None
    if args.graph:
        graph = torch.cuda.CUDAGraph()
        g0 = sf.counters()["kernel_launches"]
        with torch.cuda.graph(graph, stream=stream):
            step()
        graph_launches = sf.counters()["kernel_launches"] - g0  # kernel nodes per replayed step
        with torch.cuda.stream(stream):
            for _ in range(3):
                graph.replay()
        torch.cuda.synchronize()
        barrier()
        timed_step = graph.replay

    # Timed region: K steps, no per-launch instrumentation inside it.
    c0 = sf.counters()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    t_start = time.perf_counter()
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for _ in range(args.steps):
            timed_step()
        ev1.record(stream)
    torch.cuda.synchronize()
    t_end = time.perf_counter()
    barrier()
    clocks = sampler.stop((t_start, t_end)) if sampler else None
    c1 = sf.counters()
    # Per-launch CUDA events (kernel durations, bytes, NVLink bytes for the
    # roofline) over a second pass of the same steps.
    sf.timing_enable(True)
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            step()
    torch.cuda.synchronize()
    sf.timing_enable(False)
    timing = sf.timing_collect()
    barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_max = allreduce(ms, "max")
    launches = sum(v["launches"] for v in timing.values())
    bytes_step = sum(v["bytes"] for v in timing.values()) / args.steps
    bytes_all = allreduce(bytes_step, "sum")
    value = bytes_all / (ms_max * 1e-3) / 1e9
    kl = allreduce(float(c1["kernel_launches"] - c0["kernel_launches"] if graph_launches is None
                         else graph_launches * args.steps), "sum")
    net_bytes = allreduce(float(c1["bytes_sent"] - c0["bytes_sent"]) / args.steps, "sum")

    # roofline of the dominant kernel (largest device time in the region)
    peak, peak_kind = peaks()
    dom_tag, dom = max(((k, v) for k, v in timing.items() if v["bytes"] > 0),
                       key=lambda kv: kv[1]["total_ms"])
    per_launch_bytes = dom["bytes"] / dom["launches"]
    per_launch_ms = dom["total_ms"] / dom["launches"]
    achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"P{world}", {}).get(dom_tag)
        except Exception:
            traffic = None
    share = dom["total_ms"] / max(1e-9, ev0.elapsed_time(ev1))

    # remote exchange over NVLink. Inside the step the exchange launch (p2p:
    # puts + receives; nccl: the grouped send/recv) runs on the comm stream
    # while the interior copy, the step's dominant kernel, holds the SMs and
    # HBM: its duration there is how long it stays hidden under that copy, not
    # a link rate. The link figures (achieved / frac) come from the halo-only
    # exchange timed on its own (halo_exchange).
    link_recs = [v for v in timing.values() if v.get("link_bytes", 0) > 0]
    nvlink = None
    if world > 1:
        lb = sum(v["link_bytes"] for v in link_recs)
        lms = sum(v["total_ms"] for v in link_recs)
        lus = allreduce(1e3 * lms / max(1, sum(v["launches"] for v in link_recs)), "max")
        nvlink = {"in_step_exchange_launch_us": lus,
                  "in_step_note": "exchange launch duration inside the step, sharing the GPU with the interior copy",
                  "bytes_per_exchange": lb / max(1, sum(v["launches"] for v in link_recs))}
        nvlink.update(halo_exchange(args, sf, comm, graphs, torch, rank, world, allreduce, barrier))

    # end-to-end through the public API: every step copies its root vector in
    # from pinned host memory, runs Bcast+Reduce and copies the result back.
    # Three device root buffers pipeline the steps: step k's H2D (copy
    # stream), step k-1's SF work (SF stream) and step k-1's D2H (copy stream)
    # overlap, each buffer reused only after its previous D2H finished. (With
    # two buffers H2D(k) waits for D2H(k-2), which itself started one SF step
    # after H2D(k-2): the SF time adds to every period.)
    e2e = None
    if not args.no_e2e:
        host_in = root.cpu().pin_memory()
        host_out = torch.empty_like(host_in).pin_memory()
        NB = 3
        bufs = [root] + [torch.empty_like(root) for _ in range(NB - 1)]
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        h2d = [torch.cuda.Event() for _ in range(NB)]
        done = [torch.cuda.Event() for _ in range(NB)]
        d2h = [torch.cuda.Event() for _ in range(NB)]

        def run_e2e(k_steps, e0=None, e1=None):
            for b in range(NB):
                d2h[b].record(s_out)
            if e0 is not None:
                e0.record(s_in)
            for k in range(k_steps):
                b = k % NB
                s_in.wait_event(d2h[b])
                with torch.cuda.stream(s_in):
                    bufs[b].copy_(host_in, non_blocking=True)
                h2d[b].record(s_in)
                stream.wait_event(h2d[b])
                with torch.cuda.stream(stream):
                    step_on(bufs[b])
                done[b].record(stream)
                s_out.wait_event(done[b])
                with torch.cuda.stream(s_out):
                    host_out.copy_(bufs[b], non_blocking=True)
                d2h[b].record(s_out)
            if e1 is not None:
                s_out.wait_event(h2d[(k_steps - 1) % NB])
                e1.record(s_out)

        run_e2e(NB)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        run_e2e(args.e2e_steps, e0, e1)
        torch.cuda.synchronize()
        barrier()
        ems = allreduce(e0.elapsed_time(e1) / args.e2e_steps, "max")
        hb = allreduce(float(geo.n_owned * 8), "sum")
        e2e = {"value": bytes_all / (ems * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ems,
               "h2d_bytes_per_step": int(hb), "d2h_bytes_per_step": int(hb),
               "pipelined": "3 root buffers: H2D, SF work and D2H of consecutive steps overlap"}
        # every step starts from host_in: Reduce SUM folds each root with its
        # interior copy and one copy per neighbour ghosting it (any N)
        want = graphs.g2l_reduce_expect(geo, host_in.cuda()).cpu()
        ok = float(torch.equal(host_out, want))
        e2e["result_ok"] = bool(allreduce(ok, "sum") == world)
        del want

    # Result check at full size on every rank, any N (after the timed work):
    # roots = their local ids, one Bcast REPLACE + Reduce SUM, closed form.
    ids = torch.arange(geo.n_owned, dtype=torch.float64, device="cuda")
    leaf.fill_(-1.0)
    torch.cuda.synchronize()  # ids / leaf were written on the default stream
    barrier()
    with torch.cuda.stream(stream):
        step_on(ids)
    torch.cuda.synchronize()
    chk = graphs.g2l_check(geo, leaf, ids)
    del ids
    nbad = allreduce(0.0 if (chk["leaf_ok"] and chk["root_ok"]) else 1.0, "sum")
    nleaf = allreduce(0.0 if chk["leaf_ok"] else 1.0, "sum")
    check = {"result_ok": nbad == 0, "ranks_failed": int(nbad), "ranks_leaf_failed": int(nleaf),
             "what": "roots = local ids; Bcast REPLACE + Reduce SUM; every leaf of the ghosted box "
                     "and every root equal their closed form (id, neighbour's id, id*(2+ghost copies))"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args)
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "error": str(e)}

    if rank == 0:
        px, py, pz = args.dims or graphs.proc_grid(world)
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": "g2l_halo_7pt (BASELINE config 2: DMDA global->local SF, "
                                   "Bcast REPLACE + Reduce SUM)",
                       "grid": [args.N] * 3, "decomposition": [px, py, pz],
                       "parallelism": f"sf{world}", "us_per_op": ms_max * 1e3 / 2,
                       "launch": "CUDA graph replay per step" if args.graph else "eager API calls per step",
                       "bytes_per_step": bytes_all, "nvlink_bytes_per_step": net_bytes,
                       "l2": "inputs > L2: 1.07 GB roots + 1.09 GB leaves per rank at N=1",
                       "setup_s": setup_s, "set_graph_s": set_graph_s, "device_setup": dsetup,
                       "graph_gen_s": gen_s, "deterministic": True,
                       "transport": args.transport if world > 1 else "none (self edges only)"},
            "gpu_launches": int(kl),
            "roofline": {"bound": "hbm", "kernel": dom_tag, "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "bytes_per_launch": per_launch_bytes,
                         "us_per_launch": per_launch_ms * 1e3, "share_of_step": share},
            "kernels": {k: {"launches": v["launches"], "us_per_launch": 1e3 * v["total_ms"] / v["launches"],
                            "GBps": v["bytes"] / (v["total_ms"] * 1e-3) / 1e9 if v["total_ms"] else None}
                        for k, v in timing.items()},
            "nvlink": nvlink,
            "check": check,
            "result_ok": check["result_ok"],
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    ours(args, rank, world, local)


if __name__ == "__main__":
    main()
