"""Halo-only Bcast (config 2 ghost faces of 512^3, 2 ranks) with the two
ranks as THREADS of one process (peer pointers) instead of processes (CUDA
IPC): same graph-replay steady-state timing as bench_configs.py config 2.
Usage: python scripts/halo_threads.py [N]"""
import os
import statistics
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2102_13018_b200 import graphs, sf  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
P = 2
K = 50
bar = threading.Barrier(P)


def body(comm):
    r = comm.rank()
    spec = graphs.g2l_halo(N, P, r, interior=False)
    geo = graphs.G2L(N, P, r)
    f = sf.StarForest(comm)
    f.set_graph_spec(spec)
    f.setup()
    u = sf.Unit(sf.Kind.float64)
    root = torch.rand(geo.n_owned, dtype=torch.float64, device="cuda")
    leaf = torch.zeros(geo.n_local, dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        for _ in range(3):
            sf.bcast_end(sf.bcast_begin(f, u, root, leaf, sf.ReduceOp.replace, st))
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st, capture_error_mode="thread_local"):
        for _ in range(K):
            sf.bcast_end(sf.bcast_begin(f, u, root, leaf, sf.ReduceOp.replace, st))
    torch.cuda.synchronize()
    per = []
    for _ in range(5):
        bar.wait()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            g.replay()
            e0.record(st)
            g.replay()
            e1.record(st)
        st.synchronize()
        per.append(e0.elapsed_time(e1) * 1e3 / K)
    del g, f
    return statistics.median(per)


got = sf.run_ranks(sf.CommConfig(nranks=P, backend="p2p"), body, devices=[0, 1])
us = max(got)
print(f'{{"what": "halo-only Bcast, 2 thread ranks", "us_per_op": {us:.2f}, '
      f'"egress_GBps": {2 * N * N * 8 / (us * 1e-6) / 1e9:.1f}, "per_rank": {got}}}')
