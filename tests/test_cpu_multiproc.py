"""World-size-2 multi-process tests on CPU (gloo): the N>1 host path — SetUp
discovery and multi-SF slot exchange across processes through the
torch.distributed control plane — and bench.py's rank decomposition /
max-over-ranks plumbing."""
import os
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = textwrap.dedent("""
    import os, sys, json
    sys.path.insert(0, %(root)r)
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2102_13018_b200 import graphs, sf
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    out = {}
    # 1) G2L decomposition of bench.py: every RootRef lands on a real root.
    spec = graphs.g2l_halo(12, world, rank)
    allspecs = [None] * world
    dist.all_gather_object(allspecs, (spec.nroots, spec.remote_rank.tolist(), spec.remote_off.tolist()))
    for (nr, rr, ro) in allspecs:
        for r, o in zip(rr, ro):
            assert 0 <= o < allspecs[r][0]
    # 2) SetUp across processes over the torch.distributed control plane.
    comm = sf.Comm.from_torch_distributed(device=-1)
    f = sf.StarForest(comm)
    f.set_graph_spec(spec)
    f.setup()
    ti = f.two_sided()
    out["g2l"] = [ti.root_ranks, ti.leaf_ranks, f.compute_degrees().tolist(), f.multi_sf().nroots(),
                  [g.pattern.kind for g in f.root_groups()]]
    specs = graphs.random_graph_specs(11, world, 30)
    g = sf.StarForest(comm)
    g.set_graph_spec(specs[rank])
    g.setup()
    ti = g.two_sided()
    out["rand"] = [ti.root_ranks, ti.leaf_ranks, g.compute_degrees().tolist(), g.multi_sf().nroots()]
    # 3) bench-style max over ranks
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out["max"] = float(t.item())
    allout = [None] * world
    dist.all_gather_object(allout, out)
    if rank == 0:
        print("RESULT" + json.dumps(allout))
    dist.destroy_process_group()
""")


def _threads_reference(specs):
    from paper_2102_13018_b200 import sf

    def body(c):
        f = sf.StarForest(c)
        f.set_graph_spec(specs[c.rank()])
        f.setup()
        ti = f.two_sided()
        return [ti.root_ranks, ti.leaf_ranks, f.compute_degrees().tolist(), f.multi_sf().nroots()]
    return sf.run_ranks(sf.CommConfig(nranks=len(specs)), body, devices=[-1] * len(specs))


def test_two_process_gloo_setup_matches_in_process(tmp_path):
    import json

    from paper_2102_13018_b200 import graphs

    w = tmp_path / "worker.py"
    w.write_text(WORKER % {"root": ROOT})
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr", "127.0.0.1", "--master-port",
                        "29561", str(w)], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT")][0]
    got = json.loads(line[len("RESULT"):])
    want_g2l = _threads_reference([graphs.g2l_halo(12, 2, q) for q in range(2)])
    want_rand = _threads_reference(graphs.random_graph_specs(11, 2, 30))
    for q in range(2):
        def norm(x):
            return json.loads(json.dumps(x))
        assert norm(got[q]["g2l"][:4]) == norm(want_g2l[q])
        assert norm(got[q]["rand"]) == norm(want_rand[q])
        assert set(got[q]["g2l"][4]) <= {"contiguous", "affine"}
        assert got[q]["max"] == 2.0


def test_control_plane_allgather_threads():
    """sfg_comm_allgather over the in-process control plane (host-only ranks)."""
    from paper_2102_13018_b200 import sf

    def body(c):
        return c.allgather_int64([c.rank() * 10, c.rank() + 1]).tolist()

    got = sf.run_ranks(sf.CommConfig(nranks=3), body, devices=[-1] * 3)
    assert all(g == [[0, 1], [10, 2], [20, 3]] for g in got)
