"""One-process-per-GPU parity worker (launched by tests/test_gpu_multi.py via
torch.distributed.run). Control plane and data plane both over NCCL, as in
bench.py at N>1. Rank 0 compares every rank's results with the oracle and
exits non-zero on any mismatch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2102_13018_b200 import graphs, sf  # noqa: E402
from tests.helpers import assert_same, rank_data, set_graph_device  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    fails = []
    backend = sys.argv[1] if len(sys.argv) > 1 else "nccl"
    for deterministic in (True, False):
        obj = [sf.nccl_unique_id() if rank == 0 else None]  # one id per communicator
        dist.broadcast_object_list(obj, src=0)
        comm = sf.Comm(world, rank, local, sf.CommConfig(nranks=world, backend=backend,
                                                         deterministic=deterministic), nccl_id=obj[0])
        cases = [("g2l", [graphs.g2l_halo(9, world, r) for r in range(world)])]
        for seed in range(4):
            cases.append((f"rand{seed}", graphs.random_graph_specs(seed + 77, world, 40)))
        cases.append(("cfg4", graphs.random_leaf_root(1 << 14, 1 << 7, world, seed=9)))
        for name, specs in cases:
            f = sf.StarForest(comm)
            f.set_graph_spec(specs[rank])
            f.setup()
            dt = np.float64
            roots = rank_data(specs, 3, dt, 1, 100, "root")
            leaves = rank_data(specs, 3, dt, 1, 200, "leaf")
            iroots = rank_data(specs, 3, np.int64, 1, 300, "root", 1, 1000)
            ileaves = rank_data(specs, 3, np.int64, 1, 400, "leaf", 1, 1000)
            u = sf.Unit(sf.Kind.float64)
            ui = sf.Unit(sf.Kind.int64)
            dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
            lb = dev(leaves[rank])
            sf.bcast(f, u, dev(roots[rank]), lb, sf.ReduceOp.replace)
            rb = dev(roots[rank])
            sf.reduce(f, u, dev(leaves[rank]), rb, sf.ReduceOp.sum)
            ri = dev(iroots[rank])
            li = dev(ileaves[rank])
            upd = torch.zeros_like(li)
            sf.fetch_and_op(f, ui, ri, li, upd, sf.ReduceOp.sum)
            deg = f.compute_degrees()
            multi = torch.zeros(int(deg.sum()), dtype=torch.float64, device="cuda")
            sf.gather(f, u, dev(leaves[rank]), multi)
            mine = [lb.cpu().numpy(), rb.cpu().numpy(), ri.cpu().numpy(), upd.cpu().numpy(),
                    multi.cpu().numpy()]
            allr = [None] * world
            dist.all_gather_object(allr, mine)
            if rank == 0:
                try:
                    assert_same([a[0] for a in allr], O.bcast(specs, roots, leaves), what=f"{name} bcast")
                    assert_same([a[1] for a in allr], O.reduce(specs, leaves, roots, "sum"),
                                fp_tol=not deterministic, what=f"{name} reduce")
                    orr, ou = O.fetch_and_op(specs, iroots, ileaves, [np.zeros_like(x) for x in ileaves], "sum")
                    assert_same([a[2] for a in allr], orr, what=f"{name} fetch root")
                    if deterministic:
                        assert_same([a[3] for a in allr], ou, what=f"{name} fetch update")
                    assert_same([a[4] for a in allr], O.gather(specs, leaves), what=f"{name} gather")
                except AssertionError as e:
                    fails.append(f"det={deterministic} {e}")
            if name.startswith("rand") and deterministic:
                # CUDA-graph capture of Bcast(REPLACE) + Reduce(SUM): replayed with new
                # root values it must give what eager calls give (the p2p protocol's
                # message counters live on the device).
                st = torch.cuda.Stream()
                r0 = dev(roots[rank])
                lg = dev(leaves[rank])
                racc = dev(roots[rank])
                with torch.cuda.stream(st):
                    for _ in range(2):
                        sf.bcast_end(sf.bcast_begin(f, u, r0, lg, sf.ReduceOp.replace, st))
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    sf.bcast_end(sf.bcast_begin(f, u, r0, lg, sf.ReduceOp.replace, st))
                    sf.reduce_end(sf.reduce_begin(f, u, lg, racc, sf.ReduceOp.sum, st))
                for it in range(3):
                    r0.copy_(dev(roots[rank] * (it + 2)))
                    racc.copy_(dev(roots[rank]))
                    g.replay()
                    torch.cuda.synchronize()
                    got = [lg.cpu().numpy(), racc.cpu().numpy()]
                    allg = [None] * world
                    dist.all_gather_object(allg, got)
                    if rank == 0:
                        try:
                            scaled = [x * (it + 2) for x in roots]
                            wl = O.bcast(specs, scaled, leaves)
                            assert_same([a[0] for a in allg], wl, what=f"{name} graph bcast {it}")
                            assert_same([a[1] for a in allg], O.reduce(specs, wl, roots, "sum"),
                                        what=f"{name} graph reduce {it}")
                        except AssertionError as e:
                            fails.append(f"graph {e}")
                del g
                # FetchAndOp SUM in a graph: every replay serialises the same
                # contributions again on top of the previous roots.
                ri0 = dev(iroots[rank])
                li0 = dev(ileaves[rank])
                up = torch.zeros_like(li0)
                with torch.cuda.stream(st):
                    sf.fetch_and_op_end(sf.fetch_and_op_begin(f, ui, ri0, li0, up, sf.ReduceOp.sum, st))
                torch.cuda.synchronize()
                ri0.copy_(dev(iroots[rank]))
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    sf.fetch_and_op_end(sf.fetch_and_op_begin(f, ui, ri0, li0, up, sf.ReduceOp.sum, st))
                cur = [x.copy() for x in iroots]
                for it in range(2):
                    g.replay()
                    torch.cuda.synchronize()
                    got = [ri0.cpu().numpy(), up.cpu().numpy()]
                    allg = [None] * world
                    dist.all_gather_object(allg, got)
                    if rank == 0:
                        try:
                            orr, ou = O.fetch_and_op(specs, cur, ileaves, [np.zeros_like(x) for x in ileaves], "sum")
                            assert_same([a[0] for a in allg], orr, what=f"{name} graph fetch root {it}")
                            assert_same([a[1] for a in allg], ou, what=f"{name} graph fetch update {it}")
                        except AssertionError as e:
                            fails.append(f"graph {e}")
                    cur = orr if rank == 0 else cur
                    obj = [cur]
                    dist.broadcast_object_list(obj, src=0)
                    cur = obj[0]
                del g
            if deterministic:
                # Device SetUp (dsetup.cu) across processes: the same plan as
                # the host planner, and the same Bcast / Reduce results.
                fd = sf.StarForest(comm)
                set_graph_device(fd, specs[rank])
                fd.setup()
                same = (fd.two_sided() == f.two_sided()
                        and [g.pattern for g in fd.root_groups()] == [g.pattern for g in f.root_groups()]
                        and [g.pattern for g in fd.leaf_groups()] == [g.pattern for g in f.leaf_groups()])
                lb2 = dev(leaves[rank])
                sf.bcast(fd, u, dev(roots[rank]), lb2, sf.ReduceOp.replace)
                rb2 = dev(roots[rank])
                sf.reduce(fd, u, dev(leaves[rank]), rb2, sf.ReduceOp.sum)
                same = same and torch.equal(lb2, lb) and torch.equal(rb2.view(torch.int64), rb.view(torch.int64))
                flags = [None] * world
                dist.all_gather_object(flags, same)
                if rank == 0 and not all(flags):
                    fails.append(f"{name} device setup differs on ranks {[i for i, x in enumerate(flags) if not x]}")
                del fd
            del f
        comm.close()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        if fails:
            print("FAIL", *fails, sep="\n")
            sys.exit(1)
        print(f"mp_worker ok world={world} backend={backend}")


if __name__ == "__main__":
    main()
