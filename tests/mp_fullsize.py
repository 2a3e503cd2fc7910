"""Full-size config 2 parity at N>1 (launched by tests/test_gpu_multi.py via
torch.distributed.run, one process per GPU): the 512^3 G2L forest over the
run's ranks, Bcast REPLACE of root ids + Reduce SUM through the public API,
checked on every rank by the closed form of graphs.g2l_check (the reference's
distributed path, /root/reference/proj/src/ops.cpp:276-376, computes exactly
these values). argv: backend [N] [px,py,pz]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2102_13018_b200 import graphs, sf  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    backend = sys.argv[1]
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    dims = tuple(int(v) for v in sys.argv[3].split(",")) if len(sys.argv) > 3 else None
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [sf.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = sf.Comm(world, rank, local, sf.CommConfig(nranks=world, backend=backend), nccl_id=obj[0])
    geo = graphs.G2L(N, world, rank, dims=dims)
    f = sf.StarForest(comm)
    f.set_graph_spec(graphs.g2l_halo(N, world, rank, dims=dims))
    f.setup()
    u = sf.Unit(sf.Kind.float64)
    ids = torch.arange(geo.n_owned, dtype=torch.float64, device="cuda")
    leaf = torch.full((geo.n_local,), -1.0, dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    torch.cuda.synchronize()  # ids / leaf were written on the default stream
    dist.barrier()
    with torch.cuda.stream(st):
        sf.bcast_end(sf.bcast_begin(f, u, ids, leaf, sf.ReduceOp.replace, st))
        sf.reduce_end(sf.reduce_begin(f, u, leaf, ids, sf.ReduceOp.sum, st))
    st.synchronize()
    chk = graphs.g2l_check(geo, leaf, ids)
    # The same with arbitrary (non-integer) values: the sequential fold of the
    # root with its copies, rounded per addition.
    r0 = torch.rand(geo.n_owned, dtype=torch.float64, device="cuda")
    r = r0.clone()
    torch.cuda.synchronize()
    dist.barrier()
    with torch.cuda.stream(st):
        sf.bcast_end(sf.bcast_begin(f, u, r, leaf, sf.ReduceOp.replace, st))
        sf.reduce_end(sf.reduce_begin(f, u, leaf, r, sf.ReduceOp.sum, st))
    st.synchronize()
    chk["fold_ok"] = bool(torch.equal(r, graphs.g2l_reduce_expect(geo, r0)))
    allc = [None] * world
    dist.all_gather_object(allc, chk)
    del f
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        bad = [(i, c) for i, c in enumerate(allc) if not all(c.values())]
        if bad:
            print("FAIL", bad)
            sys.exit(1)
        print(f"mp_fullsize ok world={world} backend={backend} N={N} dims={geo.px},{geo.py},{geo.pz}")


if __name__ == "__main__":
    main()
