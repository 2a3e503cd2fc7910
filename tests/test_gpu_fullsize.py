"""Parity at the BASELINE configurations' full sizes, one GPU.

Config 1 (4,194,304 leaves -> 1,048,576 roots) and config 4 (16,777,216
leaves -> 65,536 roots) are checked bit-exactly against the C oracle (it
finishes them in seconds); config 2 (the 512^3 G2L forest, 134M leaves) through
size-independent properties of the ghosted-box map: Bcast REPLACE of root ids
puts every owned point's id at its ghosted-box position (and leaves the ghost
frame untouched), Reduce SUM of those leaves doubles every root, Bcast+Reduce
REPLACE is the identity. Config 4 FetchAndOp SUM of ones is checked by its
serialization property (selfcheck.cpp:631-672): each root's fetched values are
init, init+1, ... in ascending leaf order.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2102_13018_b200 import graphs, sf
from tests.helpers import assert_same, run_gpu

pytestmark = pytest.mark.gpu


def test_config1_full_size_vs_oracle():
    L, R = 4194304, 1048576
    specs = graphs.random_leaf_root(L, R, 1, seed=1)
    roots = [graphs.gen_f64(1, 100, R)]
    leaves = [graphs.gen_f64(1, 200, L)]
    out = run_gpu(specs, "bcast", [roots, leaves])
    assert_same(out[1], O.bcast(specs, roots, leaves))
    for det in (True, False):
        out = run_gpu(specs, "reduce", [leaves, roots], op="sum",
                      config=sf.CommConfig(deterministic=det))
        assert_same(out[1], O.reduce(specs, leaves, roots, "sum"))


def test_config4_full_size_reduce_and_fetch():
    L, R = 16777216, 65536
    specs = graphs.random_leaf_root(L, R, 1, seed=4)
    roots = [graphs.gen_f64(4, 100, R)]
    leaves = [graphs.gen_f64(4, 200, L)]
    out = run_gpu(specs, "reduce", [leaves, roots], op="sum")
    assert_same(out[1], O.reduce(specs, leaves, roots, "sum"))  # bit-exact, L2-tiled CSR
    # FetchAndOp SUM of ones on int64: serialization in ascending leaf order
    init = (np.arange(R, dtype=np.int64) * 7) % 1000
    ones = np.ones(L, np.int64)
    upd = np.zeros(L, np.int64)
    r, _, u = run_gpu(specs, "fetch_and_op", [[init], [ones], [upd]], op="sum")
    root_of = specs[0].remote_off
    deg = np.bincount(root_of, minlength=R)
    assert np.array_equal(r[0], init + deg)
    order = np.argsort(root_of, kind="stable")  # per root, ascending leaf
    starts = np.concatenate([[0], np.cumsum(deg)[:-1]])
    rank_in_root = np.empty(L, np.int64)
    rank_in_root[order] = np.arange(L) - np.repeat(starts, deg)
    assert np.array_equal(u[0], init[root_of] + rank_in_root)


def test_config2_g2l_512_properties():
    import torch

    N = 512
    spec = graphs.g2l_halo(N, 1, 0)
    g = graphs.G2L(N, 1, 0)
    unit = sf.Unit(sf.Kind.float64)

    def body(comm):
        f = sf.StarForest(comm)
        f.set_graph_spec(spec)
        f.setup()
        root = torch.arange(g.n_owned, dtype=torch.float64, device="cuda")
        leaf = torch.full((g.n_local,), -1.0, dtype=torch.float64, device="cuda")
        sf.bcast(f, unit, root, leaf, sf.ReduceOp.replace)
        box = leaf.view(g.Z, g.Y, g.X)
        ok_interior = bool(torch.equal(box[1:-1, 1:-1, 1:-1].reshape(-1), root))
        frame = box.clone()
        frame[1:-1, 1:-1, 1:-1] = -1.0
        ok_frame = bool((frame == -1.0).all())
        sf.reduce(f, unit, leaf, root, sf.ReduceOp.sum)
        ok_double = bool(torch.equal(root, 2.0 * torch.arange(g.n_owned, dtype=torch.float64,
                                                              device="cuda")))
        before = root.clone()
        sf.bcast(f, unit, root, leaf, sf.ReduceOp.replace)
        sf.reduce(f, unit, leaf, root, sf.ReduceOp.replace)
        ok_identity = bool(torch.equal(root, before))
        return ok_interior, ok_frame, ok_double, ok_identity

    got = sf.run_ranks(sf.CommConfig(nranks=1), body, devices=[0])[0]
    assert got == (True, True, True, True)
