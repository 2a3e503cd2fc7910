"""Device SetUp (csrc/dsetup.cu) against the host planner.

The host planner is pinned to the reference (test_cpu_planner.py: golden
two-sided info, the reference's random forests); here a forest set from device
arrays must produce the identical plan — group ranks, items in order, pattern
kind and parameters — the same validation messages (starforest.cpp:29-76,
116-123), and operations over it must match the oracle bit for bit.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2102_13018_b200 import graphs, sf
from tests.helpers import assert_same, rank_data, run_gpu, set_graph_device

pytestmark = pytest.mark.gpu


def plan(f):
    ti = f.two_sided()
    return (f.nroots(), f.nleaves(), f.leaf_index_bound(), f.contiguous_leaves(), ti.self_first,
            ti.root_ranks, ti.leaf_ranks, [g.pattern for g in f.root_groups()],
            [g.pattern for g in f.leaf_groups()])


def both_plans(specs, extra=None):
    """Per rank: (host plan, device plan[, extra(host forest, device forest)])."""
    def body(c):
        h = sf.StarForest(c)
        h.set_graph_spec(specs[c.rank()])
        h.setup()
        d = sf.StarForest(c)
        set_graph_device(d, specs[c.rank()])
        d.setup()
        out = [plan(h), plan(d)]
        if extra:
            out.append(extra(h, d))
        return out

    return sf.run_ranks(sf.CommConfig(nranks=len(specs)), body,
                        devices=[0] * len(specs))


def shuffled(specs, seed):
    """Same forests with the leaves listed in a random (non-increasing) order."""
    rng = np.random.default_rng(seed)
    out = []
    for s in specs:
        idx = s.local if s.local is not None else np.arange(s.nleaves, dtype=np.int64)
        p = rng.permutation(s.nleaves)
        out.append(sf.GraphSpec(s.nroots, s.nleaves, np.asarray(idx, np.int64)[p],
                                np.asarray(s.remote_rank, np.int32)[p], np.asarray(s.remote_off, np.int64)[p]))
    return out


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_device_plan_equals_host_plan_random(seed, P):
    specs = graphs.random_graph_specs(700 + seed, P, 40)
    for r in both_plans(specs):
        assert r[0] == r[1]
    for r in both_plans(shuffled(specs, seed)):
        assert r[0] == r[1]


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_device_plan_g2l_structured(P):
    specs = [graphs.g2l_halo(12, P, r) for r in range(P)]
    for r in both_plans(specs):
        assert r[0] == r[1]
        assert all(p.kind in ("contiguous", "affine") for p in r[1][7] + r[1][8])


def test_device_plan_indexed_with_duplicates_and_large_span():
    # dense duplicates (bitmap distinct count) and a sparse span (sorted uniques)
    dense = sf.GraphSpec(50, 400, None, np.zeros(400, np.int32),
                         (np.arange(400, dtype=np.int64) * 7919) % 50)
    rng = np.random.default_rng(3)
    sparse = sf.GraphSpec(1 << 40, 300, None, np.zeros(300, np.int32),
                          rng.integers(0, 1 << 40, 300, dtype=np.int64))
    sparse.remote_off[5] = sparse.remote_off[77]
    for spec in (dense, sparse):
        r = both_plans([spec])[0]
        assert r[0] == r[1]
        assert r[1][8][0].has_duplicates


def test_degrees_multi_sf_graph_spec_from_device_forest():
    specs = graphs.random_graph_specs(77, 3, 30)

    def extra(h, d):
        return (h.compute_degrees().tolist() == d.compute_degrees().tolist(),
                h.multi_sf().two_sided() == d.multi_sf().two_sided(),
                h.graph_spec().remote_off.tolist() == d.graph_spec().remote_off.tolist())

    for r in both_plans(specs, extra):
        assert r[2] == (True, True, True)


def test_device_set_graph_messages():
    import torch

    def body(c):
        f = sf.StarForest(c)
        t = lambda a, dt: torch.tensor(a, dtype=dt, device="cuda")  # noqa: E731
        i32, i64 = torch.int32, torch.int64
        with pytest.raises(sf.Error, match="duplicate leaf index 3 violates the forest property"):
            f.set_graph_device(9, 3, t([3, 1, 3], i64), t([0, 0, 0], i32), t([0, 0, 0], i64))
        with pytest.raises(sf.Error, match="negative leaf index"):
            f.set_graph_device(9, 2, t([-1, 4], i64), t([0, 0], i32), t([0, 0], i64))
        with pytest.raises(sf.Error, match="negative leaf index"):
            f.set_graph_device(9, 2, t([4, -1], i64), t([0, 0], i32), t([0, 0], i64))
        with pytest.raises(sf.Error, match="root rank 5 outside communicator"):
            f.set_graph_device(9, 2, None, t([0, 5], i32), t([0, 0], i64))
        with pytest.raises(sf.Error, match="negative root offset"):
            f.set_graph_device(9, 2, None, t([0, 0], i32), t([0, -2], i64))
        with pytest.raises(sf.Error, match="length does not match"):
            f.set_graph_device(9, 3, None, t([0, 0], i32), t([0, 0], i64))
        f.set_graph_device(4, 2, None, t([0, 0], i32), t([1, 9], i64))
        with pytest.raises(sf.Error, match="references root offset 9 but this rank has only 4 roots"):
            f.setup()
        return True

    assert sf.run_ranks(sf.CommConfig(nranks=1), body, devices=[0]) == [True]


@pytest.mark.parametrize("seed", range(4))
def test_ops_over_device_forest_match_oracle(seed):
    P = 3
    specs = shuffled(graphs.random_graph_specs(900 + seed, P, 60), seed)
    cfg = lambda: sf.CommConfig(nranks=P)  # noqa: E731
    roots = rank_data(specs, seed, np.float64, which="root")
    leaves = rank_data(specs, seed, np.float64, salt0=200, which="leaf")
    out = run_gpu(specs, "bcast", [roots, leaves], config=cfg(), devices=[0] * P, device_graph=True)
    assert_same(out[1], O.bcast(specs, roots, leaves))
    out = run_gpu(specs, "reduce", [leaves, roots], op="sum", config=cfg(), devices=[0] * P,
                  device_graph=True)
    assert_same(out[1], O.reduce(specs, leaves, roots, "sum"))
    ri = rank_data(specs, seed, np.int64, which="root")
    li = rank_data(specs, seed, np.int64, salt0=300, which="leaf")
    ui = [np.zeros_like(x) for x in li]
    out = run_gpu(specs, "fetch_and_op", [ri, li, ui], op="sum", config=cfg(), devices=[0] * P,
                  device_graph=True)
    want = O.fetch_and_op(specs, ri, li, ui, "sum")
    assert_same(out[0], want[0])
    assert_same(out[2], want[1])


def test_config2_g2l_512_device_setup():
    """The 134M-leaf G2L forest planned on the device: the same plan as the
    host planner, and Bcast REPLACE of root ids lands every owned point."""
    import time

    import torch

    N = 512
    spec = graphs.g2l_halo(N, 1, 0)
    g = graphs.G2L(N, 1, 0)

    def body(c):
        h = sf.StarForest(c)
        h.set_graph_spec(spec)
        t = time.perf_counter()
        h.setup()
        t_host = time.perf_counter() - t
        d = sf.StarForest(c)
        loc = torch.from_numpy(spec.local).cuda()
        rr = torch.from_numpy(spec.remote_rank).cuda()
        ro = torch.from_numpy(spec.remote_off).cuda()
        torch.cuda.synchronize()
        t = time.perf_counter()
        d.set_graph_device(spec.nroots, spec.nleaves, loc, rr, ro)
        d.setup()
        t_dev = time.perf_counter() - t
        same = [g.pattern for g in h.root_groups()] == [g.pattern for g in d.root_groups()] and \
            [g.pattern for g in h.leaf_groups()] == [g.pattern for g in d.leaf_groups()]
        del h
        root = torch.arange(g.n_owned, dtype=torch.float64, device="cuda")
        leaf = torch.full((g.n_local,), -1.0, dtype=torch.float64, device="cuda")
        sf.bcast(d, sf.Unit(sf.Kind.float64), root, leaf, sf.ReduceOp.replace)
        ok = bool(torch.equal(leaf.view(g.Z, g.Y, g.X)[1:-1, 1:-1, 1:-1].reshape(-1), root))
        print(f"G2L 512^3 setup: host {t_host * 1e3:.1f} ms, device {t_dev * 1e3:.1f} ms")
        return same, ok

    assert sf.run_ranks(sf.CommConfig(nranks=1), body, devices=[0])[0] == (True, True)


def test_gather_scatter_over_device_forest():
    """Gather / Scatter go through the multi-SF, which a device-set forest
    builds from host copies made on demand (host_graph)."""
    P = 3
    specs = shuffled(graphs.random_graph_specs(31, P, 50), 5)
    leaves = rank_data(specs, 7, np.float64, salt0=200, which="leaf")
    deg = O.degrees(specs)
    multi = [np.zeros(int(d.sum()), np.float64) for d in deg]
    out = run_gpu(specs, "gather", [leaves, multi], config=sf.CommConfig(nranks=P), devices=[0] * P,
                  device_graph=True)
    want = O.gather(specs, leaves)
    assert_same(out[1], want)
    back = [np.full_like(x, -1.0) for x in leaves]
    out = run_gpu(specs, "scatter", [want, back], config=sf.CommConfig(nranks=P), devices=[0] * P,
                  device_graph=True)
    assert_same(out[1], O.scatter(specs, want, back))
