"""GPU parity tests: every operation through the C ABI against the oracle and
the reference's golden vectors. Mirrors /root/reference/proj/tests/test_sfops.cpp
and the selfcheck suites (src/selfcheck.cpp:85-163, 386-418, 574-679)."""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2102_13018_b200 import graphs, sf
from tests.helpers import assert_same, rank_data, run_gpu, to_dev, to_host

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig2.json")))
FIG = sf.graph_text_parse(GOLD["graph_text"])
I64 = sf.Unit(sf.Kind.int64)


def fig_arrays(key):
    return [np.array(x, np.int64) for x in GOLD[key]]


# ------------------------------------------------------------- Fig. 2 golden
def test_fig2_bcast_replace():
    out = run_gpu(FIG, "bcast", [fig_arrays("roots"), fig_arrays("leaves")])
    assert_same(out[1], fig_arrays("bcast_replace_leaves"))


def test_fig2_bcast_sum():
    leaves = [np.zeros(len(x), np.int64) for x in GOLD["leaves"]]
    leaves[2][0] = 100
    out = run_gpu(FIG, "bcast", [fig_arrays("roots"), leaves], op="sum")
    assert out[1][2][0] == GOLD["bcast_sum_rank2_leaf0_from_100"]


def test_fig2_reduce_sum():
    roots = [np.zeros(len(x), np.int64) for x in GOLD["roots"]]
    out = run_gpu(FIG, "reduce", [fig_arrays("leaves"), roots], op="sum")
    assert_same(out[1], fig_arrays("reduce_sum_from_zero_roots"))


def test_fig2_gather_and_scatter_roundtrip():
    multi = [np.full(int(n), -7777, np.int64) for n in GOLD["multi_nroots"]]
    out = run_gpu(FIG, "gather", [fig_arrays("leaves"), multi])
    assert_same(out[1], fig_arrays("gather_multiroot"))
    back = run_gpu(FIG, "scatter", [out[1], [np.zeros(len(x), np.int64) for x in GOLD["leaves"]]])
    want = fig_arrays("leaves")
    want[1][2] = 0  # isolated leaf 230 is untouched by scatter
    assert_same(back[1], want)


def test_fig2_fetch_sum_ascending_rank_order():
    specs = [sf.GraphSpec(1, 0), sf.GraphSpec(0, 1, None, np.array([0], np.int32), np.array([0])),
             sf.GraphSpec(0, 1, None, np.array([0], np.int32), np.array([0]))]
    g = GOLD["fetch_sum_one_root"]
    roots = [np.array([g["root0"]]), np.zeros(0, np.int64), np.zeros(0, np.int64)]
    leaves = [np.zeros(0, np.int64), np.array([g["leaf_rank1"]]), np.array([g["leaf_rank2"]])]
    upd = [np.zeros(0, np.int64), np.array([-1]), np.array([-1])]
    r, _, u = run_gpu(specs, "fetch_and_op", [roots, leaves, upd], op="sum")
    assert r[0][0] == g["root_after"]
    assert u[1][0] == g["update_rank1"] and u[2][0] == g["update_rank2"]


def test_fig2_fetch_prod_degree_one():
    specs = [sf.GraphSpec(1, 0), sf.GraphSpec(0, 1, None, np.array([0], np.int32), np.array([0]))]
    g = GOLD["fetch_prod_degree_one"]
    r, _, u = run_gpu(specs, "fetch_and_op",
                      [[np.array([g["root0"]]), np.zeros(0, np.int64)],
                       [np.zeros(0, np.int64), np.array([g["leaf"]])],
                       [np.zeros(0, np.int64), np.array([-1])]], op="prod")
    assert r[0][0] == g["root_after"] and u[1][0] == g["update"]


def test_reduce_max_keeps_larger_root():
    specs = [sf.GraphSpec(1, 0), sf.GraphSpec(0, 1, None, np.array([0], np.int32), np.array([0]))]
    r = run_gpu(specs, "reduce", [[np.zeros(0, np.int64), np.array([3])],
                                  [np.array([5]), np.zeros(0, np.int64)]], op="max")
    assert r[1][0][0] == 5


def test_edge_free_forest_leaves_data_untouched():
    specs = [sf.GraphSpec(2, 0), sf.GraphSpec(2, 0)]
    out = run_gpu(specs, "bcast", [[np.array([5, 6])] * 2, [np.array([7, 8])] * 2])
    assert_same(out[1], [np.array([7, 8])] * 2)


def test_opaque_bytes_move_verbatim():
    specs = [sf.GraphSpec(2, 0), sf.GraphSpec(0, 2, None, np.array([0, 0], np.int32), np.array([1, 0]))]
    root = [np.arange(6, dtype=np.uint8), np.zeros(0, np.uint8)]
    leaf = [np.zeros(0, np.uint8), np.zeros(6, np.uint8)]
    out = run_gpu(specs, "bcast", [root, leaf], blocklen=3)
    assert out[1][1].tolist() == [3, 4, 5, 0, 1, 2]


# -------------------------------------------------- random forests vs oracle
SEEDS = list(range(12))


def _trial(seed):
    meta = graphs.Rng(graphs.mix_seed(seed, 0x11))
    nranks = meta.range(1, 6)
    return graphs.random_graph_specs(seed * 7919 + 13, nranks, 40)


@pytest.mark.parametrize("seed", SEEDS)
@pytest.mark.parametrize("dtype", [np.int64, np.float64, np.int32])
def test_random_all_ops_vs_oracle(seed, dtype):
    specs = _trial(seed)
    bl = 1 + seed % 3
    roots = rank_data(specs, seed, dtype, bl, 100, "root")
    leaves = rank_data(specs, seed, dtype, bl, 200, "leaf")
    bops = ["replace", "sum", "max", "min", "prod"]
    rops = ["sum", "max", "min", "prod", "replace"] + (["bor", "band", "land", "lor"] if dtype != np.float64 else [])
    bop, rop = bops[seed % len(bops)], rops[seed % len(rops)]
    fp = np.dtype(dtype) == np.float64
    # bcast
    out = run_gpu(specs, "bcast", [roots, leaves], op=bop, blocklen=bl)
    assert_same(out[1], O.bcast(specs, roots, leaves, bop, bl), what=f"bcast {bop}")
    # reduce (replace with duplicate roots is 'any one contribution': skip exact check)
    if rop != "replace":
        out = run_gpu(specs, "reduce", [leaves, roots], op=rop, blocklen=bl)
        assert_same(out[1], O.reduce(specs, leaves, roots, rop, bl), what=f"reduce {rop}")
    # gather / scatter
    deg = O.degrees(specs)
    multi = [np.zeros(int(d.sum()) * bl, dtype) for d in deg]
    out = run_gpu(specs, "gather", [leaves, multi], blocklen=bl)
    og = O.gather(specs, leaves, bl)
    assert_same(out[1], og, what="gather")
    out = run_gpu(specs, "scatter", [og, leaves], blocklen=bl)
    assert_same(out[1], O.scatter(specs, og, leaves, bl), what="scatter")
    # fetch-and-op, deterministic order: bit-exact even for float64
    fop = ["sum", "max", "min", "prod"][seed % 4]
    upd = [np.array(l, copy=True) for l in leaves]
    r, _, u = run_gpu(specs, "fetch_and_op", [roots, leaves, upd], op=fop, blocklen=bl)
    orr, ou = O.fetch_and_op(specs, roots, leaves, upd, fop, bl)
    assert_same(r, orr, what=f"fetch root {fop}")
    assert_same(u, ou, what=f"fetch update {fop}")


@pytest.mark.parametrize("seed", SEEDS[:6])
def test_split_transparency_force_remote(seed):
    """selfcheck.cpp:386-418: routing self edges through the transport gives
    identical results."""
    specs = _trial(seed)
    roots = rank_data(specs, seed, np.float64, 1, 100, "root")
    leaves = rank_data(specs, seed, np.float64, 1, 200, "leaf")
    for opk, data, op in (("bcast", [roots, leaves], "sum"), ("reduce", [leaves, roots], "sum")):
        a = run_gpu(specs, opk, data, op=op)
        b = run_gpu(specs, opk, data, op=op, config=sf.CommConfig(force_remote=True))
        assert_same(b[1], a[1], what=f"{opk} force_remote")
    upd = [np.zeros_like(l) for l in leaves]
    a = run_gpu(specs, "fetch_and_op", [roots, leaves, upd], op="sum")
    b = run_gpu(specs, "fetch_and_op", [roots, leaves, upd], op="sum",
                config=sf.CommConfig(force_remote=True))
    assert_same(b[0], a[0])
    assert_same(b[2], a[2])


@pytest.mark.parametrize("seed", SEEDS[:4])
def test_p2p_put_path_single_rank_force_remote(seed):
    """The one-sided put/signal path (backend p2p) on one GPU: with
    force_remote the self edges become a remote group whose put kernel stores
    into this rank's own mapped slot, raises its arrive flag and frees it —
    the same kernels and stream waits the multi-GPU path runs."""
    specs = graphs.random_graph_specs(seed * 31 + 7, 1, 400)
    roots = rank_data(specs, seed, np.float64, 2, 100, "root")
    leaves = rank_data(specs, seed, np.float64, 2, 200, "leaf")
    cfg = lambda: sf.CommConfig(backend="p2p", force_remote=True)  # noqa: E731
    out = run_gpu(specs, "bcast", [roots, leaves], op="replace", blocklen=2, config=cfg())
    assert_same(out[1], O.bcast(specs, roots, leaves, "replace", 2), what="bcast")
    out = run_gpu(specs, "reduce", [leaves, roots], op="sum", blocklen=2, config=cfg())
    assert_same(out[1], O.reduce(specs, leaves, roots, "sum", 2), what="reduce")
    upd = [np.zeros_like(x) for x in leaves]
    r, _, u = run_gpu(specs, "fetch_and_op", [roots, leaves, upd], op="sum", blocklen=2, config=cfg())
    orr, ou = O.fetch_and_op(specs, roots, leaves, upd, "sum", 2)
    assert_same(r, orr, what="fetch root")
    assert_same(u, ou, what="fetch update")
    deg = O.degrees(specs)
    multi = [np.zeros(int(d.sum()) * 2) for d in deg]
    out = run_gpu(specs, "gather", [leaves, multi], blocklen=2, config=cfg())
    assert_same(out[1], O.gather(specs, leaves, 2), what="gather")


@pytest.mark.parametrize("seed", SEEDS[:6])
def test_free_order_mode(seed):
    """deterministic=False: integer results exact, float within 1e-12, fetch
    updates form a valid serialization (selfcheck.cpp:631-672)."""
    specs = _trial(seed)
    cfg = sf.CommConfig(deterministic=False)
    roots = rank_data(specs, seed, np.int64, 1, 100, "root", 1, 1000)
    leaves = rank_data(specs, seed, np.int64, 1, 200, "leaf", 1, 1000)
    out = run_gpu(specs, "reduce", [leaves, roots], op="sum", config=cfg)
    assert_same(out[1], O.reduce(specs, leaves, roots, "sum"))
    fr = [r.astype(np.float64) / 7 for r in roots]
    fl = [l.astype(np.float64) / 3 for l in leaves]
    out = run_gpu(specs, "reduce", [fl, fr], op="sum", config=cfg)
    assert_same(out[1], O.reduce(specs, fl, fr, "sum"), fp_tol=True)
    upd = [np.zeros_like(l) for l in leaves]
    r, _, u = run_gpu(specs, "fetch_and_op", [roots, leaves, upd], op="sum", config=cfg)
    orr, _ = O.fetch_and_op(specs, roots, leaves, upd, "sum")
    assert_same(r, orr)
    # prefix-chain check: per root, sorting contributions by fetched value
    # (positive contributions => strictly increasing chain) reproduces it.
    rr, ro, lr, li = O.edges(specs)
    per_root = {}
    for e in range(rr.size):
        per_root.setdefault((rr[e], ro[e]), []).append((u[lr[e]][li[e]], leaves[lr[e]][li[e]]))
    for (rk, off), pairs in per_root.items():
        acc = roots[rk][off]
        for fetched, c in sorted(pairs):
            assert fetched == acc
            acc += c
        assert acc == r[rk][off]


# ------------------------------------------------------------- API behaviour
def _one_rank(body, cfg=None):
    return sf.run_ranks(cfg or sf.CommConfig(nranks=1), body)[0]


def _identity(comm, n):
    f = sf.StarForest(comm)
    f.set_graph(n, n, None, [(comm.rank(), i) for i in range(n)])
    f.setup()
    return f


def test_double_end_and_wrong_kind_rejected():
    def body(c):
        f = _identity(c, 2)
        root, leaf = to_dev(np.array([1, 2])), to_dev(np.zeros(2, np.int64))
        h = sf.bcast_begin(f, I64, root, leaf, sf.ReduceOp.replace)
        with pytest.raises(sf.Error, match="different operation"):
            sf.reduce_end(h)
        sf.bcast_end(h)
        with pytest.raises(sf.Error, match="already ended"):
            sf.bcast_end(h)
        return True
    assert _one_rank(body)


def test_fetch_rejects_replace_and_bytes_reject_sum():
    def body(c):
        f = _identity(c, 2)
        a = to_dev(np.array([1, 2]))
        with pytest.raises(sf.Error, match="no fetch semantics"):
            sf.fetch_and_op(f, I64, a, a.clone(), a.clone(), sf.ReduceOp.replace)
        b = to_dev(np.zeros(8, np.uint8))
        with pytest.raises(sf.Error, match="non-opaque"):
            sf.bcast(f, sf.Unit(sf.Kind.bytes, 4), b, b.clone(), sf.ReduceOp.sum)
        sf.bcast(f, sf.Unit(sf.Kind.bytes, 4), b, b.clone(), sf.ReduceOp.replace)
        return True
    assert _one_rank(body)


def test_simultaneous_handles_end_out_of_order():
    """test_sfops.cpp:219-237."""
    def body(c):
        r = c.rank()
        f = sf.StarForest(c)
        f.set_graph_spec(FIG[r])
        f.setup()
        roots = to_dev(np.array(GOLD["roots"][r]))
        roots2 = roots * 2
        la = to_dev(np.array(GOLD["leaves"][r]))
        lb = la.clone()
        ha = sf.bcast_begin(f, I64, roots, la, sf.ReduceOp.replace)
        hb = sf.bcast_begin(f, I64, roots2, lb, sf.ReduceOp.replace)
        sf.bcast_end(hb)
        sf.bcast_end(ha)
        import torch
        torch.cuda.synchronize()
        return to_host(la).tolist(), to_host(lb).tolist()
    got = sf.run_ranks(sf.CommConfig(nranks=3), body)
    assert got[0][0] == [23, 21, 21, 13]
    assert got[0][1] == [46, 42, 42, 26]


def test_debug_checksum_detects_mutation():
    def body(c):
        f = _identity(c, 2)
        root, leaf = to_dev(np.array([1, 2])), to_dev(np.zeros(2, np.int64))
        h = sf.bcast_begin(f, I64, root, leaf, sf.ReduceOp.replace)
        root[0] = 99
        sf.bcast_end(h)
    with pytest.raises(sf.HarnessError, match="mutated"):
        sf.run_ranks(sf.CommConfig(nranks=1, debug_checksum=True), body)


def test_operation_requires_setup():
    def body(c):
        f = sf.StarForest(c)
        f.set_graph(1, 1, None, [(0, 0)])
        a = to_dev(np.array([1]))
        with pytest.raises(sf.Error, match="set-up"):
            sf.bcast(f, I64, a, a.clone(), sf.ReduceOp.replace)
        return True
    assert _one_rank(body)


# ---------------------------------------------------- BASELINE-shaped graphs
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_g2l_halo_bcast_reduce_vs_oracle(P):
    N = 12
    specs = [graphs.g2l_halo(N, P, r) for r in range(P)]
    g = [graphs.G2L(N, P, r) for r in range(P)]
    roots = [graphs.gen_f64(5, r, x.n_owned) for r, x in enumerate(g)]
    leaves = [np.full(x.n_local, -1.0) for x in g]
    out = run_gpu(specs, "bcast", [roots, leaves])
    want = O.bcast(specs, roots, leaves)
    assert_same(out[1], want, what="g2l bcast")
    out2 = run_gpu(specs, "reduce", [want, roots], op="sum")
    assert_same(out2[1], O.reduce(specs, want, roots, "sum"), what="g2l reduce")


def test_config1_shape_small():
    specs = graphs.random_leaf_root(1 << 14, 1 << 12)
    roots = [graphs.gen_f64(1, 7, 1 << 12)]
    leaves = [np.zeros(1 << 14)]
    out = run_gpu(specs, "bcast", [roots, leaves])
    assert_same(out[1], O.bcast(specs, roots, leaves))
    out = run_gpu(specs, "reduce", [[graphs.gen_f64(1, 8, 1 << 14)], roots], op="sum")
    assert_same(out[1], O.reduce(specs, [graphs.gen_f64(1, 8, 1 << 14)], roots, "sum"))


@pytest.mark.parametrize("P", [1, 4])
@pytest.mark.parametrize("dtype", [np.int64, np.float64])
def test_config4_high_contention(P, dtype):
    L, R = 1 << 16, 1 << 8
    specs = graphs.random_leaf_root(L, R, P, seed=4)
    roots = rank_data(specs, 4, dtype, 1, 100, "root", 1, 1000)
    leaves = rank_data(specs, 4, dtype, 1, 200, "leaf", 1, 1000)
    out = run_gpu(specs, "reduce", [leaves, roots], op="sum")
    assert_same(out[1], O.reduce(specs, leaves, roots, "sum"))
    upd = [np.zeros_like(l) for l in leaves]
    r, _, u = run_gpu(specs, "fetch_and_op", [roots, leaves, upd], op="sum")
    orr, ou = O.fetch_and_op(specs, roots, leaves, upd, "sum")
    assert_same(r, orr)
    assert_same(u, ou)


def test_csr_l2_pieces_exact_order():
    """Leaf array (64 MB) several times a 16 MB piece: the warp CSR walks
    L2-sized leaf windows piece-major (kernels.cu run_csr_warp). Fold order
    per root is unchanged, so float64 Reduce/FetchAndOp stay bit-exact."""
    L, R = 1 << 23, 1 << 16
    specs = graphs.random_leaf_root(L, R, 1, seed=4)
    roots = rank_data(specs, 4, np.float64, 1, 100, "root", 1, 1000)
    leaves = rank_data(specs, 4, np.float64, 1, 200, "leaf", 1, 1000)
    out = run_gpu(specs, "reduce", [leaves, roots], op="sum")
    assert_same(out[1], O.reduce(specs, leaves, roots, "sum"))
    upd = [np.zeros_like(x) for x in leaves]
    r, _, u = run_gpu(specs, "fetch_and_op", [roots, leaves, upd], op="sum")
    orr, ou = O.fetch_and_op(specs, roots, leaves, upd, "sum")
    assert_same(r, orr)
    assert_same(u, ou)


@pytest.mark.parametrize("permute", [None, 3])
def test_config3_ghost_sf(permute):
    specs = [graphs.laplacian27_ghosts(10, (2, 2, 2), r, permute) for r in range(8)]
    roots = [graphs.gen_f64(3, r, int(s.nroots)) for r, s in enumerate(specs)]
    leaves = [np.zeros(s.leaf_bound()) for s in specs]
    out = run_gpu(specs, "bcast", [roots, leaves])
    assert_same(out[1], O.bcast(specs, roots, leaves))
    out = run_gpu(specs, "reduce", [leaves, roots], op="sum")
    assert_same(out[1], O.reduce(specs, leaves, roots, "sum"))


def test_pingpong_shape():
    specs = graphs.pingpong(1 << 12)
    n = 1 << 9
    roots = [np.arange(n, dtype=np.int64), np.zeros(0, np.int64)]
    leaves = [np.zeros(0, np.int64), np.zeros(n, np.int64)]
    out = run_gpu(specs, "bcast", [roots, leaves])
    assert out[1][1].tolist() == list(range(n))
    out = run_gpu(specs, "reduce", [out[1], [np.zeros(n, np.int64), np.zeros(0, np.int64)]])
    assert out[1][0].tolist() == list(range(n))
