"""Host-side planner (SetUp) through the C ABI on host-only communicators:
golden two-sided info, degrees, multi-SF, validation messages, pattern
classification. Mirrors /root/reference/proj/tests/test_sfgraph.cpp and
test_pattern.cpp; cross-checked against the reference library when built."""
import json
import os

import numpy as np
import pytest

from paper_2102_13018_b200 import graphs, sf

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig2.json")))
FIG = sf.graph_text_parse(GOLD["graph_text"])
HOST = sf.CommConfig


def run_host(n, body, **kw):
    return sf.run_ranks(sf.CommConfig(nranks=n, **kw), body, devices=[-1] * n)


def setup_all(specs, alg=sf.SetupAlg.automatic):
    def body(c):
        f = sf.StarForest(c)
        f.set_graph_spec(specs[c.rank()])
        f.setup(alg)
        return f.two_sided(), f.compute_degrees().tolist(), f.multi_sf().nroots(), \
            [g.pattern for g in f.root_groups()], [g.pattern for g in f.leaf_groups()]
    return run_host(len(specs), body)


@pytest.mark.parametrize("alg", list(sf.SetupAlg))
def test_fig2_two_sided_golden(alg):
    got = setup_all(FIG, alg)
    for r in range(3):
        ti = got[r][0]
        want = GOLD["two_sided"][str(r)]
        assert [[g, it] for g, it in ti.root_ranks] == want["root_ranks"]
        assert [[g, it] for g, it in ti.leaf_ranks] == want["leaf_ranks"]
    assert got[0][0].self_first and not got[1][0].self_first


def test_fig2_degrees_and_multi_sf():
    got = setup_all(FIG)
    assert [g[1] for g in got] == GOLD["degrees"]
    assert [g[2] for g in got] == GOLD["multi_nroots"]


def test_set_graph_validation_messages():
    def body(c):
        f = sf.StarForest(c)
        with pytest.raises(sf.Error, match="forest property"):
            f.set_graph(1, 2, [0, 0], [(0, 0), (0, 0)])
        with pytest.raises(sf.Error, match="negative leaf index"):
            f.set_graph(1, 1, [-1], [(0, 0)])
        with pytest.raises(sf.Error, match="outside communicator"):
            f.set_graph(1, 1, None, [(5, 0)])
        with pytest.raises(sf.Error, match="length does not match"):
            f.set_graph(1, 2, [0], [(0, 0), (0, 0)])
        with pytest.raises(sf.Error, match="negative root or leaf count"):
            f.set_graph(-1, 0, None, [])
        with pytest.raises(sf.Error):
            f.setup()  # not graph-set
        f.set_graph(1, 1, None, [(0, 0)])
        with pytest.raises(sf.Error, match="set-up"):
            f.two_sided()
        f.setup()
        assert f.state() == sf.SfState.set_up
        with pytest.raises(sf.Error):
            f.setup()  # second setup
        return True
    assert run_host(1, body) == [True]


def test_setup_validates_root_offsets():
    """test_sfgraph.cpp:167-184."""
    def body(c):
        f = sf.StarForest(c)
        if c.rank() == 0:
            f.set_graph(1, 1, None, [(1, 7)])
        else:
            f.set_graph(2, 0, None, [])
        f.setup()
    with pytest.raises(sf.HarnessError, match="root offset"):
        run_host(2, body, timeout_s=5.0)


def test_self_only_forest_puts_self_first():
    def body(c):
        f = sf.StarForest(c)
        f.set_graph(2, 2, None, [(c.rank(), 1), (c.rank(), 0)])
        f.setup()
        ti = f.two_sided()
        return ti.self_first, ti.root_ranks[0][0], ti.leaf_ranks[0][0]
    got = run_host(2, body)
    assert got == [(True, 0, 0), (True, 1, 1)]


def test_edge_free_and_degree_one_multi_sf():
    def body(c):
        f = sf.StarForest(c)
        f.set_graph(3, 0, None, [])
        f.setup()
        g = sf.StarForest(c)
        other = 1 - c.rank()
        g.set_graph(3, 3, None, [(other, i) for i in range(3)])
        g.setup()
        m = g.multi_sf()
        return f.compute_degrees().tolist(), f.multi_sf().nroots(), m.nroots(), \
            m.graph_spec().remote_rank.tolist()
    got = run_host(2, body)
    assert got[0][0] == [0, 0, 0] and got[0][1] == 0
    assert got[0][2] == 3 and got[0][3] == [1, 1, 1]


# ---------------------------------------------------------------- patterns
def test_pattern_kats():
    """test_pattern.cpp KATs (reference classification = infer_affine False)."""
    p = sf.analyze([4, 5, 6, 7])
    assert p.kind == "contiguous" and p.start == 4 and p.count == 4
    p = sf.analyze([10, 11, 14, 15], infer_affine=False, extents=(4, 16))
    assert (p.kind, p.start, p.dx, p.dy, p.dz, p.s1, p.s2) == ("affine", 10, 2, 2, 1, 4, 16)
    idx = [7 + 20 * k + 5 * j + i for k in range(2) for j in range(3) for i in range(2)]
    p = sf.analyze(idx, infer_affine=False, extents=(5, 20))
    assert (p.dx, p.dy, p.dz, p.count) == (2, 3, 2, 12)
    # reference: no blind inference without extents
    assert sf.analyze([10, 11, 14, 15], infer_affine=False).kind == "indexed"
    p = sf.analyze([3, 1, 3])
    assert p.kind == "indexed" and p.has_duplicates
    assert not sf.analyze([3, 1, 2]).has_duplicates
    assert sf.analyze([]).bound == 0
    assert sf.analyze([9, 2, 5]).bound == 10


def test_affine_inference_without_extents():
    """The planner's own inference: faces and subblocks of
    a ghosted box are recognised from the indices alone."""
    X, XY = 14, 14 * 13
    sub = [3 + XY * k + X * j + i for k in range(4) for j in range(5) for i in range(6)]
    p = sf.analyze(sub)
    assert (p.kind, p.dx, p.dy, p.dz, p.s1, p.s2) == ("affine", 6, 5, 4, X, XY)
    xface = [X * j + XY * k for k in range(1, 4) for j in range(1, 5)]
    p = sf.analyze(xface)
    assert p.kind == "affine" and p.dx == 1 and p.count == 12
    rng = np.random.default_rng(0)
    for _ in range(100):
        idx = rng.integers(0, 60, size=rng.integers(0, 40))
        p = sf.analyze(idx)
        enum = _enumerate(p, idx)
        assert enum == list(idx)


def _enumerate(p, idx):
    if p.kind == "contiguous":
        return list(range(p.start, p.start + p.count))
    if p.kind == "affine":
        return [p.start + p.s2 * k + p.s1 * j + x for k in range(p.dz) for j in range(p.dy)
                for x in range(p.dx)]
    return list(idx)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_g2l_plan_patterns_are_structured(P):
    """Config 2: every group of the G2L SF is contiguous or affine (no index arrays)."""
    specs = [graphs.g2l_halo(10, P, r) for r in range(P)]
    got = setup_all(specs)
    for r in range(P):
        for pat in got[r][3] + got[r][4]:
            assert pat.kind in ("contiguous", "affine"), (r, pat)


def test_planner_matches_reference_two_sided():
    """SetUp parity with the reference library on its own random forests."""
    from oracle import ref

    if not ref.available():
        pytest.skip("reference library not built")
    for seed in range(15):
        nranks = 1 + seed % 6
        specs = graphs.random_graph_specs(seed, nranks, 30)
        want = ref.two_sided(specs)
        got = setup_all(specs)
        for r in range(nranks):
            assert [list(x) for x in got[r][0].root_ranks] == [list(x) for x in want[r][0]]
            assert [list(x) for x in got[r][0].leaf_ranks] == [list(x) for x in want[r][1]]


def _relation_trial(t):
    """selfcheck.cpp:243-283 shapes: random relations up to 8 ranks,
    including empty and all-to-one relations."""
    rng = graphs.Rng(graphs.mix_seed(t, 0x5D))
    nranks = rng.range(1, 8)
    kind = t % 4
    specs = []
    for r in range(nranks):
        if kind == 0:  # empty relation
            specs.append(sf.GraphSpec(rng.range(0, 5), 0))
        elif kind == 1:  # all-to-one: every leaf on rank 0's roots
            n = rng.range(0, 12)
            specs.append(sf.GraphSpec(8 if r == 0 else 0, n, None, np.zeros(n, np.int32),
                                      np.array([rng.bounded(8) for _ in range(n)], np.int64)))
        else:
            specs = graphs.random_graph_specs(9000 + t, nranks, 24)
            break
    return specs


@pytest.mark.parametrize("t", range(24))
def test_setup_duality_dense_vs_consensus(t):
    """selfcheck.cpp:285-327 (SPEC.md acceptance 3): dense and consensus
    discovery give identical TwoSidedInfo, and the (root rank, root offset,
    leaf rank) edge multisets seen from the root side and from the leaf side
    both equal the graph's."""
    specs = _relation_trial(t)
    n = len(specs)

    def body(c):
        a, b = sf.StarForest(c), sf.StarForest(c)
        a.set_graph_spec(specs[c.rank()])
        b.set_graph_spec(specs[c.rank()])
        a.setup(sf.SetupAlg.dense)
        b.setup(sf.SetupAlg.consensus)
        return a.two_sided(), b.two_sided()

    got = run_host(n, body)
    from_root, from_leaf, from_graph = [], [], []
    for q in range(n):
        dense, cons = got[q]
        assert dense == cons, q
        spec = specs[q]
        for rank, ords in dense.root_ranks:
            from_root += [(rank, int(spec.remote_off[o]), q) for o in ords]
        for rank, offs in dense.leaf_ranks:
            from_leaf += [(q, int(o), rank) for o in offs]
        from_graph += [(int(spec.remote_rank[o]), int(spec.remote_off[o]), q) for o in range(int(spec.nleaves))]
    assert sorted(from_root) == sorted(from_graph)
    assert sorted(from_leaf) == sorted(from_graph)
