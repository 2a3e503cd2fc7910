"""Graph algebra (starforest.hpp:150-171) on host-only communicators: the
reference's own test cases (test_sfgraph.cpp:266-484) — identities, the
sequential reachability join oracle over 12 random trials, inversion,
preconditions, embeddings of the worked example."""
import numpy as np
import pytest

from paper_2102_13018_b200 import graphs, sf
from paper_2102_13018_b200.graphs import GraphSpec, Rng, mix_seed
from tests.test_cpu_planner import FIG, run_host


def edges_of(f):
    """Local edge multiset (root rank, root off, leaf index) of a forest."""
    s = f.graph_spec()
    idx = s.local if s.local is not None else np.arange(s.nleaves)
    return sorted(zip(s.remote_rank.tolist(), s.remote_off.tolist(), list(map(int, idx))))


def global_edges(specs):
    out = []
    for r, s in enumerate(specs):
        idx = s.local if s.local is not None else np.arange(s.nleaves)
        for i in range(s.nleaves):
            out.append((int(s.remote_rank[i]), int(s.remote_off[i]), r, int(idx[i])))
    return sorted(out)


def test_compose_with_identity_is_the_other_graph():
    spec = graphs.random_graph_specs(5, 3, 12)

    def body(c):
        b = sf.StarForest(c)
        b.set_graph_spec(spec[c.rank()])
        b.setup()
        idr = sf.identity_sf(c, b.nroots())
        idr.setup()
        left = sf.compose(idr, b)
        idl = sf.identity_sf(c, b.leaf_index_bound())
        idl.setup()
        right = sf.compose(b, idl)
        return edges_of(left) == edges_of(b), edges_of(right) == edges_of(b), left.nroots() == b.nroots()

    assert all(all(x) for x in run_host(3, body))


def b_specs_for(seed, a_specs, nranks):
    """test_sfgraph.cpp:292-312: B's root space covers A's leaf space."""
    rng = Rng(mix_seed(seed, 0x81))
    b_roots = []
    for r in range(nranks):
        s = a_specs[r]
        idx = s.local if s.local is not None else np.arange(s.nleaves)
        bound = int(idx.max()) + 1 if s.nleaves else 0
        b_roots.append(bound + rng.range(0, 3))
    out = []
    for r in range(nranks):
        want = rng.range(0, 8)
        rr, ro = [], []
        for _ in range(want):
            owner = rng.bounded(nranks)
            if b_roots[owner] == 0:
                continue
            rr.append(owner)
            ro.append(rng.range(0, b_roots[owner] - 1))
        out.append(GraphSpec(b_roots[r], len(rr), None, np.array(rr, np.int32), np.array(ro, np.int64)))
    return out


@pytest.mark.parametrize("t", range(12))
def test_compose_matches_sequential_join(t):
    seed = 400 + t
    P = 4
    a_specs = graphs.random_graph_specs(seed, P, 10)
    b_specs = b_specs_for(seed, a_specs, P)
    a_by_leaf = {(lr, li): (rr, ro) for rr, ro, lr, li in global_edges(a_specs)}
    expect = sorted((*a_by_leaf[(rr, ro)], lr, li) for rr, ro, lr, li in global_edges(b_specs)
                    if (rr, ro) in a_by_leaf)

    def body(c):
        a, b = sf.StarForest(c), sf.StarForest(c)
        a.set_graph_spec(a_specs[c.rank()])
        b.set_graph_spec(b_specs[c.rank()])
        a.setup()
        b.setup()
        ab = sf.compose(a, b)
        assert ab.nroots() == a.nroots()
        return ab.graph_spec()

    got = run_host(P, body)
    assert global_edges(got) == expect


def test_compose_inverse_of_identity_inverts():
    n = 4

    def body(c):
        b = sf.StarForest(c)
        b.set_graph(n, n, None, [((c.rank() + 1) % 3, i) for i in range(n)])
        b.setup()
        idf = sf.identity_sf(c, n)
        idf.setup()
        ab = sf.compose_inverse(idf, b)
        s = ab.graph_spec()
        idx = s.local if s.local is not None else np.arange(s.nleaves)
        return (ab.nleaves() == n and all(int(r) == (c.rank() + 2) % 3 for r in s.remote_rank)
                and all(int(o) == int(i) for o, i in zip(s.remote_off, idx)))

    assert all(run_host(3, body))


def test_compose_inverse_with_identity_b_returns_a():
    spec = graphs.random_graph_specs(9, 2, 10)

    def body(c):
        a = sf.StarForest(c)
        a.set_graph_spec(spec[c.rank()])
        a.setup()
        idf = sf.identity_sf(c, a.leaf_index_bound())
        idf.setup()
        return edges_of(sf.compose_inverse(a, idf)) == edges_of(a)

    assert all(run_host(2, body))


def test_compose_inverse_rejects_degree_two():
    def body(c):
        b = sf.StarForest(c)
        if c.rank() == 0:
            b.set_graph(1, 2, None, [(0, 0), (0, 0)])
        else:
            b.set_graph(0, 0, None, [])
        b.setup()
        idf = sf.identity_sf(c, b.leaf_index_bound())
        idf.setup()
        with pytest.raises(sf.Error, match="degree"):
            sf.compose_inverse(idf, b)
        return True

    assert all(run_host(2, body))


def _fig(c):
    f = sf.StarForest(c)
    f.set_graph_spec(FIG[c.rank()])
    f.setup()
    return f


def leaf_indices(f):
    s = f.graph_spec()
    idx = s.local if s.local is not None else np.arange(s.nleaves)
    return [int(i) for i in idx]


def test_embed_root_keeps_selected_roots_edges():
    def body(c):
        f = _fig(c)
        e = sf.embed_root(f, [0] if c.rank() == 1 else [])
        assert e.nroots() == f.nroots()
        return leaf_indices(e)

    assert run_host(3, body) == [[1, 2], [], [1]]


def test_embed_root_everything_and_nothing():
    spec = graphs.random_graph_specs(21, 3, 12)

    def body(c):
        f = sf.StarForest(c)
        f.set_graph_spec(spec[c.rank()])
        f.setup()
        allr = list(range(f.nroots())) * 2  # duplicates collapse silently
        none = sf.embed_root(f, [])
        return edges_of(sf.embed_root(f, allr)) == edges_of(f), none.nleaves() == 0, none.nroots() == f.nroots()

    assert all(all(x) for x in run_host(3, body))


def test_embed_validates_selection_range():
    def body(c):
        f = sf.identity_sf(c, 3)
        f.setup()
        with pytest.raises(sf.Error, match="out of range"):
            sf.embed_root(f, [3])
        with pytest.raises(sf.Error, match="negative"):
            sf.embed_leaf(f, [-1])
        return True

    assert all(run_host(1, body))


def test_embed_leaf_filters_without_remapping():
    def body(c):
        return leaf_indices(sf.embed_leaf(_fig(c), [0, 1]))

    assert run_host(3, body) == [[0, 1], [0, 1], [0, 1]]
