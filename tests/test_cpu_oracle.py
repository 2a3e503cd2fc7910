"""Pin the C oracle: against the reference's golden vectors (Fig. 2), against
fixtures produced by the reference library itself (ref_random.npz), and — when
oracle/_ref is built — live against the reference's distributed CPU path. Also
pins the generators' splitmix64 port and random-forest port."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle import ref
from paper_2102_13018_b200 import graphs, sf
from tests.helpers import assert_same, load_golden_cases, rank_data

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig2.json")))
FIG = sf.graph_text_parse(GOLD["graph_text"])
needs_ref = pytest.mark.skipif(not ref.available(), reason="reference library not built")


def arrs(key):
    return [np.array(x, np.int64) for x in GOLD[key]]


def test_oracle_fig2_golden():
    assert_same(O.bcast(FIG, arrs("roots"), arrs("leaves")), arrs("bcast_replace_leaves"))
    zero_roots = [np.zeros_like(x) for x in arrs("roots")]
    assert_same(O.reduce(FIG, arrs("leaves"), zero_roots, "sum"), arrs("reduce_sum_from_zero_roots"))
    assert_same(O.gather(FIG, arrs("leaves")), arrs("gather_multiroot"))
    assert [d.tolist() for d in O.degrees(FIG)] == GOLD["degrees"]
    leaves = [np.zeros_like(x) for x in arrs("leaves")]
    leaves[2][0] = 100
    assert O.bcast(FIG, arrs("roots"), leaves, "sum")[2][0] == GOLD["bcast_sum_rank2_leaf0_from_100"]
    g = GOLD["fetch_sum_one_root"]
    specs = [sf.GraphSpec(1, 0), sf.GraphSpec(0, 1, None, np.array([0], np.int32), np.array([0])),
             sf.GraphSpec(0, 1, None, np.array([0], np.int32), np.array([0]))]
    r, u = O.fetch_and_op(specs, [np.array([10]), np.zeros(0, np.int64), np.zeros(0, np.int64)],
                          [np.zeros(0, np.int64), np.array([5]), np.array([7])],
                          [np.zeros(0, np.int64), np.array([-1]), np.array([-1])], "sum")
    assert r[0][0] == g["root_after"] and u[1][0] == g["update_rank1"] and u[2][0] == g["update_rank2"]


CASES = load_golden_cases()


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_oracle_matches_reference_fixtures(ci):
    opk, dt, op, bl, specs, ins, outs = CASES[ci]
    if opk == "bcast":
        got = [O.bcast(specs, ins[0], ins[1], op, bl)]
    elif opk == "reduce":
        got = [O.reduce(specs, ins[0], ins[1], op, bl)]
    elif opk == "fetch_and_op":
        got = list(O.fetch_and_op(specs, ins[0], ins[1], ins[2], op, bl))
    elif opk == "gather":
        got = [O.gather(specs, ins[0], bl)]
    else:
        got = [O.scatter(specs, ins[0], ins[1], bl)]
    for g, w in zip(got, outs):
        assert_same(g, w, what=f"{opk} {dt} {op} bl={bl}")


@needs_ref
def test_rng_port_matches_reference():
    for seed in (0, 1, 42, 2 ** 63 + 5):
        want, mixed = ref.rng(seed, 64, salt=0x5F0C)
        r = graphs.Rng(seed)
        assert [r.next() for _ in range(32)] == want[:32].tolist()
        assert graphs.Rng(seed).stream(64).tolist() == want.tolist()
        assert graphs.mix_seed(seed, 0x5F0C) == mixed


@needs_ref
@pytest.mark.parametrize("seed", range(20))
def test_random_graph_port_matches_reference(seed):
    nranks = 1 + seed % 8
    want = ref.random_graph(seed, nranks, 40)
    got = graphs.random_graph_specs(seed, nranks, 40)
    for (nr, nl, loc, rr, ro), s in zip(want, got):
        assert (nr, nl) == (s.nroots, s.nleaves)
        assert (loc is None) == (s.local is None)
        if loc is not None:
            assert loc.tolist() == s.local.tolist()
        assert rr.tolist() == s.remote_rank.tolist() and ro.tolist() == s.remote_off.tolist()


@needs_ref
@pytest.mark.parametrize("seed", range(10))
@pytest.mark.parametrize("dtype", [np.int64, np.float64])
def test_oracle_matches_live_reference(seed, dtype):
    specs = graphs.random_graph_specs(seed + 500, 1 + seed % 6, 30)
    roots = rank_data(specs, seed, dtype, 1, 100, "root")
    leaves = rank_data(specs, seed, dtype, 1, 200, "leaf")
    _, b, _ = ref.run(specs, "reduce", leaves, roots, None, "sum")
    assert_same(O.reduce(specs, leaves, roots, "sum"), b)
    upd = [np.zeros_like(x) for x in leaves]
    a, _, c = ref.run(specs, "fetch_and_op", roots, leaves, upd, "sum")
    orr, ou = O.fetch_and_op(specs, roots, leaves, upd, "sum")
    assert_same(orr, a)
    assert_same(ou, c)
    _, b, _ = ref.run(specs, "reduce", leaves, roots, None, "sum", force_remote=True)
    assert_same(O.reduce(specs, leaves, roots, "sum"), b)


def _g2l_brute(N, P, r):
    """Direct restatement of the DMDA global->local map for checking g2l_halo."""
    g = graphs.G2L(N, P, r)
    X, Y = g.X, g.Y
    out = []
    for k in range(g.Z):
        for j in range(Y):
            for i in range(X):
                coords = [(i, g.nx, g.bx, g.px, g.xs), (j, g.ny, g.by, g.py, g.ys),
                          (k, g.nz, g.bz, g.pz, g.zs)]
                outside = [c for c in coords if c[0] == 0 or c[0] == c[1] + 1]
                if len(outside) > 1:
                    continue
                b = [g.bx, g.by, g.bz]
                loc = [i - 1, j - 1, k - 1]
                if outside:
                    ax = coords.index(outside[0])
                    v, n, bb, pp, parts = outside[0]
                    if v == 0 and bb == 0 or v == n + 1 and bb == pp - 1:
                        continue
                    b[ax] += -1 if v == 0 else 1
                    loc[ax] = parts[b[ax]][1] - 1 if v == 0 else 0
                nxo, nyo = g.xs[b[0]][1], g.ys[b[1]][1]
                owner = b[0] + g.px * (b[1] + g.py * b[2])
                out.append((i + X * (j + Y * k), owner, loc[0] + nxo * (loc[1] + nyo * loc[2])))
    return out


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_g2l_generator_matches_brute_force(P):
    for r in range(P):
        s = graphs.g2l_halo(7, P, r)
        want = _g2l_brute(7, P, r)
        got = list(zip(s.local.tolist(), s.remote_rank.tolist(), s.remote_off.tolist()))
        assert got == want
