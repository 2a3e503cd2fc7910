"""Pin the closed-form config 2 checks (graphs.g2l_check / g2l_reduce_expect),
which bench.py and the full-size multi-GPU test apply at 512^3 where the
oracle cannot run, against the C oracle on small grids at every process-grid
shape the bench uses (and the 2,2,1 / 2,2,2 x-face shapes)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2102_13018_b200 import graphs


@pytest.mark.parametrize("N,P,dims", [(7, 1, None), (8, 2, None), (9, 4, None), (10, 4, (2, 2, 1)),
                                      (9, 8, None), ((11, 7, 6), 8, (2, 2, 2)), (6, 3, None)])
def test_g2l_closed_form_matches_oracle(N, P, dims):
    specs = [graphs.g2l_halo(N, P, r, dims=dims) for r in range(P)]
    geo = [graphs.G2L(N, P, r, dims=dims) for r in range(P)]
    ids = [np.arange(g.n_owned, dtype=np.float64) for g in geo]
    leaves = O.bcast(specs, ids, [np.full(g.n_local, -1.0) for g in geo], "replace")
    roots = O.reduce(specs, leaves, ids, "sum")
    for r, g in enumerate(geo):
        chk = graphs.g2l_check(g, torch.from_numpy(leaves[r]), torch.from_numpy(roots[r]))
        assert chk == {"leaf_ok": True, "root_ok": True}, (r, chk)
    # arbitrary values: the per-addition rounded fold
    vals = [graphs.gen_f64(5, r, g.n_owned) * 3.7 for r, g in enumerate(geo)]
    lv = O.bcast(specs, vals, [np.zeros(g.n_local) for g in geo], "replace")
    rv = O.reduce(specs, lv, vals, "sum")
    for r, g in enumerate(geo):
        want = graphs.g2l_reduce_expect(g, torch.from_numpy(vals[r])).numpy()
        assert np.array_equal(want.view(np.int64), rv[r].view(np.int64)), r


def test_g2l_check_detects_a_wrong_ghost():
    N, P = 8, 2
    specs = [graphs.g2l_halo(N, P, r) for r in range(P)]
    geo = [graphs.G2L(N, P, r) for r in range(P)]
    ids = [np.arange(g.n_owned, dtype=np.float64) for g in geo]
    leaves = O.bcast(specs, ids, [np.full(g.n_local, -1.0) for g in geo], "replace")
    roots = O.reduce(specs, leaves, ids, "sum")
    bad = leaves[1].copy()
    g = geo[1]
    bad[g.X * g.Y * 0 + g.X * 2 + 3] += 1.0  # a zl-face ghost of rank 1
    assert graphs.g2l_check(g, torch.from_numpy(bad), torch.from_numpy(roots[1]))["leaf_ok"] is False
    r2 = roots[0].copy()
    r2[-1] += 1.0
    assert graphs.g2l_check(geo[0], torch.from_numpy(leaves[0]), torch.from_numpy(r2))["root_ok"] is False
