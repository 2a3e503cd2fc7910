"""GPU SpMV over the star forest (spmv.hpp:147-169) vs the sequential oracle
(pinned to the reference in test_cpu_spmv.py): bit-exact for float64 and
int64, forward and transpose, random matrices over 1-4 ranks (threads of one
process on one GPU) and the config-3 27-point Laplacian over 8 ranks."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2102_13018_b200 import sf
from paper_2102_13018_b200 import spmv as S
from tests.test_cpu_spmv import trial

pytestmark = pytest.mark.gpu


def run_spmv(A, layout, x, transpose=False, backend="threads", devices=None):
    import torch

    P = layout.nranks()
    dt = torch.float64 if A.vals.dtype == np.float64 else torch.int64

    def body(comm):
        r = comm.rank()
        m = S.split_matrix(A, layout, layout, r)
        f = S.build_ghost_sf(comm, m)
        D, B = S.Matrix(comm, m.diag), S.Matrix(comm, m.offdiag)
        xo = torch.from_numpy(np.ascontiguousarray(x[layout.begin(r):layout.end(r)])).cuda()
        lvec = torch.zeros(len(m.garray), dtype=dt, device="cuda")
        y = torch.full((layout.local_size(r),), 7, dtype=dt, device="cuda")  # overwritten
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            (S.spmv_transpose if transpose else S.spmv)(f, D, B, xo, lvec, y, st)
        st.synchronize()
        return y.cpu().numpy()

    cfg = sf.CommConfig(nranks=P, backend=backend)
    return np.concatenate(sf.run_ranks(cfg, body, devices=devices))


@pytest.mark.parametrize("t", range(12))
def test_random_spmv_bit_exact(t):
    nranks, A, x = trial(t)
    layout = S.Layout.contiguous(A.rows, nranks)
    for transpose in (False, True):
        got = run_spmv(A, layout, x, transpose)
        want = O.spmv(A, layout, x, transpose)
        assert np.array_equal(got.view(np.int64), want.view(np.int64)), (t, transpose)


def test_laplacian27_eight_ranks():
    N, dims = 8, (2, 2, 2)
    blocks = [S.laplacian27_block(N, dims, r) for r in range(8)]
    layout = blocks[0][1]
    rp = np.concatenate([[0]] + [b[0][0][1:] + sum(int(bb[0][0][-1]) for bb in blocks[:r])
                                 for r, b in enumerate(blocks)])
    A = S.Csr(layout.total(), layout.total(), rp.astype(np.int64),
              np.concatenate([b[0][1] for b in blocks]), np.concatenate([b[0][2] for b in blocks]))
    x = np.cos(np.arange(A.rows) * 0.37)
    assert np.array_equal(run_spmv(A, layout, x), O.spmv(A, layout, x))
    assert np.array_equal(run_spmv(A, layout, x, True), O.spmv(A, layout, x, True))


def test_mismatched_blocks_rejected():
    import torch

    A = S.laplacian_5pt(4, 4)
    L = S.Layout.contiguous(16, 2)

    def body(comm):
        m = S.split_matrix(A, L, L, comm.rank())
        f = S.build_ghost_sf(comm, m)
        D = S.Matrix(comm, m.diag)
        x = torch.zeros(8, dtype=torch.float64, device="cuda")
        with pytest.raises(sf.Error, match="do not match the ghost forest"):
            S.spmv(f, D, D, x, x, x)
        return True

    assert all(sf.run_ranks(sf.CommConfig(nranks=2), body))


def _selection_trial(t, seed=1):
    """selfcheck.cpp:765-797 draw for draw (Rng(mix_seed(seed + t*911, 0x77))):
    4 ranks, 8-40 columns, random reduced column lists, disjoint selections
    (trial 0 selects everything); oracle = position in rank-then-list order."""
    from paper_2102_13018_b200 import graphs

    rng = graphs.Rng(graphs.mix_seed(seed + t * 911, 0x77))
    nranks = 4
    ncols = rng.range(8, 40)
    garray = [[c for c in range(ncols) if rng.chance(0.4)] for _ in range(nranks)]
    selected = [[] for _ in range(nranks)]
    for c in range(ncols):
        if t != 0 and rng.chance(0.4):
            continue
        selected[rng.bounded(nranks)].append(c)
    new_index, nxt = {}, 0
    for r in range(nranks):
        for c in selected[r]:
            new_index[c] = nxt
            nxt += 1
    return S.Layout.contiguous(ncols, nranks), garray, selected, new_index


@pytest.mark.parametrize("t", range(20))
def test_select_submatrix_columns(t):
    """SPEC.md acceptance 9 / selfcheck submatrix_selection: a Reduce REPLACE
    + Bcast REPLACE composition over two column forests on the device."""
    layout, garray, selected, new_index = _selection_trial(t)

    def body(comm):
        r = comm.rank()
        sf_a = S.build_column_sf(comm, layout, garray[r])
        sf_b = S.build_column_sf(comm, layout, selected[r])
        return S.select_submatrix_columns(sf_a, sf_b, selected[r]).cpu().numpy()

    got = sf.run_ranks(sf.CommConfig(nranks=4), body)
    for r in range(4):
        want = [new_index.get(c, -1) for c in garray[r]]
        assert got[r].tolist() == want, (t, r)
