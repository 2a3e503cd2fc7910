"""SpMV consumer (spmv.hpp:147-169) on the CPU: the sequential oracle
restatement (oracle.spmv) pinned bit-exactly to the reference's own
distributed SpMV (oracle/_ref, selfcheck.cpp spmv_trial shape), and the host
structures (Layout, split_matrix, build_column_sf graph)."""
import numpy as np
import pytest

from oracle import oracle as O
from oracle import ref
from paper_2102_13018_b200 import graphs
from paper_2102_13018_b200 import spmv as S

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def trial(t: int):
    """selfcheck.cpp:684-699: 1-4 ranks, n in [8, 64], 1-6 nonzeros per row."""
    rng = graphs.Rng(graphs.mix_seed(1 + t * 4391, 0x66))
    nranks = rng.range(1, 4)
    n = rng.range(8, 64)
    dtype = np.float64 if t % 4 < 2 else np.int64
    A = S.random_sparse(rng, n, rng.range(1, 6), dtype)
    if dtype == np.int64:
        x = np.array([rng.range(-100, 100) for _ in range(n)], np.int64)
    else:
        x = np.array([rng.uniform01() * 4.0 - 2.0 for _ in range(n)])
    return nranks, A, x


@needs_ref
@pytest.mark.parametrize("t", range(16))
def test_oracle_matches_reference_spmv(t):
    nranks, A, x = trial(t)
    layout = S.Layout.contiguous(A.rows, nranks)
    for transpose in (False, True):
        want = ref.spmv(nranks, A.rowptr, A.colind, A.vals, x, transpose)
        got = O.spmv(A, layout, x, transpose)
        assert np.array_equal(got.view(np.int64), want.view(np.int64)), (t, transpose)


@needs_ref
def test_laplacian_5pt_reference():
    A = S.laplacian_5pt(9, 7)
    x = np.linspace(-1, 1, A.rows)
    for P in (1, 2, 3):
        layout = S.Layout.contiguous(A.rows, P)
        assert np.array_equal(O.spmv(A, layout, x), ref.spmv(P, A.rowptr, A.colind, A.vals, x))


def test_layout_and_split():
    L = S.Layout.contiguous(10, 3)
    assert list(L.starts) == [0, 4, 7, 10]
    assert list(L.owner([0, 3, 4, 6, 7, 9])) == [0, 0, 1, 1, 2, 2]
    with pytest.raises(Exception, match="outside the layout"):
        L.owner([10])
    A = S.laplacian_5pt(5, 2)
    m = S.split_matrix(A, L, L, 1)
    assert m.diag.rows == 3 and m.diag.cols == 3
    assert list(m.garray) == sorted(set(m.garray)) and all((g < 4) or (g >= 7) for g in m.garray)
    spec = S.column_sf_spec(L, 1, m.garray)
    assert spec.nroots == 3 and spec.nleaves == len(m.garray)
    assert all(L.begin(r) + o == g for r, o, g in zip(spec.remote_rank, spec.remote_off, m.garray))


def test_laplacian27_block_rows():
    (rp, ci, v), L = S.laplacian27_block(6, (2, 1, 1), 0)
    assert L.total() == 216 and len(rp) - 1 == 108
    deg = np.diff(rp)
    assert deg.min() == 8 and deg.max() == 27  # corners / interior
    assert np.all(np.diff(ci[rp[5]:rp[6]]) > 0)  # columns ascending within a row
