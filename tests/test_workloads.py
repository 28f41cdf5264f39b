"""Input generators (workloads/): structure of the synthetic matrices."""
import numpy as np

import workloads as W


def test_grid_structure():
    N, th = 9, 0.24
    A = W.grid_gmrf(N, th)
    A.check()
    assert A.nnz == N * N + 4 * N * (N - 1)  # reading G15 nnz formula
    D = W.to_dense(A)
    assert np.array_equal(D, D.T)
    assert np.all(np.diag(D) == 1.0)
    off = D - np.eye(N * N)
    assert set(np.unique(off)) <= {0.0, -th}
    # 4-neighbour, free boundary: corner has 2 neighbours, interior 4
    assert (off[0] != 0).sum() == 2 and (off[N + 1] != 0).sum() == 4


def test_grid_rectangular_and_config_sizes():
    A = W.grid_gmrf(4, 0.1, 7)
    A.check()
    assert A.n_rows == 28
    wl = W.get_workload("gmrf5000")
    assert wl.d == 25_000_000 and wl.a == 1 - 4 * 0.24 and wl.b == 1 + 4 * 0.24


def test_torus_structure():
    T = W.torus_laplacian(6)
    T.check()
    D = W.to_dense(T)
    assert np.array_equal(D, D.T)
    assert np.all(D.sum(1) == 0) and np.all(np.diag(D) == 4)
    assert np.all(np.diff(T.row_ptr) == 5)


def test_random_nonsingular_structure():
    d = 2000
    B = W.random_nonsingular(d, 3)
    B.check()  # sorted unique columns per row
    assert np.all(np.diff(B.row_ptr) == 9)
    D = W.to_dense(B)
    assert np.all(np.diag(D) == 3.0)
    off = D[~np.eye(d, dtype=bool)]
    nz = off[off != 0]
    assert nz.size == 8 * d and np.all(np.abs(nz) < 0.1)
    # deterministic in the seed
    assert np.array_equal(W.random_nonsingular(d, 3).val, B.val)
    assert not np.array_equal(W.random_nonsingular(d, 4).col_idx, B.col_idx)


def test_transpose_exact():
    B = W.random_nonsingular(500, 1)
    Bt = W.transpose(B)
    Bt.check()
    assert np.array_equal(W.to_dense(Bt), W.to_dense(B).T)
    assert np.array_equal(W.transpose(Bt).col_idx, B.col_idx)


def test_random_spd_is_spd():
    S = W.random_spd(300, 2)
    S.check()
    D = W.to_dense(S)
    assert np.array_equal(D, D.T)
    assert np.linalg.eigvalsh(D).min() > 0
