"""Canonical CSR container (sorted, unique column indices).

Layout is the one the C-ABI takes (include/cheb_logdet.h, cl_csr):
row_ptr int64[n_rows+1], col_idx int32[nnz], val float64[nnz].
"""
from dataclasses import dataclass

import numpy as np


@dataclass
class CSR:
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray  # int64 [n_rows+1]
    col_idx: np.ndarray  # int32 [nnz]
    val: np.ndarray      # float64 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def check(self) -> None:
        """Validate canonical form; raises ValueError."""
        rp, ci = self.row_ptr, self.col_idx
        if rp.dtype != np.int64 or ci.dtype != np.int32 or self.val.dtype != np.float64:
            raise ValueError("dtypes must be int64/int32/float64")
        if rp.shape != (self.n_rows + 1,) or rp[0] != 0:
            raise ValueError("bad row_ptr")
        if np.any(np.diff(rp) < 0):
            raise ValueError("row_ptr not monotone")
        if ci.shape != (self.nnz,) or self.val.shape != (self.nnz,):
            raise ValueError("bad nnz arrays")
        if self.nnz and (ci.min() < 0 or ci.max() >= self.n_cols):
            raise ValueError("column out of range")
        # sorted & unique within each row: consecutive diffs > 0 except at row starts
        if self.nnz > 1:
            d = np.diff(ci.astype(np.int64))
            starts = np.zeros(self.nnz - 1, dtype=bool)
            rs = rp[1:-1]
            rs = rs[(rs > 0) & (rs < self.nnz)]
            starts[rs - 1] = True
            if np.any((d <= 0) & ~starts):
                raise ValueError("columns not sorted/unique within a row")


def from_coo(n_rows: int, n_cols: int, rows, cols, vals) -> CSR:
    """Build canonical CSR from COO triplets with unique (row, col) pairs."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    counts = np.bincount(rows, minlength=n_rows)
    rp = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    return CSR(n_rows, n_cols, rp, cols.astype(np.int32), vals)


def transpose(A: CSR) -> CSR:
    """Exact CSR transpose (values copied bit-for-bit)."""
    rows = np.repeat(np.arange(A.n_rows, dtype=np.int64), np.diff(A.row_ptr))
    cols = A.col_idx.astype(np.int64)
    order = np.lexsort((rows, cols))  # by new row (= old col), then new col (= old row)
    counts = np.bincount(cols, minlength=A.n_cols)
    rp = np.zeros(A.n_cols + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    return CSR(A.n_cols, A.n_rows, rp, rows[order].astype(np.int32), A.val[order].copy())


def to_dense(A: CSR) -> np.ndarray:
    M = np.zeros((A.n_rows, A.n_cols), dtype=np.float64)
    rows = np.repeat(np.arange(A.n_rows), np.diff(A.row_ptr))
    M[rows, A.col_idx] = A.val
    return M
