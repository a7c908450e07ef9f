"""Conversions between the oracle's Csr and the product's CsrMatrix."""
import numpy as np


def to_product(c):
    from paper_2106_12836_b200 import CsrMatrix

    return CsrMatrix(c.nrows, c.ncols, c.row_ptr, c.col_idx, c.values)


def to_oracle(m):
    from oracle.oracle import Csr

    return Csr(m.nrows, m.ncols, m.row_ptr, m.col_idx, m.values)


def bitwise_equal_csr(a, b):
    """a, b: objects with nrows/ncols/row_ptr/col_idx/values (either type)."""
    if (a.nrows, a.ncols) != (b.nrows, b.ncols):
        return False
    if not np.array_equal(a.row_ptr, b.row_ptr) or not np.array_equal(a.col_idx, b.col_idx):
        return False
    if a.values is None or b.values is None:
        return a.values is None and b.values is None
    return np.array_equal(np.asarray(a.values).view(np.uint64), np.asarray(b.values).view(np.uint64))


def bitwise_equal(x, y):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return x.shape == y.shape and np.array_equal(x.view(np.uint64), y.view(np.uint64))
