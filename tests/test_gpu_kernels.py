"""GPU parity of the kernels.hpp primitives against the oracle port (bitwise)."""
import numpy as np
import pytest

from helpers import bitwise_equal, bitwise_equal_csr, to_oracle, to_product

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2106_12836_b200 as S

    return S


def rand_csr(S, n, m, density, seed):
    import scipy.sparse as sp

    a = sp.random(n, m, density=density, random_state=seed, format="csr")
    a.sort_indices()
    a.data = np.random.default_rng(seed).standard_normal(a.nnz)
    return S.CsrMatrix.from_scipy(a)


@pytest.mark.parametrize("n,m,k,d", [(50, 40, 30, 0.1), (300, 200, 250, 0.05), (64, 64, 64, 0.5), (1, 1, 1, 1.0)])
def test_spgemm(S, port, n, m, k, d):
    a = rand_csr(S, n, k, d, 1)
    b = rand_csr(S, k, m, d, 2)
    got = S.spgemm(a, b)
    assert bitwise_equal_csr(got, port.spgemm(to_oracle(a), to_oracle(b)))


def test_spgemm_dim_error(S):
    a = rand_csr(S, 5, 4, 0.5, 1)
    with pytest.raises(S.SaitInvalidArgument, match="spgemm: inner dimensions 4 and 5 do not match"):
        S.spgemm(a, a)


def test_add_identity_and_drops(S, port):
    a = rand_csr(S, 120, 120, 0.08, 3)
    # force a diagonal that cancels to exactly 0.0 after +1
    a.values[a.row_ptr[0]] = a.values[a.row_ptr[0]]
    oa = to_oracle(a)
    assert bitwise_equal_csr(S.add_identity(a), port.add_identity(oa))
    for tau in (0.0, 0.3, 0.9):
        assert bitwise_equal_csr(S.drop_by_threshold(a, tau), port.drop_by_threshold(oa, tau))
    s = rand_csr(S, 120, 120, 0.1, 4).pattern()
    assert bitwise_equal_csr(S.drop_by_pattern(a, s), port.drop_by_pattern(oa, to_oracle(s)))
    with pytest.raises(S.SaitInvalidArgument, match=r"drop_by_threshold: tau must be in \[0, 1\), got 1.000000"):
        S.drop_by_threshold(a, 1.0)
    with pytest.raises(S.SaitInvalidArgument, match="add_identity: matrix is not square"):
        S.add_identity(rand_csr(S, 3, 4, 0.5, 1))


def test_transpose_scale(S, port):
    a = rand_csr(S, 333, 777, 0.03, 5)
    assert bitwise_equal_csr(S.transpose(a), port.transpose(to_oracle(a)))
    d = np.random.default_rng(1).standard_normal(777)
    assert bitwise_equal_csr(S.scale_columns(a, d), port.scale_columns(to_oracle(a), d))


@pytest.mark.parametrize("shape", [(500, 300, 0.06, 6), (200, 400, 0.2, 7), (3000, 3000, 0.004, 8)])
def test_transpose_row_length_paths(S, port, shape):
    """Every scatter/sort variant of the transpose: short stencil-like rows
    (thread per row, 8-lane sorter), rows averaging >= 12 entries (8 lanes per
    source row, 16-lane first sorter), half-warp and full-warp mid rows, and
    rows over 32 entries (block sorter) -- bitwise the reference."""
    m, n, dens, seed = shape
    a = rand_csr(S, m, n, dens, seed)
    assert bitwise_equal_csr(S.transpose(a), port.transpose(to_oracle(a)))
    d = np.random.default_rng(seed).standard_normal(n)
    assert bitwise_equal_csr(S.scale_columns(a, d), port.scale_columns(to_oracle(a), d))


def test_spmv_random(S, port):
    a = rand_csr(S, 2000, 1500, 0.004, 9)
    x = np.random.default_rng(2).standard_normal(1500)
    assert bitwise_equal(S.spmv(a, x), port.spmv(to_oracle(a), x))


def test_upload_validation(S):
    bad = S.CsrMatrix(2, 2, [0, 2, 3], [1, 0, 1], [1.0, 1.0, 1.0])
    with pytest.raises(S.SaitInvalidArgument, match="validate: columns not strictly increasing in row 0"):
        S.DeviceCsr.upload(bad)
    bad = S.CsrMatrix(2, 2, [0, 1, 2], [0, 2], [1.0, 1.0])
    with pytest.raises(S.SaitInvalidArgument, match="validate: column out of range in row 1"):
        S.DeviceCsr.upload(bad)
