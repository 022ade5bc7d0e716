"""Sparse operands on device (SparseAccessor, rlra/accessors.py:40-64;
SURVEY.md §8(f) row 4): CSR SpMM products for A X and A^T X, never densified,
and the drivers on scipy.sparse input against the oracle on the same matrix."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import rlra_oracle as O

pytestmark = pytest.mark.gpu


def sample_sparse(m=30, n=20, density=0.2, seed=0):
    """pkg/tests/test_accessors.py:14-17 (shape / density / seed)."""
    rng = np.random.default_rng(seed)
    return sp.random(m, n, density=density, format="csc", dtype=np.float64, random_state=rng)


def test_sparse_products_match_dense(cuda_dev):
    """pkg/tests/test_accessors.py:32-41."""
    import paper_2002_07138_b200 as P
    from paper_2002_07138_b200 import ops

    a = sample_sparse()
    acc = P.as_accessor(a)
    assert isinstance(acc, P.SparseDeviceMatrix) and acc.shape == (30, 20)
    dense = acc.to_dense()
    x = O.gaussian(4, 20, 3)
    y = O.gaussian(5, 30, 3)
    assert np.allclose(ops.to_numpy(acc.matmul(x)), dense @ x, atol=1e-14)
    assert np.allclose(ops.to_numpy(acc.rmatmul(y)), dense.T @ y, atol=1e-14)
    assert abs(acc.fro_norm() - float(np.sqrt((a.data ** 2).sum()))) <= 1e-15 * acc.fro_norm()
    # empty rows / columns and an all-zero matrix
    z = sp.csc_matrix((7, 5))
    zacc = P.as_accessor(z)
    assert np.array_equal(ops.to_numpy(zacc.matmul(np.ones((5, 2)))), np.zeros((7, 2)))
    assert zacc.fro_norm() == 0.0


def lowrank_sparse(m, n, seed, scale=15.0):
    """Sparse with a decaying spectrum: a sparse random matrix times a diagonal
    decay on its columns."""
    s = sample_sparse(m, n, 0.05, seed).tocsc()
    return s @ sp.diags(np.exp(-np.arange(n) / scale))


@pytest.mark.parametrize("v", [2, 3, 4])
def test_powerlu_on_sparse_matches_oracle(cuda_dev, v):
    import paper_2002_07138_b200 as P

    a = lowrank_sparse(600, 400, seed=v)
    acc = P.InstrumentedAccessor(a)
    f = P.powerlu(acc, 20, q_os=10, v=v, seed=1)
    assert acc.product_count == v
    f = f.to_numpy() if f.on_device else f
    dense = a.toarray()
    g = O.powerlu(dense, 20, 10, v, 1)
    assert np.array_equal(f.p, g.p) and np.array_equal(f.q, g.q)
    assert abs(O.rel_fro_error_factor(dense, f) - O.rel_fro_error_factor(dense, g)) <= 1e-10


def test_powerlu_fp_on_sparse_matches_oracle(cuda_dev):
    import paper_2002_07138_b200 as P

    a = lowrank_sparse(500, 300, seed=9, scale=4.0)
    fac, out = P.powerlu_fp(a, P.PrecisionParams(1e-3, 5, 60, 4), seed=0)
    dense = a.toarray()
    gf, go = O.powerlu_fp(dense, 1e-3, 5, 60, 4, 0)
    assert out.rank == go.rank
    assert np.array_equal(fac.p, gf.p) and np.array_equal(fac.q, gf.q)
