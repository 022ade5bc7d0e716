"""K4 numerics: device Householder QR + explicit Q against LAPACK
(np.linalg.qr, what the reference calls at rlra/kernels.py:60).  Same sign
convention, so Q matches entrywise to ~cond * eps; orthogonality to 1e-13."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def dev_qr(x):
    from paper_2002_07138_b200 import ops

    dev = ops.check_device()
    d = ops.from_numpy(x, dev)
    qr = ops.QR(d)
    q = ops.to_numpy(qr.q())
    r = np.triu(ops.to_numpy(qr.r_view()))
    cnt = int(ops.count_nonzero_diag(qr.r_view()).item())
    return q, r, cnt


@pytest.mark.parametrize("m,n", [(30, 8), (2000, 60), (10000, 220), (3000, 97), (512, 512), (33, 33),
                                 (50000, 72), (120000, 40), (160000, 20)])
def test_qr_matches_lapack(cuda_dev, m, n):
    x = np.random.default_rng(m + n).standard_normal((m, n))
    q, r, cnt = dev_qr(x)
    q_ref, r_ref = np.linalg.qr(x)
    assert cnt == n
    assert np.allclose(q.T @ q, np.eye(n), atol=1e-13)
    assert np.allclose(q @ r, x, atol=1e-12 * np.linalg.norm(x))
    np.testing.assert_allclose(np.diag(r), np.diag(r_ref), rtol=1e-11)
    np.testing.assert_allclose(q, q_ref, rtol=0, atol=1e-11)


def test_qr_exact_zero_diagonal_on_structural_deficiency(cuda_dev):
    # rows 3..7 of A^T Omega vanish exactly (pkg/tests/test_rangefinder.py:102-107)
    a = np.diag([1.0, 1.0, 1.0, 0, 0, 0, 0, 0])
    om = np.random.default_rng(0).standard_normal((8, 5))
    x = a.T @ om
    _, r, cnt = dev_qr(x)
    r_ref = np.linalg.qr(x)[1]
    assert cnt == int(np.count_nonzero(np.diag(r_ref))) == 3


def test_qr_ill_conditioned_orthogonality(cuda_dev):
    rng = np.random.default_rng(1)
    u, _ = np.linalg.qr(rng.standard_normal((5000, 300)))
    v, _ = np.linalg.qr(rng.standard_normal((300, 300)))
    x = (u * np.logspace(0, -9, 300)) @ v.T
    q, r, _ = dev_qr(x)
    assert np.abs(q.T @ q - np.eye(300)).max() < 1e-13
    assert np.allclose(q @ r, x, atol=1e-13 * np.linalg.norm(x))


# ---- K4 fast path: CholeskyQR2 (csrc/cholqr.cu), used for powerlu's internal basis
@pytest.mark.parametrize("n,l", [(10000, 220), (3000, 64), (500, 200), (64, 1), (2000, 230)])
def test_cholqr2_spans_the_householder_range(cuda_dev, n, l):
    from paper_2002_07138_b200 import ops

    rng = np.random.default_rng(l)
    # graded columns (cond ~ 1e4), like powerlu's final sketch
    x = rng.standard_normal((n, l)) * np.logspace(0, -4, l)[None, :]
    q, flag = ops.cholqr2(ops.from_numpy(x, cuda_dev))
    assert int(flag.item()) == 0
    q = ops.to_numpy(q)
    assert np.abs(q.T @ q - np.eye(l)).max() < 1e-13
    q_ref, _ = np.linalg.qr(x)
    d = np.sign(np.sum(q * q_ref, axis=0))  # column signs may differ from LAPACK's
    assert np.all(np.abs(d) == 1)
    assert np.abs(q - q_ref * d[None, :]).max() < 1e-10


def test_cholqr2_flags_rank_collapse_and_ill_conditioning(cuda_dev):
    from paper_2002_07138_b200 import ops

    rng = np.random.default_rng(3)
    x = rng.standard_normal((400, 30))
    x[:, 7] = x[:, 3]  # exactly dependent column
    _, flag = ops.cholqr2(ops.from_numpy(x, cuda_dev))
    assert int(flag.item()) == 1
    y = rng.standard_normal((400, 30)) * np.logspace(0, -12, 30)[None, :]
    _, flag = ops.cholqr2(ops.from_numpy(y, cuda_dev))
    assert int(flag.item()) == 1


@pytest.mark.parametrize("l", [1, 2, 15, 16, 17, 31, 32, 33, 47, 100, 129, 220, -1])
def test_chol_inv_block_edges(cuda_dev, l):
    """chol_kernel's 16-column blocks, the 4-warp next-block update and the
    4 x 8 super-tiles of the trailing update at every ragged edge (l = -1: the
    largest l the shared-memory layout takes)."""
    import torch

    from paper_2002_07138_b200 import ops

    l = ops.cholqr_max_l() if l < 0 else l
    rng = np.random.default_rng(100 + l)
    z = rng.standard_normal((3 * l + 5, l)) * np.logspace(0, -3, l)[None, :]
    g = z.T @ z
    out = ops.fmat(l, l, cuda_dev)
    flag = torch.zeros(1, dtype=torch.int32, device=cuda_dev)
    ops.chol_inv(ops.from_numpy(g, cuda_dev), out, flag, 1e8)
    assert int(flag.item()) == 0
    rinv = ops.to_numpy(out)
    assert np.all(np.tril(rinv, -1) == 0)
    # R^{-T} G R^{-1} = I to working precision (cond(G) ~ 1e6 here)
    assert np.abs(rinv.T @ g @ rinv - np.eye(l)).max() < 1e-9


def test_chol_inv_matches_numpy(cuda_dev):
    import torch

    from paper_2002_07138_b200 import ops

    rng = np.random.default_rng(9)
    z = rng.standard_normal((600, 150))
    g = z.T @ z
    out = ops.fmat(150, 150, cuda_dev)
    flag = torch.zeros(1, dtype=torch.int32, device=cuda_dev)
    ops.chol_inv(ops.from_numpy(g, cuda_dev), out, flag, 1e8)
    r = np.linalg.cholesky(g).T
    np.testing.assert_allclose(ops.to_numpy(out), np.linalg.inv(r), rtol=0, atol=1e-12 * np.abs(np.linalg.inv(r)).max())
    assert int(flag.item()) == 0


@pytest.mark.parametrize("l", [300, 544, 1024])
def test_blocked_cholesky_inverse(cuda_dev, l):
    """ops.chol_inv_blocked: diagonal blocks by the one-CTA kernel, panels and
    trailing updates on the DMMA GEMM, R^{-1} assembled by blocks."""
    import torch

    from paper_2002_07138_b200 import ops

    rng = np.random.default_rng(l)
    x = rng.standard_normal((3 * l, l)) * np.exp(rng.uniform(-3, 3, size=(1, l)))
    g = x.T @ x
    r_ref = np.linalg.cholesky(g).T
    gd = ops.from_numpy(g, cuda_dev)
    out = ops.fmat(l, l, cuda_dev)
    flag = torch.zeros(1, dtype=torch.int32, device=cuda_dev)
    ops.chol_inv_blocked(gd, out, flag, 1e30)
    rinv = ops.to_numpy(out)
    assert int(flag.item()) == 0
    assert np.allclose(np.tril(rinv, -1), 0.0)
    assert np.abs(r_ref @ rinv - np.eye(l)).max() <= 1e-9
    # the condition bound across blocks
    flag.zero_()
    ops.chol_inv_blocked(ops.from_numpy(g, cuda_dev), out, flag, 2.0)
    assert int(flag.item()) == 1


@pytest.mark.parametrize("n,l,cond", [(4000, 300, 1e3), (6000, 544, 1e10), (9000, 1024, 1e11)])
def test_shifted_cholesky_qr3(cuda_dev, n, l, cond):
    """ops.scholqr3: orthonormal to working precision and spanning range(Z) for
    cond(Z) far beyond CholeskyQR2's ~u^-1/2 (C5's final sketch: ~1e9)."""
    from paper_2002_07138_b200 import ops

    rng = np.random.default_rng(int(cond) % 1000 + l)
    u, _ = np.linalg.qr(rng.standard_normal((n, l)))
    w, _ = np.linalg.qr(rng.standard_normal((l, l)))
    z = (u * np.logspace(0, -np.log10(cond), l)) @ w.T
    q, flag = ops.scholqr3(ops.from_numpy(z, cuda_dev))
    assert int(flag.item()) == 0
    qh = ops.to_numpy(q)
    assert np.abs(qh.T @ qh - np.eye(l)).max() <= 1e-13
    assert np.linalg.norm(z - qh @ (qh.T @ z)) <= 1e-13 * np.linalg.norm(z)


def test_cholesky_qr_declines_structural_collapse(cuda_dev):
    """An exactly zero column (Householder's exact zero R_ii, rlra/rangefinder.py
    :55-64) and cond beyond ~u^-1/2 with a harmless diagonal ratio both raise
    the decline flag, so the driver redoes the basis by Householder."""
    from paper_2002_07138_b200 import ops

    rng = np.random.default_rng(3)
    z = rng.standard_normal((3000, 400))
    z[:, 17] = 0.0
    _, flag = ops.scholqr3(ops.from_numpy(z, cuda_dev))
    assert int(flag.item()) == 1
    # ill-conditioned but equal column norms: R diag ratio stays small, the Gram identity check catches it
    u, _ = np.linalg.qr(rng.standard_normal((3000, 100)))
    w, _ = np.linalg.qr(rng.standard_normal((100, 100)))
    zz = (u * np.logspace(0, -12, 100)) @ w.T
    zz /= np.linalg.norm(zz, axis=0)
    _, flag = ops.cholqr2(ops.from_numpy(zz, cuda_dev))
    assert int(flag.item()) == 1
