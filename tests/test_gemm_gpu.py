"""K1/K2/K5 numerics: the FP64 DMMA GEMM against a float64 reference product
(NumPy on the host).  Tolerance: |C - C_ref| <= 4 * K * eps * (|A| |B|)
elementwise (standard FP64 GEMM error bound with any summation order)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

EPS = np.finfo(np.float64).eps


def run(ta, tb, m, n, k, alpha=1.0, beta=0.0, seed=0, odd_ld=False):
    import torch

    from paper_2002_07138_b200 import ops

    dev = ops.check_device()
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((k, m) if ta else (m, k))
    b = rng.standard_normal((n, k) if tb else (k, n))
    c0 = rng.standard_normal((m, n))
    da, db = ops.from_numpy(a, dev), ops.from_numpy(b, dev)
    if odd_ld:  # sub-view with a leading dimension larger than the rows
        big = ops.fmat(m + 3, n, dev)
        dc = big[1:m + 1, :]
        dc.copy_(torch.from_numpy(np.asfortranarray(c0)))
    else:
        dc = ops.from_numpy(c0, dev)
    ops.gemm(da, db, dc, ta=ta, tb=tb, alpha=alpha, beta=beta)
    got = ops.to_numpy(dc)
    opa = a.T if ta else a
    opb = b.T if tb else b
    ref = alpha * (opa @ opb) + beta * c0
    bound = 4 * max(k, 1) * EPS * (np.abs(alpha) * (np.abs(opa) @ np.abs(opb)) + np.abs(beta * c0)) + 1e-300
    assert np.all(np.abs(got - ref) <= bound), float(np.max(np.abs(got - ref) / bound))


@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("m,n,k", [(1000, 220, 700), (257, 61, 333), (33, 544, 1000), (4096, 512, 96),
                                   (10000, 200, 16), (7, 9, 5), (128, 80, 2048), (1024, 61, 700),
                                   (132, 1000, 4), (2000, 544, 3000)])
def test_gemm_matches_fp64_reference(cuda_dev, ta, tb, m, n, k):
    run(ta, tb, m, n, k)


@pytest.mark.parametrize("ta", [False, True])
def test_gemm_alpha_beta_and_subviews(cuda_dev, ta):
    run(ta, False, 300, 112, 500, alpha=-1.5, beta=0.75, odd_ld=True)
    run(ta, True, 301, 113, 501, alpha=2.0, beta=1.0, odd_ld=True)


def test_gemm_k_zero_scales_c(cuda_dev):
    run(False, False, 50, 40, 0, alpha=1.0, beta=0.5)


def test_gemm_split_k_pass_shapes(cuda_dev):
    # the C2 pass shapes scaled down in m: TN with long K, NN with N = 220
    run(True, False, 2500, 220, 20000, seed=3)
    run(False, False, 20000, 220, 2500, seed=4)


def test_gemm_deterministic(cuda_dev):
    import torch

    from paper_2002_07138_b200 import ops

    dev = ops.check_device()
    rng = np.random.default_rng(5)
    a = ops.from_numpy(rng.standard_normal((6000, 1000)), dev)
    w = ops.from_numpy(rng.standard_normal((6000, 220)), dev)
    z1 = ops.matmul(a, w, ta=True)
    z2 = ops.matmul(a, w, ta=True)
    assert torch.equal(z1, z2)
