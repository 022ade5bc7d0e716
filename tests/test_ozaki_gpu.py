"""K1/K2 emulated on the int8 tensor cores (csrc/ozaki.cu, Ozaki scheme II).

Accuracy contract of the raw engine (include/rlra_b200.h; the drivers add the
dynamic-range guard, tests/test_guard_gpu.py): for nmod = 14 the error of every
element is bounded by the scaling step alone,
    |C_ij - (A B)_ij| <= (2^-PA sqrt(K) ||A||_max-norm ||B_j|| + 2^-PB ...)
which we check in its normwise form against an extended-precision reference
(np.longdouble products), with tolerance
    |C - C_ref|_ij <= 2^-50 * N_A * ||B_j||_2,   N_A = max row / column norm of A,
and we also check that the emulation is at least as accurate as NumPy's
float64 DGEMM on the same inputs (max error within 4x of DGEMM's).  Results
are exact functions of the inputs, so repeated calls are bitwise identical.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ref(opa, b):
    return opa.astype(np.longdouble) @ b.astype(np.longdouble)


def run(m, n, l, trans, seed=0, scale_rows=False, nmod=14):
    from paper_2002_07138_b200 import ops

    dev = ops.check_device()
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, n))
    if scale_rows:
        a *= np.exp(rng.uniform(-3, 3, size=(m, 1)))
        a *= np.exp(rng.uniform(-3, 3, size=(1, n)))
    k = m if trans else n
    b = rng.standard_normal((k, l)) * np.exp(rng.uniform(-5, 5, size=(1, l)))
    prep = ops.OzPrep(ops.from_numpy(a, dev), nmod, guard=not scale_rows)
    c = ops.to_numpy(prep.gemm(ops.from_numpy(b, dev), trans=trans))
    opa = a.T if trans else a
    ref = _ref(opa, b)
    na = max(np.sqrt((a * a).sum(0)).max(), np.sqrt((a * a).sum(1)).max())
    nb = np.sqrt((b * b).sum(0))
    err = np.abs(c - ref).astype(np.float64)
    tol = 2.0 ** -50 * na * nb[None, :]
    assert np.all(err <= tol), float((err / tol).max())
    err_np = np.abs(opa @ b - ref).astype(np.float64)
    return c, float((err / nb).max()), float((err_np / nb).max())


@pytest.mark.parametrize("trans", [False, True])
@pytest.mark.parametrize("m,n,l", [(700, 500, 100), (1000, 1000, 220), (257, 129, 33), (130, 300, 1),
                                   (384, 256, 300), (2000, 1500, 544), (129, 127, 32)])
def test_oz_gemm_accuracy(cuda_dev, m, n, l, trans):
    _, e_oz, e_np = run(m, n, l, trans)
    assert e_oz <= 4 * e_np + 1e-300, (e_oz, e_np)


@pytest.mark.parametrize("trans", [False, True])
def test_oz_gemm_badly_scaled_rows_and_columns(cuda_dev, trans):
    run(600, 400, 64, trans, seed=3, scale_rows=True)


def test_oz_gemm_deterministic_and_zero_columns(cuda_dev):
    from paper_2002_07138_b200 import ops

    rng = np.random.default_rng(5)
    a = rng.standard_normal((500, 300))
    b = rng.standard_normal((300, 40))
    b[:, 7] = 0.0
    ad = ops.from_numpy(a, cuda_dev)
    prep = ops.OzPrep(ad)
    c1 = ops.to_numpy(prep.gemm(ops.from_numpy(b, cuda_dev)))
    c2 = ops.to_numpy(ops.OzPrep(ad).gemm(ops.from_numpy(b, cuda_dev)))
    assert np.array_equal(c1, c2)
    assert np.all(c1[:, 7] == 0.0)
    z = ops.OzPrep(ops.from_numpy(np.zeros((200, 100)), cuda_dev))
    assert np.all(ops.to_numpy(z.gemm(ops.from_numpy(b[:100], cuda_dev))) == 0.0)


@pytest.mark.parametrize("nmod", [12, 13, 15, 16])
def test_oz_gemm_other_moduli_counts(cuda_dev, nmod):
    from paper_2002_07138_b200 import ops

    rng = np.random.default_rng(nmod)
    a = rng.standard_normal((400, 300))
    b = rng.standard_normal((300, 50))
    c = ops.to_numpy(ops.OzPrep(ops.from_numpy(a, cuda_dev), nmod).gemm(ops.from_numpy(b, cuda_dev)))
    ref = _ref(a, b)
    rel = float(np.abs(c - ref).max() / np.abs(ref).max())
    # each modulus is ~7.8 bits of product budget, split between A and B
    assert rel < max(2.0 ** (-(3.9 * nmod - 8)), 2.0 ** -50), rel


@pytest.mark.parametrize("trans", [False, True])
@pytest.mark.parametrize("cache_frac", [0.0, 0.5, 1.0])
def test_oz_blocked_bit_identical_to_one_block(cuda_dev, trans, cache_frac):
    """Block-wise residues (ops.OzBlocked: one global eA, one eB of the whole
    B, exact modular accumulation over the K blocks) reproduce the one-block
    product bit for bit -- with every block cached, none, or half of them."""
    import torch

    from paper_2002_07138_b200 import ops

    dev = ops.check_device()
    rng = np.random.default_rng(5)
    m, n, l = 3000, 2600, 37
    a = rng.standard_normal((m, n)) * np.exp(rng.uniform(-4, 4, size=(m, 1)))
    b = rng.standard_normal((m if trans else n, l)) * np.exp(rng.uniform(-3, 3, size=(1, l)))
    ad, bd = ops.from_numpy(a, dev), ops.from_numpy(b, dev)
    c_full = ops.OzPrep(ad, guard=False).gemm(bd, trans=trans)
    total = 14 * m * n * 2
    blk = ops.OzBlocked(ad, block_bytes=14 * 1024 * 1024, col_cap=1000, cache_bytes=int(cache_frac * total),
                        guard=False)
    assert len(blk.rows) == 3 and len(blk.cols) == 3
    assert (blk.rebuilt == 0) == (cache_frac == 1.0)
    for _ in range(2):  # rebuilt blocks reuse the scratch workspace
        c_blk = blk.gemm(bd, trans=trans)
        assert torch.equal(c_full.view(torch.int64), c_blk.view(torch.int64))


@pytest.mark.parametrize("trans", [False, True])
@pytest.mark.parametrize("nmod", [14, 16])
def test_oz_gemm_exact_on_integer_operands(cuda_dev, trans, nmod):
    """Integer A (|a| < 2^20) and B (|b| < 2^18) with K = 1500: every product
    sum is an integer below 2^53, the scalings are exact powers of two, so the
    emulated product must equal the exact integer product bit for bit -- every
    residue plane, the fp32 epilogue reduction and the CRT are exercised with
    accumulators spread over the whole int32 range (raw engine, guard off)."""
    from paper_2002_07138_b200 import ops

    dev = ops.check_device()
    rng = np.random.default_rng(11)
    m, n, l = (1500, 520, 70) if trans else (520, 1500, 70)
    a = rng.integers(-(2 ** 20) + 1, 2 ** 20, size=(m, n)).astype(np.float64)
    k = m if trans else n
    b = rng.integers(-(2 ** 18) + 1, 2 ** 18, size=(k, l)).astype(np.float64)
    b[:, 3] = 0.0
    b[:, 5] = 2 ** 17  # constant column: every partial sum has one sign pattern per row
    opa = a.T if trans else a
    exact = opa.astype(np.int64) @ b.astype(np.int64)
    assert np.abs(exact).max() < 2 ** 53
    prep = ops.OzPrep(ops.from_numpy(a, dev), nmod, guard=False)
    c = ops.to_numpy(prep.gemm(ops.from_numpy(b, dev), trans=trans))
    assert np.array_equal(c, exact.astype(np.float64))


@pytest.mark.parametrize("trans", [False, True])
def test_oz_gemm_fused_column_energies(cuda_dev, trans):
    """RLRA_B200_OZ_COLSQ: the column energies reduced inside the CRT step
    (rlra/fixedprec.py:71-80 without a second read of G) equal the compensated
    K8 reduction over the product to 4 ulp, the product itself is unchanged
    bit for bit, repeated calls are bitwise identical, and a block-wise product
    (several output row blocks, K split) accumulates the same energies."""
    import torch

    from paper_2002_07138_b200 import ops

    dev = ops.check_device()
    rng = np.random.default_rng(3)
    m, n, l = 3100, 2300, 45
    a = rng.standard_normal((m, n))
    b = rng.standard_normal((m if trans else n, l)) * np.exp(rng.uniform(-6, 6, size=(1, l)))
    ad, bd = ops.from_numpy(a, dev), ops.from_numpy(b, dev)
    prep = ops.OzPrep(ad, guard=False)
    c0 = prep.gemm(bd, trans=trans)
    c1, e1 = prep.gemm(bd, trans=trans, colsq=True)
    c2, e2 = prep.gemm(bd, trans=trans, colsq=True)
    assert torch.equal(c0.view(torch.int64), c1.view(torch.int64))
    assert torch.equal(e1.view(torch.int64), e2.view(torch.int64))
    ref = ops.colsumsq(c0).cpu().numpy()
    exact = (ops.to_numpy(c0).astype(np.longdouble) ** 2).sum(axis=0).astype(np.float64)
    got = e1.cpu().numpy()
    assert np.all(np.abs(got - exact) <= 4 * np.spacing(exact))
    assert np.all(np.abs(got - ref) <= 4 * np.spacing(exact))
    blk = ops.OzBlocked(ad, block_bytes=14 * 1024 * 1024, col_cap=1000, cache_bytes=0, guard=False)
    assert len(blk.rows) >= 2 and len(blk.cols) >= 2
    cb, eb = blk.gemm(bd, trans=trans, colsq=True)
    assert torch.equal(cb.view(torch.int64), c0.view(torch.int64))
    assert np.all(np.abs(eb.cpu().numpy() - exact) <= 4 * np.spacing(exact))
    # out += A B: the energies are those of the updated C
    out = c0.clone()
    c3, e3 = prep.gemm(bd, trans=trans, out=out, add=True, colsq=True)
    exact3 = (ops.to_numpy(c3).astype(np.longdouble) ** 2).sum(axis=0).astype(np.float64)
    assert np.all(np.abs(e3.cpu().numpy() - exact3) <= 4 * np.spacing(exact3))
    # a NaN column of B: NaN energy there, the others untouched
    b2 = b.copy()
    b2[5, 7] = np.nan
    _, e4 = prep.gemm(ops.from_numpy(b2, dev), trans=trans, colsq=True)
    e4 = e4.cpu().numpy()
    assert np.isnan(e4[7]) and np.array_equal(np.delete(e4, 7), np.delete(got, 7))


def test_device_matrix_matmul_with_energies(cuda_dev):
    """The accessor seam used by powerlu_fp: fused inside a product session,
    K8 reduction otherwise; both agree with the energies of the product."""
    import paper_2002_07138_b200 as P
    from paper_2002_07138_b200 import ops
    from paper_2002_07138_b200.device import InstrumentedAccessor, product_session

    rng = np.random.default_rng(8)
    a = rng.standard_normal((900, 700))
    v = rng.standard_normal((700, 33))
    dm = P.DeviceMatrix(a)
    acc = InstrumentedAccessor(dm)
    with product_session(dm):
        g, e = acc.matmul_with_energies(v)
    assert acc.product_count == 1
    gn = ops.to_numpy(g)
    exact = (gn.astype(np.longdouble) ** 2).sum(axis=0).astype(np.float64)
    assert np.all(np.abs(e.cpu().numpy() - exact) <= 4 * np.spacing(exact))
    assert np.allclose(gn, a @ v, rtol=0, atol=1e-10)


def test_oz_gemm_reuses_the_skinny_operands_residues(cuda_dev):
    """RLRA_B200_OZ_REUSE_B (the single-pass sweep: every panel^T times the same
    Omega): a product that reuses the previous product's workspace -- scales
    and residues of b included -- equals the fresh product bit for bit."""
    import torch

    from paper_2002_07138_b200 import ops

    dev = ops.check_device()
    rng = np.random.default_rng(21)
    m, n, l = 2100, 768, 90
    b = ops.from_numpy(rng.standard_normal((m, l)) * np.exp(rng.uniform(-4, 4, size=(1, l))), dev)
    a1 = ops.from_numpy(rng.standard_normal((m, n)), dev)
    a2 = ops.from_numpy(rng.standard_normal((m, n)) * 3.0, dev)
    p1, p2 = ops.OzPrep(a1, guard=False), ops.OzPrep(a2, guard=False)
    _, ws = p1.gemm(b, trans=True, keep_ws=True)
    fresh = p2.gemm(b, trans=True)
    reused, ws2 = p2.gemm(b, trans=True, keep_ws=True, b_ws=ws)
    assert ws2 is ws
    assert torch.equal(fresh.view(torch.int64), reused.view(torch.int64))
    # a prep of another shape ignores the offered workspace
    p3 = ops.OzPrep(ops.from_numpy(rng.standard_normal((m, 512)), dev), guard=False)
    c3, ws3 = p3.gemm(b, trans=True, keep_ws=True, b_ws=ws)
    assert ws3 is not ws
    assert torch.equal(c3.view(torch.int64), p3.gemm(b, trans=True).view(torch.int64))


def test_tall_times_small_factor_products(cuda_dev, monkeypatch):
    """ops.tall_prep / tall_times (L = L1 U2^T, V U1^T, Q X): the int8 path,
    forced at a small size, agrees with the float64 product to DGEMM accuracy
    for s and s^T; small products and guard-rejected operands (integer-valued
    tall factor) take the DMMA GEMM and equal ops.matmul bit for bit."""
    import torch

    from paper_2002_07138_b200 import ops

    dev = ops.check_device()
    rng = np.random.default_rng(17)
    q, _ = np.linalg.qr(rng.standard_normal((3000, 90)))
    u = np.triu(rng.standard_normal((90, 90))) * np.exp(-np.arange(90) / 9.0)[:, None]  # graded rows, like U of a sketch
    qd, ud = ops.from_numpy(q, dev), ops.from_numpy(u, dev)
    assert ops.tall_prep(qd, 90) is None  # far below the work threshold: DMMA
    monkeypatch.setattr(ops, "FACTOR_OZ_MIN_WORK", 0.0)
    prep = ops.tall_prep(qd, 90)
    assert prep is not None and prep.ok is None  # lazy guard: not read yet
    got_t = ops.to_numpy(ops.tall_times(qd, ud, prep, ts=True))
    assert prep.ok == (True, True)
    got = ops.to_numpy(ops.tall_times(qd, ud, prep))
    for g, ref in ((got_t, q @ u.T), (got, q @ u)):
        bound = 1e-15 * np.sqrt(90) * np.linalg.norm(q, axis=1)[:, None] * np.linalg.norm(ref, axis=0)[None, :] + 1e-300
        assert np.all(np.abs(g - ref) <= 8 * bound + 1e-18)
    # integer-valued tall operand: the guard sends it to the FP64 GEMM
    li = ops.from_numpy(rng.integers(-3, 4, size=(3000, 90)).astype(np.float64), dev)
    pi = ops.tall_prep(li, 90)
    c = ops.tall_times(li, ud, pi, ts=True)
    assert pi.ok[0] is False
    assert torch.equal(c.view(torch.int64), ops.matmul(li, ud, tb=True).view(torch.int64))
