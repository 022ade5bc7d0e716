"""K3 parity: the device GEPP is BIT-EXACT with the reference kernel
(rlra/_lu_cython.pyx:14-55) -- checked against the reference's own golden
digests and, at larger sketch shapes, against the oracle's C restatement."""

import hashlib
import json
import os
import sys

import numpy as np
import pytest

from oracle import rlra_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
META = json.load(open(os.path.join(GOLD, "golden.json")))
GEPP = np.load(os.path.join(GOLD, "gepp.npz"))
sys.path.insert(0, GOLD)
from make_golden_inputs import gepp_input  # noqa: E402

pytestmark = pytest.mark.gpu


def sha_f64(a):
    return hashlib.sha256(np.asfortranarray(a, dtype=np.float64).tobytes(order="F")).hexdigest()


def sha_i64(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def device_lu(a):
    from paper_2002_07138_b200 import ops

    dev = ops.check_device()
    d = ops.from_numpy(a, dev)
    piv, cnt = ops.getrf_(d)
    return ops.to_numpy(d), piv.cpu().numpy(), int(cnt.item())


@pytest.mark.parametrize("name", sorted(META["gepp_cases"]))
def test_device_gepp_bit_exact_vs_reference_golden(cuda_dev, name):
    a = gepp_input(name, GEPP)
    lu, piv, cnt = device_lu(a)
    d = META["gepp_cases"][name]
    assert sha_i64(piv) == d["piv_sha"], "pivot sequence differs from the reference"
    assert sha_f64(lu) == d["lu_sha"], "packed L\\U not bit-identical to the reference"
    r = min(a.shape)
    assert cnt == int(np.count_nonzero(np.diag(lu)[:r]))


@pytest.mark.parametrize("name", ["frozen2x2", "tie", "dupcols", "int_rank5", "rand_300x120_s1"])
def test_host_seam_plu_inplace_bit_exact(cuda_dev, name):
    from paper_2002_07138_b200 import plu_inplace

    a = gepp_input(name, GEPP)
    lu = np.asfortranarray(a, dtype=np.float64).copy(order="F")
    piv = np.arange(a.shape[0], dtype=np.int64)
    plu_inplace(lu, piv)
    d = META["gepp_cases"][name]
    assert sha_f64(lu) == d["lu_sha"] and sha_i64(piv) == d["piv_sha"]


@pytest.mark.parametrize("m,n,seed", [(20000, 220, 0), (10000, 220, 1), (3001, 97, 2),
                                      (16384, 256, 3), (65, 64, 4), (64, 200, 5),
                                      (100000, 70, 6), (200000, 45, 7),
                                      # one-launch cluster GEPP (csrc/getrf_full.cu): edges of its range
                                      (24576, 256, 10), (8193, 33, 11), (2000, 60, 12), (520, 256, 13),
                                      (16385, 200, 14), (8192, 300, 15), (24576, 512, 16),
                                      # r02: widths up to 1024 (C3's 16384 x 1024 / 843 sketches)
                                      (16384, 1024, 17), (12000, 843, 18), (4096, 544, 19), (2000, 1000, 20),
                                      # r02: 16-wide grid panels up to 148 x 1784 rows (223 KB)
                                      (262144, 40, 21), (240000, 36, 22)])
def test_device_gepp_bit_exact_vs_oracle_sketch_shapes(cuda_dev, m, n, seed):
    a = np.random.default_rng(seed).standard_normal((m, n))
    if n > 40:
        a[:, 33] = a[:, 5]  # exact zero pivot across a panel boundary
        a[:, 40] = 0.0
    lu_ref = np.asfortranarray(a).copy(order="F")
    piv_ref = np.arange(m, dtype=np.int64)
    O.plu_inplace(lu_ref, piv_ref)
    lu, piv, _ = device_lu(a)
    assert np.array_equal(piv, piv_ref)
    assert np.array_equal(lu.view(np.int64), lu_ref.view(np.int64))


def test_device_gepp_integer_ties_and_zero_rows(cuda_dev):
    rng = np.random.default_rng(9)
    a = rng.integers(-3, 4, size=(5000, 70)).astype(np.float64)
    a[100:200] = 0.0
    lu_ref = np.asfortranarray(a).copy(order="F")
    piv_ref = np.arange(a.shape[0], dtype=np.int64)
    O.plu_inplace(lu_ref, piv_ref)
    lu, piv, _ = device_lu(a)
    assert np.array_equal(piv, piv_ref)
    assert np.array_equal(lu.view(np.int64), lu_ref.view(np.int64))


def test_device_gepp_empty(cuda_dev):
    from paper_2002_07138_b200 import plu_inplace

    lu = np.zeros((0, 3), order="F")
    piv = np.zeros(0, dtype=np.int64)
    plu_inplace(lu, piv)


@pytest.mark.parametrize("m,n,seed", [(700, 64, 0), (2000, 60, 12), (20000, 220, 0)])
def test_device_gepp_repeatable(cuda_dev, m, n, seed):
    """The one-launch GEPP hands panels between concurrently running clusters;
    a hand-off race shows up as run-to-run differences.  Repeat and require
    every run bit-identical to the oracle."""
    a = np.random.default_rng(seed).standard_normal((m, n))
    lu_ref = np.asfortranarray(a).copy(order="F")
    piv_ref = np.arange(m, dtype=np.int64)
    O.plu_inplace(lu_ref, piv_ref)
    for _ in range(8):
        lu, piv, _ = device_lu(a)
        assert np.array_equal(piv, piv_ref)
        assert np.array_equal(lu.view(np.int64), lu_ref.view(np.int64))
