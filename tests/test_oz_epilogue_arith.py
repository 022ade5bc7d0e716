"""The pass GEMM's epilogue arithmetic (csrc/ozaki.cu gemm_i8_kernel, warps 2-5):
t = (c y) mod m from an int32 accumulator c on the fp32 pipes.  This CPU check
restates each step in exact integer / IEEE float32 arithmetic and verifies it
for every modulus, over the whole range of the intermediate s and over random
and extreme accumulators (no GPU needed; the GPU tests check the kernel itself)."""

import numpy as np
import pytest

MODULI = [249, 247, 245, 244, 241, 239, 233, 229, 227, 223, 211, 199, 197, 193, 191, 181]
BIG = np.float32(12582912.0)  # 1.5 * 2^23


def centred(x, m):
    x %= m
    return x - m if 2 * x > m else x


def rint_magic(s, inv32):
    """fma(s, inv, BIG) - BIG in float32: the fma rounds the EXACT s*inv + BIG
    to the float32 grid (spacing 1 in [2^23, 2^24)), ties to even."""
    mant, exp = np.frexp(np.float64(inv32))  # inv = k * 2^e exactly, k a 24-bit integer
    k = np.int64(round(float(mant) * 2 ** 24))
    sh = 24 - int(exp)  # inv = k / 2^sh
    num = s.astype(np.int64) * k  # exact: |s| < 2^24, k < 2^24
    half = np.int64(1) << (sh - 1)
    fl = num >> sh  # floor
    rem = num - (fl << sh)
    q = fl + ((rem > half) | ((rem == half) & ((fl & 1) == 1)))
    return q


@pytest.mark.parametrize("m", MODULI)
def test_reduction_step_is_exact_for_every_s(m):
    inv32 = np.float32(1.0) / np.float32(m)
    bound = 124 * (2 ** 15 + 2 ** 16)
    assert bound < 2 ** 24
    s = np.arange(-bound, bound + 1, dtype=np.int64)
    q = rint_magic(s, inv32)
    r = s - q * m
    assert np.abs(r).max() <= 125 < m  # one fix-up suffices
    t = np.where(r < 0, r + m, r)
    assert np.array_equal(t, s % m)
    # the byte: low 8 bits of the float32 (2^23 + t)
    bits = (np.float32(8388608.0) + t.astype(np.float32)).view(np.uint32)
    assert np.array_equal(bits & 0xFF, t.astype(np.uint32))


@pytest.mark.parametrize("m", MODULI)
def test_split_reproduces_c_times_y_mod_m(m):
    rng = np.random.default_rng(m)
    c = np.concatenate([rng.integers(-(2 ** 31) + 1, 2 ** 31, size=200000, dtype=np.int64),
                        np.array([0, 1, -1, 65535, 65536, -65536, 2 ** 31 - 1, -(2 ** 31) + 1,
                                  127 * 127 * 133144, -127 * 127 * 133144], dtype=np.int64)])
    for y in (1, m - 1, m // 2, m // 2 + 1, int(rng.integers(1, m))):
        k1, yc = centred(65536 * y, m), centred(y, m)
        assert abs(k1) <= 124 and abs(yc) <= 124
        lo, hi = c & 0xFFFF, c >> 16  # arithmetic shift: c = hi 2^16 + lo
        assert np.array_equal(hi * 65536 + lo, c)
        # float32 images of lo / hi through the magic constants
        lof = (np.uint32(0x4B000000) | lo.astype(np.uint32)).view(np.float32) - np.float32(8388608.0)
        hif = (np.uint32(0x4B400000) + hi.astype(np.int32).view(np.uint32)).view(np.float32) - BIG
        assert np.array_equal(lof.astype(np.int64), lo) and np.array_equal(hif.astype(np.int64), hi)
        s = hi * k1 + lo * yc
        assert np.abs(s).max() < 2 ** 24
        # float32 evaluation of s is exact (every partial result an integer < 2^24)
        s32 = hif * np.float32(k1) + lof * np.float32(yc)
        assert np.array_equal(s32.astype(np.int64), s)
        q = rint_magic(s, np.float32(1.0) / np.float32(m))
        r = s - q * m
        t = np.where(r < 0, r + m, r)
        assert np.array_equal(t, (c * y) % m)
        # accumulate mode: (t_prev + t) mod m from r + prev in (-m, 2m)
        prev = rng.integers(0, m, size=c.shape)
        z = r + prev
        z = np.where(z < 0, z + m, z)
        z = np.where(z >= m, z - m, z)
        assert np.array_equal(z, (c * y + prev) % m)
