"""a1 parity: the device Omega generator reproduces the reference's host draw
np.random.default_rng(seed).standard_normal(N) (rlra/core.py:33-48) BIT FOR
BIT, including the rare tail draws and rejection chains."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,count", [(0, 1), (0, 7), (1, 1000), (2, 100003), (3, 4_400_000),
                                        (12345, 20_000_000), (2**40 + 17, 333_333)])
def test_device_gaussian_bit_exact(cuda_dev, seed, count):
    from paper_2002_07138_b200 import core

    got = core.device_gaussian_flat(seed, count, cuda_dev)
    assert got is not None, "device generator unavailable"
    ref = np.random.default_rng(seed).standard_normal(count)
    g = got.cpu().numpy()
    bad = np.nonzero(g.view(np.int64) != ref.view(np.int64))[0]
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:5]}"
    assert np.sum(np.abs(ref) > 3.6541528853610088) >= (1 if count > 100000 else 0)


def test_omega_prefix_property_and_layout(cuda_dev):
    from paper_2002_07138_b200 import core, ops

    a = ops.to_numpy(core.omega(9, 300, 7, cuda_dev))
    b = ops.to_numpy(core.omega(9, 300, 3, cuda_dev))
    assert np.array_equal(a, core.gaussian(9, 300, 7))
    assert np.array_equal(a[:, :3], b)


def test_device_gaussian_chunked_stream_continuation(cuda_dev, monkeypatch):
    """Counts beyond one device pass continue the PCG64 stream exactly."""
    from paper_2002_07138_b200 import core

    monkeypatch.setattr(core, "_CHUNK", 100_000)
    got = core.device_gaussian_flat(77, 350_001, cuda_dev)
    ref = np.random.default_rng(77).standard_normal(350_001)
    assert np.array_equal(got.cpu().numpy().view(np.int64), ref.view(np.int64))
    # continuing a stream mid-way (the C2-C5 noise term recipe)
    rng = np.random.default_rng(3)
    rng.standard_normal(12345)
    st = rng.bit_generator.state["state"]
    got = core.device_gaussian_flat(None, 200_000, cuda_dev, pcg_state=(int(st["state"]), int(st["inc"])))
    assert np.array_equal(got.cpu().numpy(), rng.standard_normal(200_000))
