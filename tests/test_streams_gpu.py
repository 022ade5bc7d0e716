"""Out-of-core single pass: RlraFileColumnStream and
the host DenseColumnStream feed HBM through the pinned, multi-slot pipeline
(paper_2002_07138_b200/streams.py).  Parity: identical pivots and the
reference's error on its own single-pass case, and bit-identical sketches to
the HBM-resident DeviceColumnStream for any panel width (ring reuse)."""

import json
import os

import numpy as np
import pytest

from oracle import rlra_oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
META = json.load(open(os.path.join(GOLD, "golden.json")))
DRV = np.load(os.path.join(GOLD, "drivers.npz"))

pytestmark = pytest.mark.gpu
REL_ERR_TOL = 1e-10


def test_file_stream_single_pass_matches_reference(cuda_dev, tmp_path):
    import paper_2002_07138_b200 as P

    a = DRV["sp_a"]
    path = tmp_path / "sp.rlm"
    P.write_rlra(path, a)
    s = P.RlraFileColumnStream(path)
    f = P.single_pass_lu(s, 20, seed=0, q_os=5)
    assert isinstance(f.L, np.ndarray)
    assert np.array_equal(f.p, DRV["sp/p"]) and np.array_equal(f.q, DRV["sp/q"])
    assert abs(O.rel_fro_error_factor(a, f) - META["drivers"]["sp"]["rel_err"]) <= REL_ERR_TOL
    assert s.columns_pulled == a.shape[1]
    with pytest.raises(RuntimeError, match="single-use"):
        next(s.panels(8))


@pytest.mark.parametrize("panel", [1, 7, 16, 256, 1000])
def test_host_streams_bit_identical_to_device_stream(cuda_dev, tmp_path, panel):
    import torch

    import paper_2002_07138_b200 as P

    rng = np.random.default_rng(panel)
    a = np.asfortranarray(rng.standard_normal((300, 130)))
    path = tmp_path / "a.rlm"
    P.write_rlra(path, a)
    ref = P.stream_sketch(P.DeviceColumnStream(a), 12, 5, panel=panel)
    for s in (P.RlraFileColumnStream(path), P.DenseColumnStream(a)):
        got = P.stream_sketch(s, 12, 5, panel=panel)
        torch.cuda.synchronize()
        assert torch.equal(got.G, ref.G) and torch.equal(got.H, ref.H)
        assert s.columns_pulled == 130


def test_file_stream_truncated(cuda_dev, tmp_path):
    import paper_2002_07138_b200 as P

    path = tmp_path / "t.rlm"
    P.write_rlra(path, np.ones((50, 40)))
    s = P.RlraFileColumnStream(path)
    with open(path, "r+b") as fh:  # truncate after the header check
        fh.truncate(20 + 8 * 50 * 30)
    with pytest.raises(IOError, match="truncated"):
        P.stream_sketch(s, 5, 0, panel=16)


@pytest.mark.parametrize("panel", [64, 256])
def test_int8_sweep_matches_products_and_streams_agree(cuda_dev, tmp_path, monkeypatch, panel):
    """The int8 (Ozaki-II) sweep, forced at a small size: G = A^T Omega and
    H = A G within DGEMM-level normwise error of the float64 products, and the
    file / host / device streams bit-identical to each other."""
    import torch

    import paper_2002_07138_b200 as P
    from paper_2002_07138_b200 import ops, singlepass

    monkeypatch.setattr(singlepass, "SWEEP_OZ_MIN_ELEMS", 0)
    monkeypatch.setattr(singlepass, "SWEEP_PANEL", 512)
    rng = np.random.default_rng(7)
    a = np.asfortranarray(rng.standard_normal((1500, 1300)) * np.exp(rng.uniform(-3, 3, size=(1, 1300))))
    path = tmp_path / "a.rlm"
    P.write_rlra(path, a)
    ref = P.stream_sketch(P.DeviceColumnStream(a), 40, 2, panel=panel)
    g, h = ops.to_numpy(ref.G), ops.to_numpy(ref.H)
    om = O.gaussian(2, 1500, 40)
    g64 = a.T @ om
    h64 = a @ g64
    na = np.linalg.norm(a)
    assert np.abs(g - g64).max() <= 1e-13 * na * np.linalg.norm(om, axis=0).max()
    assert np.abs(h - h64).max() <= 1e-12 * na * np.linalg.norm(g64, axis=0).max()
    for s in (P.RlraFileColumnStream(path), P.DenseColumnStream(a)):
        got = P.stream_sketch(s, 40, 2, panel=panel)
        torch.cuda.synchronize()
        assert torch.equal(got.G, ref.G) and torch.equal(got.H, ref.H)
