"""The .rlm container (rlra/fileio.py:14-46) as restated in
paper_2002_07138_b200/streams.py: byte layout identical to the reference's
writer, header validation errors.  CPU only."""

import os
import sys

import numpy as np
import pytest

from paper_2002_07138_b200 import streams

REF = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle", "_ref")


def test_roundtrip_and_layout(tmp_path):
    a = np.random.default_rng(0).standard_normal((7, 5))
    p = tmp_path / "a.rlm"
    streams.write_rlra(p, a)
    raw = p.read_bytes()
    assert raw[:4] == b"RLRA" and len(raw) == 20 + 8 * 35
    assert np.array_equal(np.frombuffer(raw[20:], "<f8"), a.ravel(order="F"))
    assert streams.read_rlra_header(p) == (7, 5)
    assert np.array_equal(streams.read_rlra(p), a)


def test_header_errors(tmp_path):
    p = tmp_path / "bad.rlm"
    p.write_bytes(b"NOPE" + b"\0" * 16)
    with pytest.raises(IOError, match="not an RLRA"):
        streams.read_rlra_header(p)
    streams.write_rlra(p, np.ones((3, 3)))
    with open(p, "ab") as fh:
        fh.write(b"\0" * 8)
    with pytest.raises(IOError, match="size does not match"):
        streams.read_rlra_header(p)
    with pytest.raises(ValueError):
        streams.write_rlra(p, np.ones(3))


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "rlra")), reason="reference not built in oracle/_ref")
def test_bytes_identical_to_reference_writer(tmp_path):
    sys.path.insert(0, REF)
    try:
        from rlra import fileio
    finally:
        sys.path.remove(REF)
    a = np.random.default_rng(1).standard_normal((11, 4))
    streams.write_rlra(tmp_path / "ours.rlm", a)
    fileio.write_rlra(tmp_path / "ref.rlm", a)
    assert (tmp_path / "ours.rlm").read_bytes() == (tmp_path / "ref.rlm").read_bytes()
    assert fileio.read_rlra_header(tmp_path / "ours.rlm") == (11, 4)
