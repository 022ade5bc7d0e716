"""Host logic of the deferred rank checks (rangefinder.RankChecks): the parked
CholeskyQR2 flag and every queued count come back in one transfer, and the
first collapsed count in call order raises, as rlra/rangefinder.py:55-64 does
at each check."""
import pytest
import torch

from paper_2002_07138_b200.errors import RankCollapse
from paper_2002_07138_b200.rangefinder import RankChecks


def _cnt(v):
    return torch.tensor([v], dtype=torch.int64)


def test_flag_and_counts_in_one_fetch(monkeypatch):
    c = RankChecks()
    c.add(_cnt(10), 10)
    c.add(_cnt(10), 10)
    c.defer_cholqr(torch.tensor([0], dtype=torch.int32), "z")
    fetches = []
    orig = torch.Tensor.copy_

    def spy(dst, src, *a, **k):  # device -> host transfers of the fetch (into a host buffer)
        fetches.append(src.numel())
        return orig(dst, src, *a, **k)

    monkeypatch.setattr(torch.Tensor, "copy_", spy)
    assert c.cholqr_declined() == (False, "z")
    c.raise_if_collapsed()
    assert fetches == [3]  # two counts + the flag, one transfer; nothing left afterwards


def test_declined_then_later_counts():
    c = RankChecks()
    c.add(_cnt(5), 5)
    c.defer_cholqr(torch.tensor([1], dtype=torch.int32), None)
    declined, _ = c.cholqr_declined()
    assert declined
    c.add(_cnt(3), 4)  # the Householder redo's check, queued after the fetch
    with pytest.raises(RankCollapse):
        c.raise_if_collapsed()


def test_first_collapse_in_call_order_wins():
    c = RankChecks()
    c.add(_cnt(7), 9)
    c.defer_cholqr(torch.tensor([0], dtype=torch.int32), None)
    c.cholqr_declined()
    c.add(_cnt(1), 9)
    with pytest.raises(RankCollapse) as ei:
        c.raise_if_collapsed()
    assert (ei.value.achieved, ei.value.requested) == (7, 9)
    c.raise_if_collapsed()  # state cleared
    assert c.cholqr_declined() is None
