"""CLI front-end (paper_2002_07138_b200/cli.py):
argument handling and the pass-budget mapping of rlra/cli.py:128-148 (CPU),
factor / adapt end to end on the device (GPU)."""

import csv
import json
import os

import numpy as np
import pytest

from paper_2002_07138_b200 import cli


class _Err(Exception):
    pass


def _error(msg):
    raise _Err(msg)


def test_budget_mapping_matches_the_reference():
    assert cli.resolve_budget(_error, "powerlu", None, None) == (3, None)
    assert cli.resolve_budget(_error, "powerlu", 5, None) == (5, None)
    assert cli.resolve_budget(_error, "powerlu", None, 2) == (6, 2)
    assert cli.resolve_budget(_error, "randlu", None, None) == (4, 1)
    assert cli.resolve_budget(_error, "randsvd", 6, None) == (6, 2)
    assert cli.resolve_budget(_error, "singlepass", None, None) == (None, None)
    for args in (("randlu", 5, None), ("powerlu", 3, 1), ("singlepass", 2, None)):
        with pytest.raises(_Err):
            cli.resolve_budget(_error, *args)


def test_parser_and_usage_errors():
    p = cli.build_parser()
    a = p.parse_args(["factor", "--in", "x.rlm", "--alg", "powerlu", "--rank", "5", "--device", "cuda:1",
                      "--csv", "o.csv"])
    assert (a.alg, a.rank, a.oversample, a.device, a.csv_out) == ("powerlu", 5, 10, "cuda:1", "o.csv")
    with pytest.raises(SystemExit) as e:
        p.parse_args(["factor", "--in", "x.rlm", "--alg", "nope", "--rank", "5"])
    assert e.value.code == 2
    assert cli.CSV_HEADER == ["alg", "matrix", "m", "n", "k", "eps", "v", "p", "seed", "rel_err", "rank", "passes",
                              "wall_ms"]


def test_non_cuda_device_is_refused():
    rc = cli.main(["factor", "--in", "missing.rlm", "--alg", "powerlu", "--rank", "5", "--device", "cpu"])
    assert rc == 1


def _kv(line):
    return dict(tok.split("=", 1) for tok in line.split() if "=" in tok)


@pytest.mark.gpu
def test_factor_and_adapt_on_device(cuda_dev, tmp_path, capsys):
    from oracle import rlra_oracle as O
    from paper_2002_07138_b200 import streams

    rng = np.random.default_rng(5)
    u, _ = np.linalg.qr(rng.standard_normal((300, 40)))
    v, _ = np.linalg.qr(rng.standard_normal((220, 40)))
    a = np.asfortranarray((u * np.exp(-np.arange(40) / 5.0)) @ v.T)
    path = str(tmp_path / "a.rlm")
    streams.write_rlra(path, a)
    out = str(tmp_path / "f")
    csvp = str(tmp_path / "runs.csv")
    assert cli.main(["factor", "--in", path, "--alg", "powerlu", "--rank", "15", "--passes", "4", "--seed", "3",
                     "--out-prefix", out, "--csv", csvp]) == 0
    info = _kv(capsys.readouterr().out.strip())
    ref = O.powerlu(a, 15, 10, 4, 3)
    assert (info["m"], info["n"], info["k"], info["v"], info["passes"]) == ("300", "220", "15", "4", "4")
    assert abs(float(info["rel_err"]) - O.rel_fro_error_factor(a, ref)) <= 1e-6 * O.rel_fro_error_factor(a, ref)
    assert np.array_equal(np.loadtxt(out + ".rowperm.txt").astype(np.int64), ref.p)
    assert streams.read_rlra(out + ".L.rlm").shape == (300, 15)
    for alg in ("randsvd", "randlu", "singlepass"):
        args = ["factor", "--in", path, "--alg", alg, "--rank", "15", "--csv", csvp]
        assert cli.main(args) == 0
        capsys.readouterr()
    assert cli.main(["adapt", "--in", path, "--tol", "1e-3", "--block", "5", "--l", "60", "--passes", "3",
                     "--csv", csvp]) == 0
    info = _kv(capsys.readouterr().out.strip())
    ref_f, ref_o = O.powerlu_fp(a, 1e-3, 5, 60, 3, 0)
    assert int(info["rank"]) == ref_o.rank and info["converged"] == "true"
    rows = list(csv.DictReader(open(csvp)))
    assert [r["alg"] for r in rows] == ["powerlu", "randsvd", "randlu", "singlepass", "powerlu_fp"]
    assert all(float(r["wall_ms"]) > 0 for r in rows)
    # not converged without restarts: exit code 3 (rlra/cli.py:36-38)
    assert cli.main(["adapt", "--in", path, "--tol", "1e-12", "--block", "5", "--l", "10", "--no-restart"]) == 3
