"""End-to-end parity of the drop-in drivers against the reference's golden
outputs (tests/golden/, produced by the unmodified reference) and the oracle.

Bar (BASELINE.json north_star): identical pivot sequences p, q and rank;
relative Frobenius reconstruction error within 1e-10 of the reference's."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import rlra_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
META = json.load(open(os.path.join(GOLD, "golden.json")))
DRV = np.load(os.path.join(GOLD, "drivers.npz"))

pytestmark = pytest.mark.gpu

REL_ERR_TOL = 1e-10  # |rel_err_gpu - rel_err_ref|, BASELINE.json north_star


def sha_i64(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def lu_structure_ok(f):
    return np.count_nonzero(np.triu(f.L, 1)) == 0 and np.count_nonzero(np.tril(f.U, -1)) == 0


@pytest.mark.parametrize("v", [2, 3, 4, 5, 6])
def test_powerlu_matches_reference(cuda_dev, v):
    import paper_2002_07138_b200 as P

    a = DRV["pl_a"]
    f = P.powerlu(a, 30, q_os=10, v=v, seed=1)
    assert isinstance(f.L, np.ndarray)
    assert np.array_equal(f.p, DRV[f"pl_v{v}/p"])
    assert np.array_equal(f.q, DRV[f"pl_v{v}/q"])
    err = O.rel_fro_error_factor(a, f)
    assert abs(err - META["drivers"][f"pl_v{v}"]["rel_err"]) <= REL_ERR_TOL
    assert lu_structure_ok(f)
    np.testing.assert_allclose(f.L, DRV[f"pl_v{v}/L"], rtol=0, atol=1e-9)


@pytest.mark.parametrize("v", [2, 3, 4, 5])
def test_powerlu_exact_rank_all_parities(cuda_dev, v):
    import paper_2002_07138_b200 as P

    a = DRV["exact_a"]
    f = P.powerlu(a, 8, q_os=4, v=v, seed=0)
    assert O.rel_fro_error_factor(a, f) < 1e-12  # pkg/tests/test_fixedrank.py:50-56
    assert np.array_equal(f.p, DRV[f"exact_v{v}/p"]) and np.array_equal(f.q, DRV[f"exact_v{v}/q"])


def test_basis_v2_is_qr_of_transpose_sketch(cuda_dev):
    import paper_2002_07138_b200 as P

    b = P.general_power_basis_v(P.DeviceMatrix(DRV["pl_a"]), 40, 2, 9)
    from paper_2002_07138_b200 import ops

    V = ops.to_numpy(b.V)
    assert b.passes_used == 1
    np.testing.assert_allclose(V, DRV["basis_v2/V"], rtol=0, atol=1e-12)
    b = P.general_power_basis_v(P.DeviceMatrix(DRV["pl_a"]), 40, 5, 9)
    assert b.passes_used == 4
    np.testing.assert_allclose(ops.to_numpy(b.V), DRV["basis_v5/V"], rtol=0, atol=1e-9)


def test_pass_budgets_exact(cuda_dev):
    import paper_2002_07138_b200 as P

    a = O.gaussian(10, 60, 45)
    for v in (2, 3, 4, 5, 6):
        acc = P.InstrumentedAccessor(a)
        P.powerlu(acc, 8, q_os=4, v=v, seed=0)
        assert acc.product_count == v
        acc = P.InstrumentedAccessor(a)
        P.adaptive_rank(acc, P.PrecisionParams(1e-3, 5, 20, v), seed=0)
        assert acc.product_count == v


def test_adaptive_rank_matches_reference(cuda_dev):
    import paper_2002_07138_b200 as P

    ref = META["drivers"]["fp"]
    o = P.adaptive_rank(DRV["fp_a"], P.PrecisionParams(1e-3, 5, 60, 4), seed=0)
    assert o.converged and o.rank == ref["rank"]
    assert abs(o.residual_energy - ref["residual"]) <= 1e-9 * O.fro_norm(DRV["fp_a"]) ** 2
    np.testing.assert_allclose(np.abs(o.V), np.abs(DRV["fp/V"]), atol=1e-9)
    fac, o2 = P.powerlu_fp(DRV["fp_a"], P.PrecisionParams(1e-3, 5, 60, 4), seed=0)
    assert fac.rank == o2.rank == META["drivers"]["fpfac"]["rank"]
    assert np.array_equal(fac.p, DRV["fpfac/p"]) and np.array_equal(fac.q, DRV["fpfac/q"])
    assert abs(O.rel_fro_error_factor(DRV["fp_a"], fac) - META["drivers"]["fpfac"]["rel_err"]) <= REL_ERR_TOL


def test_adaptive_rank_not_converged(cuda_dev):
    import paper_2002_07138_b200 as P

    params = P.PrecisionParams(1e-6, 10, 20, 4)
    o = P.adaptive_rank(DRV["fp_nc_a"], params, seed=0)
    assert not o.converged and o.rank == 20 and o.V.shape == (120, 20)
    assert abs(o.residual_energy - META["drivers"]["fp_nc"]["residual"]) <= 1e-12
    with pytest.raises(P.NotConverged) as exc:
        P.powerlu_fp(DRV["fp_nc_a"], params, seed=0)
    assert exc.value.outcome.rank == 20 and not exc.value.outcome.converged


def test_eps_one_stops_immediately(cuda_dev):
    import paper_2002_07138_b200 as P

    a = O.gaussian(3, 60, 60)
    o = P.adaptive_rank(a, P.PrecisionParams(1.0, 5, 20, 4), seed=0)
    assert o.converged and o.rank == 1


def test_single_pass_matches_reference(cuda_dev):
    import paper_2002_07138_b200 as P

    f = P.single_pass_lu(P.DenseColumnStream(DRV["sp_a"]), 20, seed=0, q_os=5)
    assert f.L.shape == (120, 20) and f.U.shape == (20, 100)
    assert np.array_equal(f.p, DRV["sp/p"]) and np.array_equal(f.q, DRV["sp/q"])
    assert abs(O.rel_fro_error_factor(DRV["sp_a"], f) - META["drivers"]["sp"]["rel_err"]) <= REL_ERR_TOL
    s = P.DeviceColumnStream(DRV["sp_a"])
    g, h = P.stream_sketch(s, 25, 3, panel=16)
    from paper_2002_07138_b200 import ops

    assert s.columns_pulled == 100
    np.testing.assert_allclose(ops.to_numpy(g), DRV["sk/G"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(ops.to_numpy(h), DRV["sk/H"], rtol=0, atol=1e-11)


def test_identity_stream_sketch_is_the_draw(cuda_dev):
    import paper_2002_07138_b200 as P
    from paper_2002_07138_b200 import ops

    g, h = P.stream_sketch(P.DeviceColumnStream(np.eye(30)), 6, seed=3, panel=7)
    om = O.gaussian(3, 30, 6)
    assert np.array_equal(ops.to_numpy(g), om) and np.array_equal(ops.to_numpy(h), om)


def test_single_pass_rejects_rank_above_numerical_rank(cuda_dev):
    import paper_2002_07138_b200 as P

    rng = np.random.default_rng(10)
    a = O.gaussian_from(rng, 80, 5) @ O.gaussian_from(rng, 5, 60)
    with pytest.raises(P.IllPosedPseudoinverse):
        P.single_pass_lu(P.DenseColumnStream(a), 8, seed=0)


def test_stream_single_use_and_length(cuda_dev):
    import paper_2002_07138_b200 as P

    s = P.DeviceColumnStream(np.eye(5))
    list(s.panels(2))
    with pytest.raises(RuntimeError, match="single-use"):
        list(s.panels(2))


def test_rank_collapse_from_duplicated_rows(cuda_dev):
    import paper_2002_07138_b200 as P

    base = O.gaussian(17, 5, 30)
    a = np.vstack([base] * 8)  # pkg/tests/test_fixedrank.py:159-167
    with pytest.raises(P.RankCollapse):
        P.powerlu(a, 10, q_os=5, v=4, seed=0)


def test_rank_collapse_reports_achieved_width(cuda_dev):
    import paper_2002_07138_b200 as P

    a = np.diag([1.0, 1.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0])
    with pytest.raises(P.RankCollapse) as exc:
        P.general_power_basis_v(a, 5, 2, seed=0)
    assert exc.value.achieved == 3 and exc.value.requested == 5


def test_validation_errors(cuda_dev):
    import paper_2002_07138_b200 as P

    a = O.gaussian(18, 20, 10)
    for args in [(0, 2, 3), (8, 5, 3), (4, 2, 1)]:
        with pytest.raises(ValueError):
            P.powerlu(a, args[0], q_os=args[1], v=args[2], seed=0)
    with pytest.raises(ValueError, match="width"):
        P.adaptive_rank(O.gaussian(11, 30, 25), P.PrecisionParams(1e-2, 10, 30, 4), seed=0)


def test_c1_config_matches_reference(cuda_dev):
    import paper_2002_07138_b200 as P
    from paper_2002_07138_b200 import configs

    a = configs.gen_c1()
    f = P.powerlu(a, 50, 10, 3, 0)
    ref = META["configs"]["C1"]
    assert sha_i64(f.p) == ref["p_sha"] and sha_i64(f.q) == ref["q_sha"]
    assert abs(O.rel_fro_error_factor(a, f) - ref["rel_err"]) <= REL_ERR_TOL


@pytest.mark.slow
@pytest.mark.parametrize("v", [2, 3, 4, 5, 6])
def test_c2_config_matches_reference(cuda_dev, v):
    import paper_2002_07138_b200 as P
    from paper_2002_07138_b200 import configs

    a = _c2()
    dm = P.DeviceMatrix(a)
    f = P.powerlu(dm, 200, 20, v, 0).to_numpy()
    ref = META["configs"][f"C2_v{v}"]
    pq = np.load(os.path.join(GOLD, "c2_pq.npz"))
    assert np.array_equal(f.p, pq[f"v{v}_p"]), "row pivots differ from the reference"
    assert np.array_equal(f.q, pq[f"v{v}_q"]), "column pivots differ from the reference"
    assert abs(O.rel_fro_error_factor(a, f) - ref["rel_err"]) <= REL_ERR_TOL


_C2 = {}


def _c2():
    from paper_2002_07138_b200 import configs

    if "a" not in _C2:
        _C2["a"] = configs.gen_c2()
    return _C2["a"]


def test_distributed_path_single_rank_nccl(cuda_dev):
    """The row-sharded orchestration with the CUDA ops over a 1-rank NCCL group
    reproduces the single-GPU drop-in result (multi-rank logic: gloo tests)."""
    import os

    import torch.distributed as dist

    import paper_2002_07138_b200 as P
    from paper_2002_07138_b200 import distributed as D, ops

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda_dev)
    try:
        a = DRV["pl_a"]
        A = D.ShardedMatrix(ops.from_numpy(a, cuda_dev), a.shape[0], 0, a.shape[0], D.CudaOps(cuda_dev))
        f = D.powerlu(A, 30, 10, 4, 1, O.gaussian)
        assert np.array_equal(f.p.cpu().numpy(), DRV["pl_v4/p"])
        assert np.array_equal(f.q.cpu().numpy(), DRV["pl_v4/q"])
        fd = P.LowRankLU(f.p.cpu().numpy(), f.q.cpu().numpy(), ops.to_numpy(f.L), ops.to_numpy(f.U), 30)
        assert abs(O.rel_fro_error_factor(a, fd) - META["drivers"]["pl_v4"]["rel_err"]) <= REL_ERR_TOL
        fa = DRV["fp_a"]
        B = D.ShardedMatrix(ops.from_numpy(fa, cuda_dev), fa.shape[0], 0, fa.shape[0], D.CudaOps(cuda_dev))
        fp, r = D.powerlu_fp(B, 1e-3, 5, 60, 4, 0, O.gaussian)
        assert r == META["drivers"]["fp"]["rank"]
        assert np.array_equal(fp.p.cpu().numpy(), DRV["fpfac/p"])
        # TSLU interior step on the CUDA ops (the multi-rank tournament: gloo tests):
        # W = Y U^{-1} with W unit lower at the tournament's pivot rows
        y = np.asfortranarray(O.gaussian(3, 500, 40))
        Y = D.ShardedMatrix(ops.from_numpy(y, cuda_dev), 500, 0, 500, D.CudaOps(cuda_dev))
        w = ops.to_numpy(D.tslu_basis_rows(Y, Y.local, 40))
        ref = O.plu(y)
        w_ref = O.apply_inv_row_perm(ref.p, ref.L)  # exact GEPP's P^T L: same U for one rank
        assert np.abs(w - w_ref).max() <= 1e-12 * np.abs(w_ref).max()
        # single-pass (C4's path): sharded sweep with the per-panel all-reduce
        sa = DRV["sp_a"]
        S = D.ShardedMatrix(ops.from_numpy(sa, cuda_dev), sa.shape[0], 0, sa.shape[0], D.CudaOps(cuda_dev))
        sp = D.single_pass_lu(S, 20, 0, O.gaussian, q_os=5)
        assert np.array_equal(sp.p.cpu().numpy(), DRV["sp/p"]) and np.array_equal(sp.q.cpu().numpy(), DRV["sp/q"])
        spd = P.LowRankLU(sp.p.cpu().numpy(), sp.q.cpu().numpy(), ops.to_numpy(sp.L), ops.to_numpy(sp.U), 20)
        assert abs(O.rel_fro_error_factor(sa, spd) - META["drivers"]["sp"]["rel_err"]) <= REL_ERR_TOL
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n", [(3000, 96), (600, 230), (70000, 64)])
def test_row_sharded_gepp_primitives_on_device(cuda_dev, m, n):
    """distributed.dist_getrf_ on the CUDA ops (getrf_block on the gathered
    panel, lu_trsm_rows, lu_update_split; one rank -- the multi-rank exchanges
    are the gloo tests): every bit of the packed factor and the pivots equal
    the one-launch kernel's / the reference's, cooperative and blocked panel
    paths (70000 rows)."""
    import os

    import torch
    import torch.distributed as dist

    from paper_2002_07138_b200 import distributed as D, ops

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29519")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda_dev)
    try:
        rng = np.random.default_rng(m + n)
        a = rng.standard_normal((m, n))
        a[:, 40] = a[:, 7]
        a[:, 50] = 0.0
        a = np.asfortranarray(a)
        loc = ops.from_numpy(a, cuda_dev)
        S = D.ShardedMatrix(loc, m, 0, m, D.CudaOps(cuda_dev))
        piv, urows, cnt = D.dist_getrf_(S, loc)
        lu_ref = a.copy(order="F")
        piv_ref = np.arange(m, dtype=np.int64)
        O.plu_inplace(lu_ref, piv_ref)
        assert np.array_equal(piv.cpu().numpy(), piv_ref)
        assert np.array_equal(ops.to_numpy(loc).view(np.int64), lu_ref.view(np.int64))
        assert np.array_equal(ops.to_numpy(urows).view(np.int64), lu_ref[:n].view(np.int64))
        assert int(cnt.item()) == int(np.count_nonzero(np.diag(lu_ref)))
        L = np.tril(lu_ref[:, :n], -1)
        L[np.arange(n), np.arange(n)] = 1.0
        for r0, r1 in ((0, 50), (40, 300), (400, 600)):  # straddling the last column and past it
            l_rows = D.CudaOps(cuda_dev).unit_lower_rows(loc[r0:r1], r0)
            assert np.array_equal(ops.to_numpy(l_rows), L[r0:r1])
    finally:
        dist.destroy_process_group()


def test_pipelined_upload_matches_resident(cuda_dev, monkeypatch):
    """Pinned host input: column chunks are uploaded on a copy stream and the
    first pass consumes them as they land; results equal the resident run."""
    import torch

    import paper_2002_07138_b200 as P
    from paper_2002_07138_b200 import device

    monkeypatch.setattr(device.DeviceMatrix, "PIPELINE_MIN_BYTES", 1)
    a = DRV["pl_a"]
    pinned = torch.empty((a.shape[1], a.shape[0]), dtype=torch.float64, pin_memory=True)
    ah = pinned.numpy().T
    ah[...] = a
    for v in (3, 4):
        f = P.powerlu(ah, 30, q_os=10, v=v, seed=1)
        assert np.array_equal(f.p, DRV[f"pl_v{v}/p"]) and np.array_equal(f.q, DRV[f"pl_v{v}/q"])
        assert abs(O.rel_fro_error_factor(a, f) - META["drivers"][f"pl_v{v}"]["rel_err"]) <= REL_ERR_TOL
    dm = P.DeviceMatrix(ah)
    z = dm.rmatmul(np.eye(200)[:, :5])
    from paper_2002_07138_b200 import ops

    np.testing.assert_allclose(ops.to_numpy(z), a.T @ np.eye(200)[:, :5], rtol=0, atol=1e-14)


@pytest.mark.parametrize("graded_tail", [False, True])
def test_residues_built_during_the_upload_equal_one_shot(cuda_dev, graded_tail):
    """ops.OzPipeline (residues per column chunk while A uploads, provisional
    scale from the first chunk) produces exactly OzPrep's residue set and
    header; when a later chunk raises the max norm (graded_tail) the final
    scale differs and the residues are rebuilt -- still identical."""
    import torch

    from paper_2002_07138_b200 import ops

    rng = np.random.default_rng(31)
    a = np.asfortranarray(rng.standard_normal((3000, 1900)))
    if graded_tail:
        a[:, 1500:] *= 64.0
    ad = ops.from_numpy(a, cuda_dev)
    ref = ops.OzPrep(ad)
    pipe = ops.OzPipeline(ad)
    for c0 in range(0, 1900, 512):
        pipe.chunk(c0, min(1900, c0 + 512))
    got = pipe.finish()
    got._resolve()  # the host reads the header lazily (first product)
    assert pipe.rebuilt == graded_tail
    assert got.ok == ref.ok
    assert torch.equal(got.ws[:4], ref.ws[:4])  # eA
    hdr = ops.OZ_HEADER_BYTES
    assert torch.equal(got.ws[8:40], ref.ws[8:40])  # guard statistics
    off = ref.ws.numel() - 14 * 3072 * 1920  # the residue tiles fill the tail of the workspace
    assert torch.equal(got.ws[off:], ref.ws[off:])
    b = ops.from_numpy(rng.standard_normal((1900, 30)), cuda_dev)
    assert torch.equal(got.gemm(b).view(torch.int64), ref.gemm(b).view(torch.int64))


def test_pipelined_e2e_call_uses_the_upload_residues(cuda_dev, monkeypatch):
    """The drop-in call on a pinned host A builds its residues during the
    upload (no separate pass over A afterwards) and matches the golden pivots."""
    import torch

    import paper_2002_07138_b200 as P
    from paper_2002_07138_b200 import device, ops

    monkeypatch.setattr(device.DeviceMatrix, "PIPELINE_MIN_BYTES", 1)
    built = []
    real = ops.OzPipeline.finish

    def spy(self):
        built.append(self)
        return real(self)

    monkeypatch.setattr(ops.OzPipeline, "finish", spy)
    rng = np.random.default_rng(32)
    x, _ = np.linalg.qr(rng.standard_normal((2500, 60)))
    y, _ = np.linalg.qr(rng.standard_normal((1800, 60)))
    a = np.asfortranarray((x * np.exp(-np.arange(60) / 8.0)) @ y.T + 1e-9 * rng.standard_normal((2500, 1800)))
    pinned = torch.empty((a.shape[1], a.shape[0]), dtype=torch.float64, pin_memory=True)
    ah = pinned.numpy().T
    ah[...] = a
    for v in (3, 4):
        f = P.powerlu(ah, 25, q_os=10, v=v, seed=2)
        g = O.powerlu(a, 25, q_os=10, v=v, seed=2)
        assert np.array_equal(f.p, g.p) and np.array_equal(f.q, g.q)
        assert abs(O.rel_fro_error_factor(a, f) - O.rel_fro_error_factor(a, g)) <= REL_ERR_TOL
    assert len(built) == 2 and not any(b.rebuilt for b in built)


@pytest.mark.parametrize("v", [2, 3, 4])
def test_powerlu_cholqr_decline_falls_back_to_householder(cuda_dev, monkeypatch, v):
    """Exact-rank input: the CholeskyQR2 basis declines (singular Gram); the
    deferred flag makes powerlu redo the basis, G and the assembly on the
    Householder path -- identical to running Householder from the start."""
    import paper_2002_07138_b200 as P
    from paper_2002_07138_b200 import fixedrank, ops

    a = DRV["exact_a"]
    calls = []
    orig = ops.cholqr2
    monkeypatch.setattr(ops, "cholqr2", lambda z: calls.append(1) or orig(z))
    f = P.powerlu(a, 8, q_os=4, v=v, seed=0)
    assert calls, "CholeskyQR2 path not taken"
    monkeypatch.setattr(fixedrank, "POWERLU_QR", "householder")
    g = P.powerlu(a, 8, q_os=4, v=v, seed=0)
    assert np.array_equal(f.p, g.p) and np.array_equal(f.q, g.q)
    assert np.array_equal(f.p, DRV[f"exact_v{v}/p"]) and np.array_equal(f.q, DRV[f"exact_v{v}/q"])
    assert np.abs(f.L @ f.U - g.L @ g.U).max() <= 1e-12 * np.abs(g.L @ g.U).max()


@pytest.mark.parametrize("block", [7, 2048])
def test_device_validation_metric_matches_oracle(cuda_dev, block):
    """K9 (validate.rel_err_device: L U per column block on the DMMA GEMM, the
    fused gather/difference/double-double kernel) against the oracle's
    ||A - P^T (L U) Q^T||_F / ||A||_F (rlra/fixedrank.py:149-155)."""
    import paper_2002_07138_b200 as P
    from paper_2002_07138_b200 import ops, validate

    a = DRV["pl_a"]
    f = P.powerlu(a, 30, q_os=10, v=4, seed=1)
    ref = O.rel_fro_error_factor(a, f)
    got = validate.rel_err_device(ops.from_numpy(a, cuda_dev), f, block=block)
    assert abs(got - ref) <= 1e-13 * ref
