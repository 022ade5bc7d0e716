"""Multi-rank orchestration of the row-sharded PowerLU (paper_2002_07138_b200/
distributed.py) on CPU: world_size 2 over gloo, with an ops object backed by
the ORACLE (test infrastructure) in place of the CUDA kernels.  Checks that the
sharded passes, the all-reduced A^T Y, the all-gathered exact GEPPs and the
energy all-reduce reproduce the single-process reference algorithm: identical
pivots p, q and rank, reconstruction error equal to 1e-12."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import rlra_oracle as O


class OracleOps:
    """CPU stand-in for CudaOps (column-major torch CPU tensors)."""

    def _f(self, m, n):
        return torch.empty((max(n, 1), max(m, 1)), dtype=torch.float64).t()[:m, :n]

    def upload(self, a):
        a = np.asfortranarray(a)
        t = self._f(*a.shape)
        t.copy_(torch.from_numpy(a))
        return t

    def empty(self, m, n):
        return self._f(m, n)

    def matmul(self, a, b, ta=False, tb=False):
        x = a.t() if ta else a
        y = b.t() if tb else b
        r = x @ y
        out = self._f(*r.shape)
        out.copy_(r)
        return out

    def zeros(self, m, n):
        t = self._f(m, n)
        t.zero_()
        return t

    # sharded factorizations of the replicated sketches (CholeskyQR2 / TSQR)
    decline = False  # force the CholeskyQR2 decline -> TSQR path

    def chol_inv(self, g, cond_limit, flag=None):
        flag = torch.zeros(1, dtype=torch.int32) if flag is None else flag
        gn = g.numpy()
        try:
            r = np.linalg.cholesky(gn).T
            d = np.abs(np.diag(r))
            if self.decline or d.max() > cond_limit * d.min():
                raise np.linalg.LinAlgError
            return self.upload(np.linalg.inv(r)), flag
        except np.linalg.LinAlgError:
            flag[0] = 1
            return self.upload(np.zeros_like(gn)), flag

    def cholqr_ok(self, x):
        return x.shape[0] >= x.shape[1] > 0

    wide_at = 10 ** 9  # sketches wider than this take the shifted CholeskyQR3 steps

    def cholqr_wide(self, l):
        return l > self.wide_at

    def shift_gram(self, g, n, flag):
        gn = g.numpy()
        l = gn.shape[0]
        if np.any(np.diag(gn) == 0):
            flag[0] = 1
        g += torch.eye(l, dtype=torch.float64) * (11.0 * 2.0 ** -53 * (n * l + l * (l + 1)) * np.trace(gn))

    def gram_identity_flag(self, g, flag):
        if np.abs(g.numpy() - np.eye(g.shape[0])).max() > 0.1:
            flag[0] = 1

    def flag_value(self, flag):
        return int(flag[0])

    def qr_qr(self, x):
        q, r = np.linalg.qr(x.numpy())
        return self.upload(q), self.upload(r)

    def nonzero_diag(self, r):
        return torch.tensor([int(np.count_nonzero(np.diag(r.numpy())))])

    # ---- row-sharded exact GEPP primitives (numpy restatement, reference op order)
    def gepp_state(self, m, n):
        return {"piv": torch.arange(m, dtype=torch.int64), "zflag": torch.zeros(max(n, 1), dtype=torch.int32),
                "ipiv": torch.zeros(max(n, 1), dtype=torch.int64), "cnt": torch.zeros(1, dtype=torch.int64)}

    def getrf_block(self, panel, j0, nbo, stt):
        """rlra/_lu_cython.pyx:23-55 restricted to columns [j0, j0+nbo)."""
        a = panel.numpy()
        piv, z, ip = stt["piv"].numpy(), stt["zflag"].numpy(), stt["ipiv"].numpy()
        m = a.shape[0]
        for c in range(nbo):
            j = j0 + c
            act = np.abs(a[j:, c])
            amax = act.max() if act.size else -1.0
            rel = j + int(np.argmax(act)) if act.size else j
            colmax = max(amax, np.abs(a[:j, c]).max()) if j > 0 else amax
            if amax <= 1e-14 * colmax:
                a[j + 1:, c] = 0.0
                z[j], ip[j] = 1, j
                continue
            z[j], ip[j] = 0, rel
            if rel != j:
                a[[j, rel], :] = a[[rel, j], :]
                piv[[j, rel]] = piv[[rel, j]]
            a[j + 1:, c] = a[j + 1:, c] / a[j, c]
            for cc in range(c + 1, nbo):
                a[j + 1:, cc] = a[j + 1:, cc] - a[j + 1:, c] * a[j, cc]
        stt["cnt"] += int(np.count_nonzero([a[j0 + c, c] for c in range(nbo)]))

    def ipiv_host(self, stt, j0, nbo):
        return stt["ipiv"][j0:j0 + nbo].tolist()

    def unit_lower_rows(self, local, pos0):
        rows, n = local.shape
        a = np.tril(local.numpy(), pos0 - 1)
        for i in range(rows):
            if pos0 + i < n:
                a[i, pos0 + i] = 1.0
        return self.upload(a)

    def lu_trsm_rows(self, blk, j0, nbo, c0, c1, stt):
        b = blk.numpy()
        z = stt["zflag"].numpy()
        for t in range(nbo - 1):
            if not z[j0 + t]:
                b[t + 1:, c0:c1] = b[t + 1:, c0:c1] - np.outer(b[t + 1:, j0 + t], b[t, c0:c1])

    def lu_update_split(self, local, blk, j0, nbo, r_lo, c0, c1, stt):
        a, b = local.numpy(), blk.numpy()
        z = stt["zflag"].numpy()
        for t in range(nbo):
            if not z[j0 + t]:
                a[r_lo:, c0:c1] = a[r_lo:, c0:c1] - np.outer(a[r_lo:, j0 + t], b[t, c0:c1])

    def sweep_products(self, block, prep, x, out, ta, add):
        r = (block.t() @ x) if ta else (block @ x)
        if add:
            out += r
        else:
            out.copy_(r)
        return out

    def pinv_transpose_apply(self, g, m_):
        return self.upload(O.pinv_transpose_apply(g.numpy(), m_.numpy()))

    def getrf_(self, a):
        lu = np.asfortranarray(a.numpy())
        piv = np.arange(lu.shape[0], dtype=np.int64)
        O.plu_inplace(lu, piv)
        a.copy_(torch.from_numpy(lu))
        r = min(a.shape)
        return torch.from_numpy(piv), torch.tensor([int(np.count_nonzero(np.diag(lu)[:r]))])

    def lu_basis(self, lu, piv):
        lun = lu.numpy()
        r = min(lun.shape)
        L = np.tril(lun[:, :r], -1)
        L[np.arange(r), np.arange(r)] = 1.0
        return self.upload(O.apply_inv_row_perm(piv.numpy(), L))

    def lu_extract(self, lu):
        lun = lu.numpy()
        r = min(lun.shape)
        L = np.tril(lun[:, :r], -1)
        L[np.arange(r), np.arange(r)] = 1.0
        return self.upload(L), self.upload(np.triu(lun[:r, :]))

    def qr_q(self, x):
        q, r = np.linalg.qr(x.numpy())
        return self.upload(q), torch.tensor([int(np.count_nonzero(np.diag(r)))])

    def transpose(self, a):
        return self.upload(a.numpy().T)

    def sumsq(self, a):
        return torch.tensor([float((a.numpy() ** 2).sum())], dtype=torch.float64)

    def colsumsq(self, a):
        an = a.numpy()
        return torch.tensor([float(an[:, j] @ an[:, j]) for j in range(an.shape[1])], dtype=torch.float64)

    def gather_rows(self, x, idx):
        return self.upload(x.numpy()[idx.numpy()])

    def right_solve_upper(self, x, u):
        from scipy.linalg import solve_triangular

        return self.upload(solve_triangular(u.numpy(), x.numpy().T, trans="T", lower=False).T)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2002_07138_b200 import distributed as D

    D.INTERIOR = case.get("interior", "tslu")
    D.REPL_TSLU_MIN_ROWS = case.get("repl_tslu_min_rows", 0)  # exercise the sharded n x l tournament on small cases
    try:
        a = case["a"]
        m = a.shape[0]
        r0, r1 = D.row_range(m, world, rank)
        ops = OracleOps()
        ops.decline = case.get("decline", False)
        ops.wide_at = case.get("wide_at", 10 ** 9)
        A = D.ShardedMatrix(ops.upload(a[r0:r1]), m, r0, r1, ops)
        if case["kind"] == "getrf":
            piv, urows, cnt = D.dist_getrf_(A, A.local)
            out = (piv.numpy().copy(), A.local.numpy().copy(), urows.numpy().copy(), int(cnt[0]), r0, r1)
        elif case["kind"] == "api":
            # the reference signatures on a ShardedMatrix (rlra/fixedrank.py:120,
            # rlra/fixedprec.py:152, rlra/singlepass.py:123, rlra/rangefinder.py:144)
            import paper_2002_07138_b200 as P

            A.omega_fn = O.gaussian
            f = P.powerlu(A, case["k"], case["q_os"], case["v"], case["seed"])
            fp, outc = P.powerlu_fp(A, P.PrecisionParams(1e-3, 5, 60, 4), 0)
            sp = P.single_pass_lu(A, case["k"], case["seed"], q_os=4, panel=16)
            basis = P.general_power_basis_v(A, 20, 3, 1)
            out = ([x.numpy().copy() for x in (f.p, f.q, f.L, f.U)], outc.rank, outc.G.shape,
                   [x.numpy().copy() for x in (fp.p, fp.q)], [x.numpy().copy() for x in (sp.p, sp.q)],
                   basis.V.numpy().copy(), basis.passes_used)
        elif case["kind"] == "single_pass":
            f = D.single_pass_lu(A, case["k"], case["seed"], O.gaussian, q_os=case["q_os"], panel=case["panel"])
            out = (f.p.numpy().copy(), f.q.numpy().copy(), f.full_L().numpy().copy(), f.U.numpy().copy(),
                   A.product_count)
        elif case["kind"] == "powerlu":
            f = D.powerlu(A, case["k"], case["q_os"], case["v"], case["seed"], O.gaussian)
            out = (f.p.numpy().copy(), f.q.numpy().copy(), f.full_L().numpy().copy(), f.U.numpy().copy(),
                   A.product_count)
        else:
            f, rank_ = D.powerlu_fp(A, case["eps"], case["b"], case["l"], case["v"], case["seed"], O.gaussian)
            out = (f.p.numpy().copy(), f.q.numpy().copy(), f.full_L().numpy().copy(), f.U.numpy().copy(), rank_)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def run_dist(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return res


def decay_matrix(m, n, seed, r=None):
    rng = np.random.default_rng(seed)
    r = r or min(m, n)
    u, _ = np.linalg.qr(rng.standard_normal((m, r)))
    vv, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return np.asfortranarray((u * np.exp(-np.arange(r) / 7.0)) @ vv.T)


@pytest.mark.parametrize("v", [2, 3, 4, 5])
def test_sharded_powerlu_matches_single_process(v):
    a = decay_matrix(203, 150, seed=v)  # 203 rows: uneven shards
    res = run_dist({"kind": "powerlu", "a": a, "k": 20, "q_os": 8, "v": v, "seed": 1, "interior": "tslu_always"})
    ref = O.powerlu(a, 20, 8, v, 1)
    for rank, (p, q, L, U, passes) in res.items():
        assert np.array_equal(p, ref.p) and np.array_equal(q, ref.q)
        f = O.LowRankLU(p, q, L, U, 20)
        assert abs(O.rel_fro_error_factor(a, f) - O.rel_fro_error_factor(a, ref)) <= 1e-12
        assert passes == v - 1 + 1  # v - 1 basis passes + the final G pass
    np.testing.assert_array_equal(res[0][2], res[1][2])  # replicated factors


def test_sharded_powerlu_fp_rank_matches():
    a = decay_matrix(180, 160, seed=11)
    res = run_dist({"kind": "fp", "a": a, "eps": 1e-3, "b": 5, "l": 60, "v": 4, "seed": 0})
    ref_f, ref_o = O.powerlu_fp(a, 1e-3, 5, 60, 4, 0)
    for rank, (p, q, L, U, r) in res.items():
        assert r == ref_o.rank
        assert np.array_equal(p, ref_f.p) and np.array_equal(q, ref_f.q)


def test_sharded_interior_gather_path_matches():
    """RLRA_B200_DIST_INTERIOR=gather: all-gathered exact interior GEPPs."""
    a = decay_matrix(203, 150, seed=4)
    res = run_dist({"kind": "powerlu", "a": a, "k": 20, "q_os": 8, "v": 4, "seed": 1, "interior": "gather"})
    ref = O.powerlu(a, 20, 8, 4, 1)
    for rank, (p, q, L, U, passes) in res.items():
        assert np.array_equal(p, ref.p) and np.array_equal(q, ref.q)


def test_sharded_tslu_shards_shorter_than_sketch():
    """world 4, 62 rows: shards of 16 / 16 / 16 / 14 rows < l = 20 (zero-padded
    candidate blocks in the tournament)."""
    a = decay_matrix(62, 40, seed=8)
    res = run_dist({"kind": "powerlu", "a": a, "k": 12, "q_os": 8, "v": 5, "seed": 2}, world=4)
    ref = O.powerlu(a, 12, 8, 5, 2)
    for rank, (p, q, L, U, passes) in res.items():
        assert np.array_equal(p, ref.p) and np.array_equal(q, ref.q)
        f = O.LowRankLU(p, q, L, U, 12)
        assert abs(O.rel_fro_error_factor(a, f) - O.rel_fro_error_factor(a, ref)) <= 1e-12


@pytest.mark.parametrize("world,panel,q_os", [(2, 7, 10), (3, 64, 5)])
def test_sharded_single_pass_matches_single_process(world, panel, q_os):
    """C4's path (rlra/singlepass.py:99-144) row-sharded: per-panel all-reduce
    of the partial G_J (asynchronous, overlapping the next panel), local H_i,
    gathered exact GEPP of H: same p, q as one process; error equal to 1e-12."""
    rng = np.random.default_rng(40 + world)
    x, _ = np.linalg.qr(rng.standard_normal((211, 30)))
    y, _ = np.linalg.qr(rng.standard_normal((130, 30)))
    a = np.asfortranarray((x * np.arange(1, 31) ** -1.5) @ y.T + 1e-6 * rng.standard_normal((211, 130)))
    k = 12
    res = run_dist({"kind": "single_pass", "a": a, "k": k, "q_os": q_os, "seed": 3, "panel": panel}, world=world)
    ref = O.single_pass_lu(a, k, 3, q_os=q_os, panel=panel)
    e_ref = O.rel_fro_error_factor(a, ref)
    for rank, (p, q, L, U, sweeps) in res.items():
        assert np.array_equal(p, ref.p) and np.array_equal(q, ref.q)
        assert abs(O.rel_fro_error_factor(a, O.LowRankLU(p, q, L, U, k)) - e_ref) <= 1e-12
        assert sweeps == -(-130 // panel)  # one all-reduce per panel, each column read once
    np.testing.assert_array_equal(res[0][2], res[1][2])


def test_reference_signatures_accept_a_sharded_matrix():
    """the multi-GPU path behind the drop-in API."""
    a = decay_matrix(190, 140, seed=13)
    res = run_dist({"kind": "api", "a": a, "k": 18, "q_os": 6, "v": 4, "seed": 2})
    ref = O.powerlu(a, 18, 6, 4, 2)
    ref_fp, ref_o = O.powerlu_fp(a, 1e-3, 5, 60, 4, 0)
    ref_sp = O.single_pass_lu(a, 18, 2, q_os=4, panel=16)
    ref_v = O.general_power_basis_v(a, 20, 3, 1)
    for rank, (f, r, gshape, fp, sp, v, passes) in res.items():
        assert np.array_equal(f[0], ref.p) and np.array_equal(f[1], ref.q)
        assert r == ref_o.rank and gshape[1] == r
        assert np.array_equal(fp[0], ref_fp.p) and np.array_equal(fp[1], ref_fp.q)
        assert np.array_equal(sp[0], ref_sp.p) and np.array_equal(sp[1], ref_sp.q)
        assert passes == ref_v.passes_used
        # same basis up to column signs
        assert np.allclose(np.abs(np.sum(v * ref_v.V, axis=0)), 1.0, atol=1e-10)


@pytest.mark.parametrize("v,decline,wide_at", [(5, False, 16), (4, True, 10 ** 9)])
def test_sharded_replicated_factorizations_world4(v, decline, wide_at):
    """the n x l sketch factorizations on row blocks of the
    replicated Z (sharded CholeskyQR2 with all-reduced Grams, TSQR when the
    Cholesky declines, tournament LU for the interior n x l LU) and L = L1 U2^T
    by row blocks (full_L all-gathers): p, q identical, error equal to 1e-12."""
    a = decay_matrix(400, 240, seed=20 + v)
    res = run_dist({"kind": "powerlu", "a": a, "k": 20, "q_os": 8, "v": v, "seed": 5, "decline": decline,
                    "wide_at": wide_at}, world=4)
    ref = O.powerlu(a, 20, 8, v, 5)
    e_ref = O.rel_fro_error_factor(a, ref)
    for rank, (p, q, L, U, passes) in res.items():
        assert np.array_equal(p, ref.p) and np.array_equal(q, ref.q), rank
        assert abs(O.rel_fro_error_factor(a, O.LowRankLU(p, q, L, U, 20)) - e_ref) <= 1e-12
        np.testing.assert_allclose(L, ref.L, rtol=0, atol=1e-9)


@pytest.mark.parametrize("world,m,n,seed", [(2, 150, 70, 0), (3, 203, 64, 1), (4, 120, 33, 2), (2, 90, 90, 3)])
def test_row_sharded_exact_gepp_is_bit_identical(world, m, n, seed):
    """distributed.dist_getrf_ (gathered panels factored redundantly, rows
    exchanged for the interchanges, U12 from the gathered block rows, local
    updates): pivots and every bit of the packed L\\U equal the reference
    kernel's (rlra/_lu_cython.pyx:14-55), including exact zero pivots across
    block boundaries and tied magnitudes."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((m, n))
    if n > 40:
        a[:, 33] = a[:, 5]  # exact zero pivot after a block boundary
        a[:, 40] = 0.0
    a[7] = -a[3]  # tied magnitudes
    a = np.asfortranarray(a)
    res = run_dist({"kind": "getrf", "a": a}, world=world)
    lu_ref = a.copy(order="F")
    piv_ref = np.arange(m, dtype=np.int64)
    O.plu_inplace(lu_ref, piv_ref)
    full = np.empty_like(lu_ref)
    for rank, (piv, local, urows, cnt, r0, r1) in res.items():
        assert np.array_equal(piv, piv_ref), rank
        full[r0:r1] = local
        np.testing.assert_array_equal(urows.view(np.int64), lu_ref[:min(m, n)].view(np.int64))
        assert cnt == int(np.count_nonzero(np.diag(lu_ref)))
    assert np.array_equal(full.view(np.int64), lu_ref.view(np.int64))
