"""Per-piece timing model of the row-sharded PowerLU at P = 1, 2, 4, 8 GPUs,
measured on ONE B200 ("a model built from measured
per-piece times").

Every compute piece a rank executes in distributed.powerlu is run here at the
size that rank sees at P GPUs (shard A[r0:r1] of the real C5 matrix, built in
HBM; sketches of the real widths) and timed with CUDA events (median of 3).
Collectives are modelled from their byte counts: all-reduce 2 (P-1)/P B / bw,
all-gather (P-1)/P B_total / bw, plus a per-call latency; bw and latency are
stated in the output (NVLink 5 / NVSwitch NCCL bus bandwidth, conservative).
The pieces follow distributed.py exactly (v even, fast_qr):

  TN pass  x = A_i^T Omega_i            all-reduce n x l
  LU(x)    replicated exact GEPP n x l  (sharded tournament only when n > 131072)
  NN pass  Y_i = A_i W
  LU(Y)    TSLU: local GEPP (m/P) x l, all-gather P l x l, GEPP P l x l, W_i = Y_i U^-1
           (P = 2 and m <= 131072: all-gather + exact GEPP m x l)
  TN pass  Z = sum A_i^T W_i            all-reduce n x l
  QR(Z)    sharded sCholQR3 on (n/P) x l blocks, all-reduced l x l Grams, all-gather Q
  NN pass  G_i = A_i V_k
  LU(G)    row-sharded exact GEPP (dist_getrf_: gathered 32-column panels factored
           redundantly, local updates), B^T by row blocks and its row-sharded GEPP,
           L_i = L1_i U2^T, L2 all-gathered for U = L2^T

usage: python tools/scale_model.py [C5|C2] [P ...]   -> JSON on stdout
"""

import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_07138_b200 import configs, ops  # noqa: E402
from paper_2002_07138_b200.device import OZ_MAX_RESIDUE_BYTES  # noqa: E402
from paper_2002_07138_b200.distributed import row_range  # noqa: E402

BUS_GBS = 650.0  # NCCL bus bandwidth on NVLink 5 / NVSwitch (B200 datasheet 900 GB/s per direction; conservative)
LAT_MS = 0.025  # per collective call


def allreduce_ms(nbytes, p):
    return 0.0 if p == 1 else 2.0 * (p - 1) / p * nbytes / (BUS_GBS * 1e6) + LAT_MS


def allgather_ms(total_bytes, p):
    return 0.0 if p == 1 else (p - 1) / p * total_bytes / (BUS_GBS * 1e6) + LAT_MS


def timed(fn, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


def rand(m, n, dev):
    return ops.as_fmat(torch.randn((n, m), dtype=torch.float64, device=dev).t())


def gepp_ms(m, n, dev):
    a0 = rand(m, n, dev)

    def run():
        a = ops.fmat(m, n, dev)
        a.copy_(a0)
        ops.getrf_(a)
    return timed(run)


def dist_gepp_ms(m, n, p, dev, host_sync_ms=0.03):
    """Per-rank compute of distributed.dist_getrf_ at P ranks: every 32-column
    block's gathered m x 32 panel factored (getrf_block, redundant), U12 of the
    block rows, the update of this rank's m/P rows; the per-block interchange
    read-back costs host_sync_ms.  Communication is modelled by the caller."""
    from paper_2002_07138_b200.distributed import CudaOps

    cops = CudaOps(dev)
    rows = -(-m // p)
    local = rand(rows, n, dev)
    panel0 = rand(m, 32, dev)
    stt = cops.gepp_state(m, n)

    def run():
        for j0 in range(0, n, 32):
            nbo = min(32, n - j0)
            pan = ops.fmat(m, nbo, dev)
            pan.copy_(panel0[:, :nbo])
            cops.getrf_block(pan, j0, nbo, stt)
            blk = ops.fmat(nbo, n, dev)
            blk.copy_(local[:nbo])
            if j0 + nbo < n:
                cops.lu_trsm_rows(blk, j0, nbo, j0 + nbo, n, stt)
                cops.lu_update_split(local, blk, j0, nbo, 0, j0 + nbo, n, stt)
    t = timed(run, reps=2)
    blocks = -(-n // 32)
    return t + blocks * host_sync_ms


def dist_gepp_comm_ms(m, n, p):
    blocks = -(-n // 32)
    return sum(allgather_ms(8 * m * min(32, n - 32 * b), p) + 2 * allgather_ms(8 * 32 * n * p, p)
               for b in range(blocks))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C5"
    ps = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
    dev = torch.device("cuda", 0)
    w = configs.WORKLOADS[name]
    m, n, k, l = w.m, w.n, w.k, w.k + w.q_os
    a = configs.gen_device(name, dev)
    om = rand(m, l, dev)
    wn = rand(n, l, dev)
    vk = rand(n, k, dev)
    res = {"config": name, "m": m, "n": n, "k": k, "l": l, "bus_gbs": BUS_GBS, "latency_ms": LAT_MS, "P": {}}
    cache = {}

    def gepp(mm, nn):
        if (mm, nn) not in cache:
            cache[(mm, nn)] = gepp_ms(mm, nn, dev)
        return cache[(mm, nn)]

    for p in ps:
        r0, r1 = row_range(m, p, 0)
        rows = r1 - r0
        shard = a[r0:r1]
        piece = {}

        # passes on this rank's shard (residues built once per call, as in ShardedMatrix.products)
        def passes():
            prep = ops.oz_engine(shard, OZ_MAX_RESIDUE_BYTES)
            prep.gemm(om[r0:r1], trans=True)
            y = prep.gemm(wn, trans=False)
            prep.gemm(y[:, :l], trans=True)
            prep.gemm(vk, trans=False)
        piece["passes"] = timed(passes, reps=2)
        piece["allreduce_x_z"] = 2 * allreduce_ms(8 * n * l, p)
        # interior LU of the replicated n x l sketch (exact, redundant)
        piece["lu_nxl"] = gepp(n, l)
        # interior LU of the row-sharded m x l sketch
        if p == 1:
            piece["lu_mxl"] = gepp(m, l)
        elif p >= 4 or m > 131072:
            y = rand(rows, l, dev)
            u = ops.as_fmat(torch.triu(rand(l, l, dev)) + 4 * torch.eye(l, dtype=torch.float64, device=dev))
            piece["lu_mxl_local"] = gepp(rows, l)
            piece["lu_mxl_cand"] = gepp(p * l, l)
            from paper_2002_07138_b200.distributed import CudaOps

            cops = CudaOps(dev)
            piece["lu_mxl_solve"] = timed(lambda: cops.right_solve_upper(y, u))
            piece["allgather_cand"] = allgather_ms(8 * p * l * l, p)
        else:
            piece["allgather_y"] = allgather_ms(8 * m * l, p)
            piece["lu_mxl"] = gepp(m, l)
        # final basis: sCholQR3 (l > one-CTA Cholesky) / CholeskyQR2 on (n/P) x l blocks
        c0, c1 = row_range(n, p, 0)
        zb = rand(c1 - c0, l, dev)
        if p == 1:
            piece["qr_final"] = timed(lambda: ops.scholqr3(zb) if l > ops.cholqr_max_l() else ops.cholqr2(zb))
        else:
            def local_qr():  # the same kernels on the local block (Grams are all-reduced in between)
                steps = [(True, 1e300), (False, 1e7), (False, 2.0)] if l > ops.cholqr_max_l() else \
                    [(False, ops.CHOLQR_COND), (False, 2.0)]
                flag = torch.zeros(1, dtype=torch.int32, device=dev)
                q = zb
                for shifted, limit in steps:
                    g = ops.matmul(q, q, ta=True)
                    if shifted:
                        ops._call("rlra_b200_chol_shift_diag", dev, ops.ptr(g), ops.ld_of(g), l,
                                  ops.SCHOL_C * (n * l + l * (l + 1)), ops._stream(dev))
                    rinv = ops.fmat(l, l, dev)
                    ops.chol_inv_blocked(g, rinv, flag, limit)
                    q = ops.matmul(q, rinv)
            piece["qr_final_local"] = timed(local_qr)
            nsteps = 3 if l > ops.cholqr_max_l() else 2
            piece["allreduce_grams"] = nsteps * allreduce_ms(8 * l * l, p)
            piece["allgather_q"] = allgather_ms(8 * n * l, p)
        # final LUs: row-sharded exact GEPP (distributed.dist_getrf_) of G (m x k)
        # and B^T (n x k); at P = 1 the one-GPU kernel
        if p == 1:
            piece["lu_g"] = gepp(m, k)
            piece["lu_bt"] = gepp(n, k)
        else:
            piece["lu_g_dist"] = dist_gepp_ms(m, k, p, dev)
            piece["lu_g_comm"] = dist_gepp_comm_ms(m, k, p)
            piece["lu_bt_dist"] = dist_gepp_ms(n, k, p, dev)
            piece["lu_bt_comm"] = dist_gepp_comm_ms(n, k, p)
            piece["allgather_l2"] = allgather_ms(8 * n * k, p)
            # the interior m x l LU by the same kernel, for comparison with TSLU (not summed)
            res.setdefault("alt_interior_dist_gepp_ms", {})[str(p)] = dist_gepp_ms(m, l, p, dev) + \
                dist_gepp_comm_ms(m, l, p)
        l1 = rand(rows, k, dev)
        u2 = rand(k, k, dev)
        piece["assemble_l"] = timed(lambda: ops.matmul(l1, u2, tb=True))
        total = sum(v for kk, v in piece.items())
        res["P"][str(p)] = {"pieces_ms": piece, "total_ms": total}
        print(f"P={p}: {total:8.2f} ms  " + "  ".join(f"{kk}={vv:.2f}" for kk, vv in piece.items()), file=sys.stderr,
              flush=True)
    # the real single-GPU call (P.powerlu on the whole A; block-wise residues at C5)
    import paper_2002_07138_b200 as P

    dm = P.DeviceMatrix(a)
    P.set_omega_cache(True)
    P.powerlu(dm, k, w.q_os, w.v, w.seed)
    t1m = timed(lambda: P.powerlu(dm, k, w.q_os, w.v, w.seed), reps=3)
    res["t1_measured_ms"] = t1m
    t1 = res["P"].get("1", {}).get("total_ms")
    for p in ps:
        tp = res["P"][str(p)]["total_ms"]
        if t1:
            res["P"][str(p)]["predicted_efficiency_vs_model_t1"] = t1 / (p * tp)
        res["P"][str(p)]["predicted_efficiency"] = t1m / (p * tp) if p > 1 else t1m / tp
    print(json.dumps(res))


if __name__ == "__main__":
    main()
