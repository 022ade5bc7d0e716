"""Command-line front-end on the GPU path: the
reference's `rlra factor` / `rlra adapt` (rlra/cli.py:57-85, 171-270) with
the same arguments, key=value summary lines, exit codes (0 ok, 1 library /
OS / value error, 2 usage, 3 not converged, 4 unsatisfiable) and output files
(`<prefix>.L.rlm`, `.U.rlm`, `.rowperm.txt`, `.colperm.txt`, or the SVD's
`.U.rlm`, `.S.sigma`, `.V.rlm`), plus `--device cuda[:i]` and `--csv FILE`,
which appends one row in the reference's benchmark schema (CSV_HEADER,
rlra/cli.py:24-25: alg, matrix, m, n, k, eps, v, p, seed, rel_err, rank,
passes, wall_ms).

    python -m paper_2002_07138_b200 factor --in A.rlm --alg powerlu --rank 200 --passes 4 --device cuda
    python -m paper_2002_07138_b200 adapt  --in A.rlm --tol 1e-6 --block 64 --l 1024 --passes 3

The matrix is uploaded once (`.rlm` -> HBM; `.mtx` -> the CSR operand), every
factorization runs on the device, and rel_err is the device-scale validation
metric (validate.rel_err_device) for every size -- the reference densifies
only up to DENSE_ERROR_LIMIT entries and prints nan beyond.  wall_ms covers
the factorization call (device-resident input, factors on the device), like
the reference's timer around the library call.
"""

from __future__ import annotations

import argparse
import csv
import os
import sys
import time
from dataclasses import replace

import numpy as np

CSV_HEADER = ["alg", "matrix", "m", "n", "k", "eps", "v", "p", "seed", "rel_err", "rank", "passes", "wall_ms"]
DEFAULT_PANEL = 256  # rlra/singlepass.py:19


def build_parser():
    parser = argparse.ArgumentParser(prog="rlra-b200", description="randomized low-rank factorization on B200")
    sub = parser.add_subparsers(dest="command", required=True)

    f = sub.add_parser("factor", help="fixed-rank factorization of a matrix file")
    f.add_argument("--in", dest="infile", required=True)
    f.add_argument("--alg", required=True, choices=["powerlu", "randlu", "randlu-noreorth", "randsvd", "singlepass"])
    f.add_argument("--rank", type=int, required=True)
    f.add_argument("--oversample", type=int, default=10)
    f.add_argument("--passes", type=int, help="pass budget v (v >= 2)")
    f.add_argument("--power", type=int, help="power exponent p (v = 2p + 2)")
    f.add_argument("--panel", type=int, default=DEFAULT_PANEL)
    f.add_argument("--seed", type=int, default=0)
    f.add_argument("--out-prefix", dest="prefix")
    f.add_argument("--device", default="cuda")
    f.add_argument("--csv", dest="csv_out")
    f.set_defaults(func=cmd_factor, parser=f)

    a = sub.add_parser("adapt", help="fixed-precision factorization")
    a.add_argument("--in", dest="infile", required=True)
    a.add_argument("--tol", type=float, required=True)
    a.add_argument("--block", type=int, default=10)
    a.add_argument("--l", type=int, help="sketch width (default min(50*block, min(m,n)))")
    a.add_argument("--passes", type=int, default=4)
    a.add_argument("--no-restart", action="store_true", help="fail with exit 3 instead of widening the sketch")
    a.add_argument("--seed", type=int, default=0)
    a.add_argument("--out-prefix", dest="prefix")
    a.add_argument("--device", default="cuda")
    a.add_argument("--csv", dest="csv_out")
    a.set_defaults(func=cmd_adapt, parser=a)
    return parser


def main(argv=None):
    from .errors import NotConverged, RlraError, Unsatisfiable

    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except Unsatisfiable as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 4
    except NotConverged as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
    except (RlraError, OSError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


def resolve_budget(parser_error, alg, passes, power):
    """rlra/cli.py:128-148: map --passes / --power to (v, p)."""
    if passes is not None and power is not None:
        parser_error("give exactly one of --passes or --power")
    if alg == "singlepass":
        if passes is not None or power is not None:
            parser_error("singlepass reads the matrix once; no pass budget applies")
        return None, None
    if alg == "powerlu":
        if power is not None:
            return 2 * power + 2, power
        return (passes if passes is not None else 3), None
    if power is not None:
        return 2 * power + 2, power
    if passes is None:
        return 4, 1
    if passes < 2 or passes % 2:
        parser_error(f"--passes {passes} has no exponent equivalent; use even v >= 2")
    return passes, (passes - 2) // 2


def _device(spec):
    import torch

    if not spec.startswith("cuda"):
        raise ValueError(f"--device {spec}: the B200 path runs on cuda devices only (no CPU fallback)")
    dev = torch.device(spec if ":" in spec else "cuda:0")
    torch.cuda.set_device(dev)
    return dev


def _load(path, dev):
    """A file -> (device operand, device dense A or None for sparse)."""
    from . import ops
    from .device import DeviceMatrix, SparseDeviceMatrix
    from .streams import read_rlra

    if path.endswith((".mtx", ".mm")):
        import scipy.io

        return SparseDeviceMatrix(scipy.io.mmread(path), dev.index), None
    a = read_rlra(path)
    t = ops.from_numpy(a, dev)
    return DeviceMatrix(t, dev.index), t


def _rel_err(dense, f, operand):
    from . import ops, validate

    if dense is None:  # sparse: densify on the device for the metric
        dense = ops.from_numpy(np.asarray(operand.to_dense()), operand.device)
    return validate.rel_err_device(dense, f)


def _rel_err_svd(dense, f, operand):
    from . import ops

    if dense is None:
        dense = ops.from_numpy(np.asarray(operand.to_dense()), operand.device)
    u, s, v = (ops.to_numpy(x) if x.dim() == 2 else x.cpu().numpy() for x in (f.U, f.S, f.V))
    a = ops.to_numpy(dense)
    return float(np.linalg.norm(a - (u * s) @ v.T) / np.linalg.norm(a))


def _write_lu(prefix, f):
    from .streams import write_rlra

    f = f.to_numpy() if hasattr(f, "to_numpy") else f
    write_rlra(f"{prefix}.L.rlm", np.asarray(f.L))
    write_rlra(f"{prefix}.U.rlm", np.asarray(f.U))
    np.savetxt(f"{prefix}.rowperm.txt", np.asarray(f.p), fmt="%d")
    np.savetxt(f"{prefix}.colperm.txt", np.asarray(f.q), fmt="%d")


def _write_svd(prefix, f):
    from . import ops
    from .streams import write_rlra

    write_rlra(f"{prefix}.U.rlm", ops.to_numpy(f.U))
    np.savetxt(f"{prefix}.S.sigma", f.S.cpu().numpy(), fmt="%.17g")  # rlra/fileio.py write_sigma: one value per line
    write_rlra(f"{prefix}.V.rlm", ops.to_numpy(f.V))


def _append_csv(path, row):
    new = not os.path.exists(path) or os.path.getsize(path) == 0
    with open(path, "a", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=CSV_HEADER)
        if new:
            w.writeheader()
        w.writerow(row)


def _timed(fn):
    import torch

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, 1e3 * (time.perf_counter() - t0)


def cmd_factor(args):
    import paper_2002_07138_b200 as P

    v, p = resolve_budget(args.parser.error, args.alg, args.passes, args.power)
    dev = _device(args.device)
    if args.alg == "singlepass":
        if args.infile.endswith((".mtx", ".mm")):
            raise ValueError("singlepass streams .rlm files (the Matrix Market stream is not on the GPU path)")
        stream = P.RlraFileColumnStream(args.infile)
        m, n = stream.shape
        fac, wall = _timed(lambda: P.single_pass_lu(stream, args.rank, args.seed, panel=args.panel))
        from . import ops

        dense = ops.from_numpy(P.read_rlra(args.infile), dev)
        rel = _rel_err(dense, fac, None)
        if args.prefix:
            _write_lu(args.prefix, fac)
        print(f"alg=singlepass matrix={args.infile} m={m} n={n} k={args.rank} seed={args.seed} "
              f"columns={stream.columns_pulled} rel_err={rel:.6e} wall_ms={wall:.1f}")
        if args.csv_out:
            _append_csv(args.csv_out, dict(alg="singlepass", matrix=args.infile, m=m, n=n, k=args.rank, eps="",
                                           v=1, p="", seed=args.seed, rel_err=f"{rel:.6e}", rank=args.rank,
                                           passes=1, wall_ms=f"{wall:.1f}"))
        return 0

    operand, dense = _load(args.infile, dev)
    acc = P.InstrumentedAccessor(operand)
    m, n = acc.shape
    if args.alg == "powerlu":
        fac, wall = _timed(lambda: P.powerlu(acc, args.rank, args.oversample, v, args.seed))
    elif args.alg == "randlu":
        fac, wall = _timed(lambda: P.randlu(acc, args.rank, args.oversample, p, args.seed))
    elif args.alg == "randlu-noreorth":
        fac, wall = _timed(lambda: P.randlu_noreorth(acc, args.rank, args.oversample, p, args.seed))
    else:
        fac, wall = _timed(lambda: P.randsvd(acc, args.rank, args.oversample, p, args.seed))
    if isinstance(fac, P.LowRankSVD):
        rel = _rel_err_svd(dense, fac, operand)
        if args.prefix:
            _write_svd(args.prefix, fac)
    else:
        rel = _rel_err(dense, fac, operand)
        if args.prefix:
            _write_lu(args.prefix, fac)
    budget = f"v={v}" if p is None else f"v={v} p={p}"
    print(f"alg={args.alg} matrix={args.infile} m={m} n={n} k={args.rank} {budget} seed={args.seed} "
          f"passes={acc.product_count} rel_err={rel:.6e} wall_ms={wall:.1f}")
    if args.csv_out:
        _append_csv(args.csv_out, dict(alg=args.alg, matrix=args.infile, m=m, n=n, k=args.rank, eps="", v=v,
                                       p="" if p is None else p, seed=args.seed, rel_err=f"{rel:.6e}",
                                       rank=args.rank, passes=acc.product_count, wall_ms=f"{wall:.1f}"))
    return 0


def adapt_loop(acc, params, seed, allow_restart):
    """rlra/cli.py:217-236: powerlu_fp with the retry schedules -- widen on
    NotConverged (restart_policy), narrow to the achieved width on
    RankCollapse; each retry bumps the seed."""
    import paper_2002_07138_b200 as P

    m, n = acc.shape
    cap = min(m, n)
    attempt_seed = seed
    while True:
        try:
            return P.powerlu_fp(acc, params, attempt_seed)
        except P.NotConverged as exc:
            if not allow_restart:
                raise
            params = P.restart_policy(exc.outcome, params, cap)
            attempt_seed += 1
        except P.RankCollapse as exc:
            shrunk = max(params.b, exc.achieved - exc.achieved % params.b)
            if shrunk >= params.l:
                raise
            params = replace(params, l=shrunk)
            cap = shrunk
            attempt_seed += 1


def cmd_adapt(args):
    import paper_2002_07138_b200 as P

    dev = _device(args.device)
    operand, dense = _load(args.infile, dev)
    acc = P.InstrumentedAccessor(operand)
    m, n = acc.shape
    width = args.l if args.l is not None else P.default_width(args.block, m, n)
    params = P.PrecisionParams(eps=args.tol, b=args.block, l=width, v=args.passes)
    (fac, outcome), wall = _timed(lambda: adapt_loop(acc, params, args.seed, not args.no_restart))
    rel = _rel_err(dense, fac, operand)
    if args.prefix:
        _write_lu(args.prefix, fac)
    print(f"matrix={args.infile} m={m} n={n} eps={args.tol:g} v={args.passes} seed={args.seed} "
          f"rank={outcome.rank} residual_energy={outcome.residual_energy:.6e} "
          f"converged={str(outcome.converged).lower()} passes={acc.product_count} rel_err={rel:.6e} "
          f"wall_ms={wall:.1f}")
    if args.csv_out:
        _append_csv(args.csv_out, dict(alg="powerlu_fp", matrix=args.infile, m=m, n=n, k="", eps=f"{args.tol:g}",
                                       v=args.passes, p="", seed=args.seed, rel_err=f"{rel:.6e}",
                                       rank=outcome.rank, passes=acc.product_count, wall_ms=f"{wall:.1f}"))
    return 0


if __name__ == "__main__":  # pragma: no cover
    sys.exit(main())
