#!/usr/bin/env python
"""PowerLU FP64 benchmark (BASELINE.json metric) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config C2|C1|C5] [--v 4] [--breakdown] [--no-c5]

--gpus N > 1 outside torchrun re-launches this script under
`torch.distributed.run --nproc-per-node N` (one rank per GPU, NCCL); under
torchrun (WORLD_SIZE set) every rank runs the distributed arm.

One step = one complete factorization of the workload (default C2:
powerlu(A 20000x10000, k=200, q_os=20, v=4, seed=0), BASELINE.json configs[1]).

Our arm prints ONE JSON line with:
  value      algorithmic GFLOP/s (SURVEY.md Appendix B flop count) with A and
             Omega resident in HBM, outputs left in HBM; CUDA events, K steps
  e2e        the same metric through the public API with HOST inputs (pinned
             NumPy A, uploaded in column chunks behind the first pass), Omega
             regenerated every step (device replay of NumPy's stream), factors
             returned to the host as NumPy: H2D/D2H inside the timed region
  roofline   the dominant kernel -- the int8 tensor-core pass GEMM of the
             Ozaki-II emulation (HBM bound) -- achieved GB/s from CUDA events
             on its launch stream vs MEASURED_PEAKS.json, plus its int8-tensor
             fraction and the passes' FP64-equivalent rate vs the DMMA peak
  cpu_baseline  the unmodified reference (oracle/_ref, rlra 0.1.0) on the box's
             host cores, same call, best of a bounded sample
`--impl reference` times the reference's own CPU implementation (oracle/_ref).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

FP64_PEAK_TFLOPS = 37.1  # measured DMMA m8n8k4 sustained, profiles/fp64_peak_r01.log
try:
    MEASURED = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    HBM_PEAK_SRC = "MEASURED_PEAKS.json hbm_gbs (burst copy)"
except (OSError, ValueError):
    MEASURED = {"hbm_gbs": 7700.0, "bf16_tflops": 2250.0}  # B200_PROFILING.md fallback
    HBM_PEAK_SRC = "B200_PROFILING.md fallback (7.7 TB/s nominal; MEASURED_PEAKS.json absent)"
FP64_PEAK_SRC = "measured: tools/fp64_peak.cu on this pool's B200 (profiles/fp64_peak_r01.log); MEASURED_PEAKS.json has no FP64 entry"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--v", type=int, default=None)
    ap.add_argument("--breakdown", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 (262144 x 32768) sub-record")
    ap.add_argument("--no-sweep", action="store_true", help="skip the C2 pass sweep v = 2..6 sub-record")
    ap.add_argument("--c5-steps", type=int, default=2)
    return ap.parse_args()


def workload(args):
    from paper_2002_07138_b200 import configs

    w = configs.WORKLOADS[args.config]
    v = args.v if args.v is not None else w.v
    gen = {"C1": configs.gen_c1, "C2": configs.gen_c2}.get(w.name)  # C3-C5: built in HBM (configs.gen_device)
    if w.kind == "powerlu":
        passes, fact = configs.powerlu_flops(w.m, w.n, w.k, w.k + w.q_os, v)
        desc = f"{w.name}: powerlu(A {w.m}x{w.n} float64, k={w.k}, q_os={w.q_os}, v={v}, seed={w.seed})"
    elif w.kind == "powerlu_fp":
        passes, fact = configs.powerlu_fp_flops(w.m, w.n, FP_WIDTH, v, FP_RANK)
        desc = (f"{w.name}: powerlu_fp(A {w.m}x{w.n} float64, PrecisionParams(eps={w.eps}, b={w.b}, "
                f"l={FP_WIDTH}, v={v}), seed={w.seed}) (flops at the reference's rank {FP_RANK})")
    else:
        passes, fact = configs.single_pass_flops(w.m, w.n, w.k + w.q_os)
        desc = (f"{w.name}: single_pass_lu(DeviceColumnStream(A {w.m}x{w.n} float64), k={w.k}, "
                f"seed={w.seed}, q_os={w.q_os})")
    return w, v, gen, passes, fact, desc


def configs_flops(w, v):
    from paper_2002_07138_b200 import configs

    return configs.powerlu_flops(w.m, w.n, w.k, w.k + w.q_os, v)


FP_WIDTH, FP_RANK = 1024, 843  # C3: sketch width and the reference's chosen rank (tests/golden/golden_configs.json)


def single_runner(w, v, dm):
    """The drop-in call of config w on one GPU (DeviceMatrix operand)."""
    import paper_2002_07138_b200 as P

    if w.kind == "powerlu":
        return lambda: P.powerlu(dm, w.k, w.q_os, v, w.seed)
    if w.kind == "powerlu_fp":
        return lambda: P.powerlu_fp(dm, P.PrecisionParams(w.eps, w.b, FP_WIDTH, v), w.seed)[0]
    return lambda: P.single_pass_lu(P.DeviceColumnStream(dm), w.k, w.seed, q_os=w.q_os)


def dist_runner(w, v, A, omega):
    """The same call over a row-sharded A (distributed.py)."""
    from paper_2002_07138_b200 import distributed as D

    if w.kind == "powerlu":
        return lambda: D.powerlu(A, w.k, w.q_os, v, w.seed, omega)
    if w.kind == "powerlu_fp":
        return lambda: D.powerlu_fp(A, w.eps, w.b, FP_WIDTH, v, w.seed, omega)[0]
    return lambda: D.single_pass_lu(A, w.k, w.seed, omega, q_os=w.q_os)


def ref_module():
    """The unmodified reference (oracle/_ref), else the oracle port."""
    ref = os.path.join(REPO, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref, "rlra")):
        sys.path.insert(0, ref)
        os.environ.setdefault("RLRA_BACKEND", "compiled")
        import rlra

        return rlra, "reference"
    from oracle import rlra_oracle

    return rlra_oracle, "port"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md recipe)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


KTIMERS = ("oz_gemm_i8", "oz_residue_a", "oz_norms", "oz_crt", "oz_residue_b")


def _ktimer_read(lib, name):
    import ctypes

    ms, cnt = ctypes.c_double(0.0), ctypes.c_longlong(0)
    rc = lib.rlra_b200_ktimer_read(name.encode(), ctypes.byref(ms), ctypes.byref(cnt))
    if rc != 0:
        raise RuntimeError(lib.rlra_b200_last_error().decode())
    return ms.value, cnt.value


def _ktimer_reset(lib):
    for nm in KTIMERS:
        _ktimer_read(lib, nm)


def roofline_line(w, v, passes, reps, kt, pass_ms, step_ms):
    """Roofline of the dominant kernel, the int8 tensor-core pass GEMM
    (csrc/ozaki.cu gemm_i8_kernel), from CUDA events recorded on its launch
    stream around every launch of `reps` profiled factorizations.

    Algorithmic bytes per pass of width w: the residues of
    A (nmod bytes per element, read once), the residues of the skinny operand
    (nmod * K * w) and the residue output (nmod * rows * w); K + rows = m + n
    for both orientations.  The kernel is HBM bound: its int8 work
    (nmod * 2mnw ops) at the int8 tensor peak takes less time than its bytes
    at the HBM peak."""
    from paper_2002_07138_b200 import ops

    nmod = ops.OZ_NMOD
    if w.kind == "single_pass":  # two products per sweep panel (TN then NN), K or rows = m
        from paper_2002_07138_b200.singlepass import sweep_width

        l_ = w.k + w.q_os
        sw = sweep_width(w.m, 256)
        panels = [min(sw, w.n - j0) for j0 in range(0, w.n, sw)]
        bytes_step = sum(2 * nmod * (w.m * x + (w.m + x) * l_) for x in panels)
        fp64_bytes_step = sum(2 * 8 * (w.m * x + (w.m + x) * l_) for x in panels)
        i8ops_step = sum(2 * nmod * 2.0 * w.m * x * l_ for x in panels)
    else:
        l_ = FP_WIDTH if w.kind == "powerlu_fp" else w.k + w.q_os
        widths = [l_] * v if w.kind == "powerlu_fp" else [l_] * (v - 1) + [w.k]
        bytes_step = sum(nmod * (w.m * w.n + (w.m + w.n) * x) for x in widths)
        fp64_bytes_step = sum(8 * (w.m * w.n + (w.m + w.n) * x) for x in widths)
        i8ops_step = sum(nmod * 2.0 * w.m * w.n * x for x in widths)
    g_ms, g_cnt = kt["oz_gemm_i8"]
    hbm_peak = MEASURED.get("hbm_gbs")
    if g_cnt == 0:  # DMMA pass (RLRA_B200_PASS_GEMM=dmma or operands too large for the residues)
        achieved = passes * reps / (pass_ms / 1e3) / 1e12 if pass_ms else None
        return {"bound": "tensor", "kernel": "dgemm_tma_kernel (FP64 DMMA pass products)", "achieved": achieved,
                "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS if achieved else None, "traffic": None,
                "peak_source": FP64_PEAK_SRC, "pass_ms_per_step": pass_ms / reps}
    per_launch_bytes = bytes_step * reps / g_cnt
    per_launch_ms = g_ms / g_cnt
    achieved = per_launch_bytes / (per_launch_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(REPO, "profiles", "ncu_pass_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"oz_gemm_i8_{w.name}_v{v}")
        except Exception:
            traffic = None
    i8_peak, i8_src = 2.0 * MEASURED.get("bf16_tflops", 1690.0), "2 x MEASURED_PEAKS.json bf16_tflops (assumed)"
    try:  # measured on this pool's B200 (tools/int8_peak.py, cuBLASLt int8 8192^3)
        i8 = json.load(open(os.path.join(REPO, "profiles", "r02_int8_peak.json")))
        i8_peak, i8_src = float(i8["int8_tops_burst"]), "profiles/r02_int8_peak.json (torch._int_mm burst, measured)"
    except (OSError, ValueError, KeyError):
        pass
    fp64_eq = passes * reps / (pass_ms / 1e3) / 1e12 if pass_ms else None
    other = {nm: {"ms_per_step": t / reps, "launches_per_step": c / reps} for nm, (t, c) in kt.items()}
    return {"bound": "hbm", "kernel": "gemm_i8_kernel (tcgen05 kind::i8 Ozaki-II pass products, csrc/ozaki.cu)",
            "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
            "traffic": traffic, "peak_source": HBM_PEAK_SRC,
            "algorithmic_bytes_per_launch": per_launch_bytes, "ms_per_launch": per_launch_ms,
            "launches_per_step": g_cnt / reps,
            "bytes_per_unit": f"nmod*(m*n + (m+n)*w) per pass of width w, nmod={nmod}",
            "int8_tensor": {"achieved_tops": i8ops_step * reps / (g_ms / 1e3) / 1e12, "peak_tops": i8_peak,
                            "frac": i8ops_step * reps / (g_ms / 1e3) / 1e12 / i8_peak, "peak_source": i8_src},
            "fp64_bytes_view": {
                "algorithmic_bytes_per_launch": fp64_bytes_step * reps / g_cnt,
                "achieved_gbs": fp64_bytes_step * reps / g_cnt / (per_launch_ms / 1e3) / 1e9,
                "frac": fp64_bytes_step * reps / g_cnt / (per_launch_ms / 1e3) / 1e9 / hbm_peak,
                "note": "the same launches against 8 B per element of A + the FP64 skinny operands "
                        "(the bytes a DGEMM pass would read); the int8 engine must read 14 B/element "
                        "of residues instead, so this view is capped at ~8/14"},
            "kernel_share_of_step": g_ms / reps / step_ms,
            "fp64_equivalent": {"pass_tflops": fp64_eq, "dmma_peak_tflops": FP64_PEAK_TFLOPS,
                                "frac_of_dmma_peak": fp64_eq / FP64_PEAK_TFLOPS if fp64_eq else None,
                                "pass_ms_per_step": pass_ms / reps,
                                "note": "pass products (incl. B residues + CRT) as FP64 flops 2*m*n*w"},
            "other_kernels": other}


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w, v, gen, passes, fact, desc = workload(args)
    mod, kind = ref_module()
    sample = f"{args.steps} full {w.name} factorizations (mean)"
    from paper_2002_07138_b200 import configs

    call = lambda a_: mod.powerlu(a_, w.k, w.q_os, v, w.seed)  # noqa: E731
    steps, warm = args.steps, args.warmup
    if w.name == "C5":  # 68.7 GB: the survey's C5 analogue is the bounded host sample
        a = configs.gen_lowrank_plus_noise(32768, 8192, 640, 10.0 ** (-8.0 * np.arange(640) / 639), 1e-10, 5)
        passes, fact = configs.powerlu_flops(32768, 8192, w.k, w.k + w.q_os, v)
        sample = f"{steps} factorizations of the C5 analogue 32768x8192 (SURVEY Appendix A), mean"
    elif w.name == "C4":  # 20 GB, ~100 s per call on the host: the survey's 20000^2 analogue
        a = configs.gen_lowrank_plus_noise(20000, 20000, 300, np.arange(1, 301) ** -1.5, 1e-6, 4)
        passes, fact = configs.single_pass_flops(20000, 20000, w.k + w.q_os)
        steps, warm = min(steps, 2), min(warm, 1)
        call = lambda a_: mod.single_pass_lu(mod.DenseColumnStream(a_), w.k, w.seed, q_os=w.q_os)  # noqa: E731
        sample = f"{steps} single_pass_lu of the C4 analogue 20000x20000 (SURVEY Appendix A), mean"
    elif w.name == "C3":  # ~37 s per call on the host: one warm-up-free sample
        a = configs.gen_c3()
        steps, warm = min(steps, 2), 0
        call = lambda a_: mod.powerlu_fp(a_, mod.PrecisionParams(w.eps, w.b, FP_WIDTH, v), w.seed)  # noqa: E731
        sample = f"{steps} full C3 powerlu_fp calls (mean)"
    else:
        a = gen()
    flops = passes + fact
    for _ in range(warm):
        call(a)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        call(a)
        times.append(time.perf_counter() - t0)
    sec = sum(times) / len(times)
    val = flops / sec / 1e9
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": f"PowerLU FP64 GFLOP/s ({w.name}, v={v})", "value": val,
        "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": sec * 1e3, "s_per_factorization": sec, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "m": w.m, "n": w.n, "k": w.k, "l": w.k + w.q_os, "v": v},
        "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": cores, "kind": kind,
                         "sample": f"{sample}, rlra {getattr(mod, '__version__', 'port')} "
                                   f"backend={getattr(mod, 'BACKEND', 'c-oracle')}, OpenBLAS threads=all",
                         "host": host_details()},
        "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def host_details():
    """CPU model and BLAS build of the box."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = None
    try:
        import threadpoolctl

        info = [d for d in threadpoolctl.threadpool_info() if d.get("user_api") == "blas"]
        if info:
            blas = f"{info[0].get('internal_api')} {info[0].get('version')} ({info[0].get('architecture')}, " \
                   f"{info[0].get('num_threads')} threads)"
    except Exception:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "blas": blas}


def cpu_baseline(a, w, v, flops, budget_s=30.0):
    mod, kind = ref_module()
    times, f = [], None
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        f = mod.powerlu(a, w.k, w.q_os, v, w.seed)
        times.append(time.perf_counter() - t0)
        if len(times) >= 3 or time.perf_counter() - t_start + times[-1] > budget_s:
            break
    best = min(times)
    return {"value": flops / best / 1e9, "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": kind,
            "sample": f"{len(times)} full {w.name} factorizations (best of), same A and seed; "
                      f"s/factorization {best:.3f}", "host": host_details()}, f


def cpu_baseline_analogue(w, v):
    """Bounded CPU sample for the device-built configs: the reference on the
    survey's host-feasible analogues -- C5: 32768 x 8192,
    same k, q_os, v and spectrum recipe; C4: 20000 x 20000 single pass, same
    widths; C3: the full C3 (one call) -- GFLOP/s of the same algorithm."""
    from paper_2002_07138_b200 import configs

    mod, kind = ref_module()
    if w.name == "C3":
        m, n = w.m, w.n
        a = configs.gen_c3()
        p_, f_ = configs.powerlu_fp_flops(m, n, FP_WIDTH, v, FP_RANK)
        call = lambda: mod.powerlu_fp(a, mod.PrecisionParams(w.eps, w.b, FP_WIDTH, v), w.seed)  # noqa: E731
    elif w.name == "C4":
        m, n = 20000, 20000
        a = configs.gen_lowrank_plus_noise(m, n, 300, np.arange(1, 301) ** -1.5, 1e-6, 4)
        p_, f_ = configs.single_pass_flops(m, n, w.k + w.q_os)
        call = lambda: mod.single_pass_lu(mod.DenseColumnStream(a), w.k, w.seed, q_os=w.q_os)  # noqa: E731
    else:
        m, n = 32768, 8192
        a = configs.gen_lowrank_plus_noise(m, n, 640, 10.0 ** (-8.0 * np.arange(640) / 639), 1e-10, 5)
        p_, f_ = configs.powerlu_flops(m, n, w.k, w.k + w.q_os, v)
        call = lambda: mod.powerlu(a, w.k, w.q_os, v, w.seed)  # noqa: E731
    t0 = time.perf_counter()
    call()
    sec = time.perf_counter() - t0
    return {"value": (p_ + f_) / sec / 1e9, "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": kind,
            "sample": f"1 call on the {w.name} analogue {m}x{n} (SURVEY Appendix A), {sec:.1f} s", "host": host_details()}


GOLDEN = os.path.join(REPO, "tests", "golden")


def pass_sweep(w, dm, st):
    """C2 over v = 2..6 (BASELINE configs[1]): 3 warm-up + 5 timed factorizations
    per v (CUDA events), pivots against the reference's goldens."""
    import torch

    out = {}
    for vv in (2, 3, 4, 5, 6):
        rv = single_runner(w, vv, dm)
        for _ in range(3):
            fv = rv()
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(st)
        for _ in range(5):
            fv = rv()
        s1.record(st)
        torch.cuda.synchronize()
        ms_v = s0.elapsed_time(s1) / 5
        pv, fa = configs_flops(w, vv)
        fvn = fv.to_numpy()
        out[f"v{vv}"] = dict({"ms_per_step": ms_v, "gflops": (pv + fa) / (ms_v / 1e3) / 1e9},
                             **(pq_parity("C2", vv, fvn.p, fvn.q) or {}))
        del rv, fv, fvn
    return out


def golden_pq(name, v):
    """Reference pivots of a config (tests/golden/*_pq.npz, written by the
    unmodified reference; SURVEY.md Appendix A recipes), or None."""
    try:
        if name == "C2":
            d = np.load(os.path.join(GOLDEN, "c2_pq.npz"))
            return d[f"v{v}_p"], d[f"v{v}_q"]
        from paper_2002_07138_b200 import configs

        if name in ("C1", "C3", "C4", "C5") and v == configs.WORKLOADS[name].v:
            d = np.load(os.path.join(GOLDEN, f"{name.lower()}_pq.npz"))
            return d["p"], d["q"]
    except (OSError, KeyError):
        return None
    return None


def pq_parity(name, v, p, q):
    g = golden_pq(name, v)
    if g is None:
        return None
    return {"p_identical_to_reference": bool(np.array_equal(np.asarray(p), g[0])),
            "q_identical_to_reference": bool(np.array_equal(np.asarray(q), g[1])),
            "golden": f"tests/golden/{name.lower()}_pq.npz"}


def config_record(name, steps=3):
    """One more BASELINE config on this GPU, device-built input (configs.gen_device):
    C3 = powerlu_fp (16384^2, rank 843), C4 = single-pass LU (50000^2).  One
    warm-up, `steps` timed calls (CUDA events), pivots (and C3's rank) against
    the reference's goldens (tests/golden/c3_pq.npz, c4_pq.npz)."""
    import torch

    import paper_2002_07138_b200 as P
    from paper_2002_07138_b200 import configs, core

    w = configs.WORKLOADS[name]
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    core.set_omega_cache(True)
    t0 = time.perf_counter()
    dm = P.DeviceMatrix(configs.gen_device(name, dev))
    torch.cuda.empty_cache()
    gen_s = time.perf_counter() - t0
    rank = None
    if w.kind == "powerlu_fp":
        call = lambda: P.powerlu_fp(dm, P.PrecisionParams(w.eps, w.b, FP_WIDTH, w.v), w.seed)  # noqa: E731
    else:
        call = lambda: (P.single_pass_lu(P.DeviceColumnStream(dm), w.k, w.seed, q_os=w.q_os), None)  # noqa: E731
    f, out = call()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        f, out = call()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if out is not None:
        rank = int(out.rank)
    rec = {"workload": f"{name}: {w.kind} (A {w.m}x{w.n} float64, device-built)", "ms_per_step": ms, "steps": steps,
           "warmup": 1, "input_build_s": gen_s, "parity": pq_parity(name, w.v, f.p.cpu().numpy(), f.q.cpu().numpy())}
    if rank is not None:
        rec["rank"] = rank
        rec["rank_reference"] = FP_RANK
    del dm, f, out, call
    core.set_omega_cache(False)
    torch.cuda.empty_cache()
    return rec


def c5_record(args, dist_ctx=None):
    """The north-star config on the same N GPUs: C5 = powerlu(A 262144 x 32768
    (68.7 GB, built in HBM by configs.gen_device), k=512, q_os=32, v=4).  One
    warm-up, then `--c5-steps` timed factorizations (CUDA events; max over
    ranks), pivots checked against the reference's (tests/golden/c5_pq.npz).
    dist_ctx: (rank, world, local) under torchrun, else None (one GPU)."""
    import torch

    from paper_2002_07138_b200 import configs, core

    w = configs.WORKLOADS["C5"]
    passes, fact = configs.powerlu_flops(w.m, w.n, w.k, w.k + w.q_os, w.v)
    flops = passes + fact
    local = dist_ctx[2] if dist_ctx else int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    core.set_omega_cache(True)
    t0 = time.perf_counter()
    if dist_ctx is None:
        import paper_2002_07138_b200 as P

        A = P.DeviceMatrix(configs.gen_device("C5", dev), local)
        torch.cuda.empty_cache()  # the generator's temporaries: the residue cache is sized from the free HBM
        run = lambda: P.powerlu(A, w.k, w.q_os, w.v, w.seed)  # noqa: E731
    else:
        import torch.distributed as dist

        from paper_2002_07138_b200 import distributed as D

        rank, world, _ = dist_ctx
        r0, r1 = D.row_range(w.m, world, rank)
        full = configs.gen_device("C5", dev)
        shard = D.CudaOps(dev).empty(r1 - r0, w.n)
        shard.copy_(full[r0:r1])
        del full
        torch.cuda.empty_cache()
        A = D.ShardedMatrix(shard, w.m, r0, r1, D.CudaOps(dev))
        om = lambda seed, rows, l: core.omega(seed, rows, l, dev)  # noqa: E731
        run = lambda: D.powerlu(A, w.k, w.q_os, w.v, w.seed, om)  # noqa: E731
    gen_s = time.perf_counter() - t0
    f = run()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist_ctx is not None:
        torch.distributed.barrier()
    e0.record(st)
    for _ in range(max(1, args.c5_steps)):
        f = run()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / max(1, args.c5_steps)
    if dist_ctx is not None:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    p = f.p.cpu().numpy() if hasattr(f.p, "cpu") else f.p
    q = f.q.cpu().numpy() if hasattr(f.q, "cpu") else f.q
    rec = {"workload": "C5: powerlu(A 262144x32768 float64 (68.7 GB, device-built), k=512, q_os=32, v=4, seed=0)",
           "ms_per_step": ms, "gflops": flops / (ms / 1e3) / 1e9, "steps": max(1, args.c5_steps), "warmup": 1,
           "algorithmic_gflop": flops / 1e9, "input_build_s": gen_s,
           "parity": pq_parity("C5", 4, p, q)}
    from paper_2002_07138_b200 import ops as _ops

    if dist_ctx is None and _ops.OzBlocked.last_stats is not None:
        # 120 GB of residues next to the 68.7 GB A: the blocks that do not fit are rebuilt per product
        rec["residue_blocks"] = dict(_ops.OzBlocked.last_stats)
    del A, f, run
    core.set_omega_cache(False)
    torch.cuda.empty_cache()
    return rec


def our_arm(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or os.environ.get("RLRA_B200_BENCH_DIST") == "1":
        return dist_arm(args)
    torch.cuda.set_device(local)
    import paper_2002_07138_b200 as P
    from paper_2002_07138_b200 import _native, ops

    w, v, gen, passes, fact, desc = workload(args)
    flops = passes + fact
    dev = torch.device("cuda", local)
    t0 = time.perf_counter()
    if gen is not None:
        a = gen()
        gen_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        dm = P.DeviceMatrix(a, local)
        torch.cuda.synchronize()
        upload_s = time.perf_counter() - t0
    else:  # C3-C5 (2-69 GB): same recipe, built directly in HBM (configs.gen_device)
        from paper_2002_07138_b200 import configs as _cfg

        a = None
        dm = P.DeviceMatrix(_cfg.gen_device(w.name, dev), local)
        gen_s, upload_s = time.perf_counter() - t0, 0.0
        args.no_e2e = True
    run = single_runner(w, v, dm)
    P.set_omega_cache(True)
    st = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()

    # ---- timed region: device-resident inputs and outputs
    lib = _native.load()
    clocks = Clocks(local)
    clocks.start()
    l0 = lib.rlra_b200_launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(args.steps):
        f = run()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    launches = lib.rlra_b200_launch_count() - l0
    clk = clocks.stop()
    value = flops / (ms / 1e3) / 1e9

    # ---- roofline of the dominant kernel, CUDA events per launch on its stream
    reps = max(1, min(args.steps, 3))
    ops.PROF.records.clear()
    ops.PROF.on = True
    _ktimer_reset(lib)
    lib.rlra_b200_ktimer_enable(1)
    for _ in range(reps):
        run()
    torch.cuda.synchronize()
    lib.rlra_b200_ktimer_enable(0)
    kt = {nm: _ktimer_read(lib, nm) for nm in KTIMERS}
    summ = ops.PROF.summary()
    ops.PROF.on = False
    ops.PROF.records.clear()
    pass_ms = sum(summ.get(k, (0.0, 0))[0] for k in ("pass_nn", "pass_tn", "sweep_oz"))
    roofline = roofline_line(w, v, passes, reps, kt, pass_ms, ms)
    # the exact GEPPs: latency-bound (one cluster-wide pivot exchange per column),
    # no HBM / tensor roofline applies; reported with their share of the step
    l_ = w.k + w.q_os
    gepp_cols = (v - 2) * l_ + 2 * w.k  # v - 2 interior sketch LUs of width l, the two final LUs of width k
    if w.kind == "single_pass":
        gepp_cols = 2 * l_  # GEPP of H (m x l) and of T (n x l)
    elif w.kind == "powerlu_fp":
        gepp_cols = (v - 2) * FP_WIDTH + 2 * FP_RANK
    gepp_ms = summ.get("rlra_b200_getrf", (0.0, 0))[0] / reps
    roofline["latency_bound"] = {
        "kernel": "lu_coop_kernel (bit-exact GEPP, csrc/getrf_full.cu)", "ms_per_step": gepp_ms,
        "share_of_step": gepp_ms / ms, "calls_per_step": summ.get("rlra_b200_getrf", (0.0, 0))[1] / reps,
        "us_per_column": 1e3 * gepp_ms / max(1, gepp_cols), "columns_per_step": gepp_cols}
    if args.breakdown:
        for k2, (t, c) in sorted(summ.items(), key=lambda kv: -kv[1][0]):
            print(f"  {k2:32s} {t / reps:9.3f} ms/step  {c / reps:6.1f} calls/step", file=sys.stderr)

    # ---- BASELINE configs[1] is a sweep over the pass budget: v = 2..6 on the same A
    sweep = pass_sweep(w, dm, st) if (w.name == "C2" and w.kind == "powerlu" and not args.no_sweep) else None

    # ---- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        P.set_omega_cache(False)
        pinned = torch.empty((w.n, w.m), dtype=torch.float64, pin_memory=True)
        ah = pinned.numpy().T  # F-ordered m x n view of pinned memory
        ah[...] = a
        for _ in range(max(5, args.warmup)):  # warm-up: pinned result buffers reach their steady-state reuse (the 4th call still allocated, tools/e2e_loop.py)
            fh = P.powerlu(ah, w.k, w.q_os, v, w.seed)
        ksteps = max(1, min(args.steps, 5))
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(torch.cuda.current_stream(dev))
        for _ in range(ksteps):
            fh = P.powerlu(ah, w.k, w.q_os, v, w.seed)
        s1.record(torch.cuda.current_stream(dev))
        torch.cuda.synchronize()
        e2e_ms = s0.elapsed_time(s1) / ksteps
        l_ = w.k + w.q_os
        h2d = a.nbytes  # Omega is drawn on the device from the seed (core.omega)
        d2h = fh.L.nbytes + fh.U.nbytes + fh.p.nbytes + fh.q.nbytes
        e2e = {"value": flops / (e2e_ms / 1e3) / 1e9, "unit": "GFLOP/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": ksteps,
               "path": "paper_2002_07138_b200.powerlu(pinned host ndarray) -> NumPy factors"}
        P.set_omega_cache(True)

    # ---- CPU baseline (reference on the host) + parity of this very call
    cpu = None
    parity = None
    if not args.no_cpu_baseline and a is not None:
        cpu, fref = cpu_baseline(a, w, v, flops)
        from oracle import rlra_oracle as O

        fd = f.to_numpy()
        parity = {"p_identical": bool(np.array_equal(fd.p, fref.p)),
                  "q_identical": bool(np.array_equal(fd.q, fref.q))}
        if w.m * w.n <= 5e8:
            e_gpu = O.rel_fro_error_factor(a, fd)
            e_ref = O.rel_fro_error_factor(a, fref)
            parity.update({"rel_err_gpu": e_gpu, "rel_err_ref": e_ref, "abs_diff": abs(e_gpu - e_ref)})
    elif not args.no_cpu_baseline:
        cpu = cpu_baseline_analogue(w, v)
    fd = f.to_numpy() if hasattr(f, "to_numpy") else f
    gpar = pq_parity(w.name, v, fd.p, fd.q)
    if gpar is not None:
        parity = dict(parity or {}, **gpar)

    others = None
    c5 = None
    if not args.no_c5 and w.name != "C5":
        del dm, f, fd, run
        a = None  # the host copy is no longer needed either
        if e2e is not None:
            del pinned, ah, fh
        P.set_omega_cache(False)
        import gc

        gc.collect()  # C5 needs every free byte: its residue cache is sized from the free HBM
        torch.cuda.empty_cache()
        if w.name == "C2":  # the other single-GPU configs of BASELINE.json, same process, same GPU
            others = {}
            for nm in ("C3", "C4"):
                try:
                    others[nm] = config_record(nm)
                except Exception as exc:
                    others[nm] = {"error": f"{type(exc).__name__}: {exc}"}
                gc.collect()
                torch.cuda.empty_cache()
        try:
            c5 = c5_record(args)
        except Exception as exc:  # the sub-record must never cost the headline line
            c5 = {"error": f"{type(exc).__name__}: {exc}"}

    line = {
        "metric": f"PowerLU FP64 GFLOP/s ({w.name}, v={v})", "value": value, "unit": "GFLOP/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "s_per_factorization": ms / 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "m": w.m, "n": w.n, "k": w.k, "l": w.k + w.q_os, "v": v,
                   "algorithmic_gflop": flops / 1e9, "pass_gflop": passes / 1e9,
                   "l2": f"inputs larger than L2 (A = {8 * w.m * w.n / 1e9:.2f} GB > 126 MB L2)",
                   "omega": "device replay of NumPy's PCG64 + ziggurat stream (bit-exact rlra.core.gaussian); "
                            "cached across steps for value, redrawn every step for e2e",
                   "parallelism": "single GPU"},
        "gpu_launches": int(launches), "gpu_launches_per_step": launches / args.steps,
        "clocks": clk, "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu, "parity": parity,
        "host_prep": {"generate_A_s": gen_s, "upload_A_s": upload_s},
        "comm": None, "pass_sweep": sweep, "other_configs": others, "C5": c5,
    }
    print(json.dumps(line), flush=True)
    return 0


def dist_arm(args):
    """N GPUs under torchrun: A row-sharded (one shard per rank, NCCL over
    NVLink; paper_2002_07138_b200/distributed.py), the same workload and
    metric as N=1 (strong scaling).  value: device-resident shards, max over
    ranks of the CUDA-event time; e2e: every step uploads each rank's shard
    from pinned host memory and rank 0 downloads the factors."""
    import torch
    import torch.distributed as dist

    from paper_2002_07138_b200 import _native, configs, core, ops
    from paper_2002_07138_b200 import distributed as D

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29541")
    if os.environ.get("RLRA_B200_BENCH_DRYRUN") == "1":  # launcher test (CPU, gloo): report and leave
        dist.init_process_group("gloo", rank=rank, world_size=world)
        print(json.dumps({"dryrun": True, "arm": "dist", "rank": rank, "world": dist.get_world_size()}), flush=True)
        dist.destroy_process_group()
        return 0
    # communicator evidence: NCCL's init lines (rank r nranks N) on stderr, so
    # stdout keeps exactly one JSON line
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    comm = {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
            "nccl_version": ".".join(str(x) for x in torch.cuda.nccl.version())}
    w, v, gen, passes, fact, desc = workload(args)
    flops = passes + fact
    r0, r1 = D.row_range(w.m, world, rank)
    cops = D.CudaOps(dev)
    host_shard = None
    if gen is not None:
        a = gen()
        host_shard = torch.empty((w.n, r1 - r0), dtype=torch.float64, pin_memory=True)  # column-major shard
        host_shard.numpy().T[...] = a[r0:r1]
        del a
        shard = cops.empty(r1 - r0, w.n)
        shard.copy_(host_shard.t())
    else:  # C5: built in HBM, this rank keeps its rows
        full = configs.gen_device(w.name, dev)
        shard = cops.empty(r1 - r0, w.n)
        shard.copy_(full[r0:r1])
        del full
        torch.cuda.empty_cache()
    A = D.ShardedMatrix(shard, w.m, r0, r1, cops)
    core.set_omega_cache(True)
    omega = lambda seed, rows, l: core.omega(seed, rows, l, dev)  # noqa: E731
    run = dist_runner(w, v, A, omega)
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()
    dist.barrier()
    lib = _native.load()
    clocks = Clocks(local)
    clocks.start()
    l0 = lib.rlra_b200_launch_count()
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dist.barrier()
    e0.record(st)
    for _ in range(args.steps):
        run()
    e1.record(st)
    torch.cuda.synchronize()
    dist.barrier()
    launches = lib.rlra_b200_launch_count() - l0
    clk = clocks.stop()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    nl = torch.tensor([float(launches)], device=dev)
    dist.all_reduce(nl, op=dist.ReduceOp.SUM)
    clks = [None] * world
    dist.all_gather_object(clks, clk)

    e2e = None
    if host_shard is not None and not args.no_e2e:
        ksteps = max(1, min(args.steps, 5))
        d2h = 0

        core.set_omega_cache(False)  # as at N=1: Omega is redrawn every e2e step

        def e2e_step():
            sh = cops.empty(r1 - r0, w.n)
            sh.copy_(host_shard.t(), non_blocking=True)
            f = dist_runner(w, v, D.ShardedMatrix(sh, w.m, r0, r1, cops), omega)()
            big_l = f.full_L()  # row blocks of L -> rank 0 (collective)
            return ops.to_numpy_many([f.p, f.q, big_l, f.U]) if rank == 0 else []

        for _ in range(max(5, args.warmup)):
            e2e_step()
        dist.barrier()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(st)
        for _ in range(ksteps):
            hp = e2e_step()
            d2h = sum(x.nbytes for x in hp)
        s1.record(st)
        torch.cuda.synchronize()
        em = torch.tensor([s0.elapsed_time(s1) / ksteps], device=dev)
        dist.all_reduce(em, op=dist.ReduceOp.MAX)
        e2e_ms = float(em.item())
        e2e = {"value": flops / (e2e_ms / 1e3) / 1e9, "unit": "GFLOP/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(8 * w.m * w.n), "d2h_bytes_per_step": int(d2h), "steps": ksteps,
               "path": "distributed.powerlu over pinned host row shards -> NumPy factors on rank 0"}
        core.set_omega_cache(True)
    fin = run()
    parity = pq_parity(w.name, v, fin.p.cpu().numpy(), fin.q.cpu().numpy()) if rank == 0 else None
    del fin, A, shard, run
    core.set_omega_cache(False)
    torch.cuda.empty_cache()
    c5 = None
    if not args.no_c5 and w.name != "C5":
        try:
            c5 = c5_record(args, (rank, world, local))
        except Exception as exc:
            c5 = {"error": f"{type(exc).__name__}: {exc}"}
    if rank == 0:
        msv = float(ms.item())
        sm = [c.get("sm_mhz") for c in clks if c and c.get("sm_mhz")]
        reasons = sorted({r for c in clks if c for r in c.get("reasons", [])})
        line = {"metric": f"PowerLU FP64 GFLOP/s ({w.name}, v={v})", "value": flops / (msv / 1e3) / 1e9,
                "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": msv, "s_per_factorization": msv / 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": desc, "m": w.m, "n": w.n, "k": w.k, "l": w.k + w.q_os, "v": v,
                           "parallelism": f"A row-sharded over {world} GPUs; NCCL all-reduce of A^T Y, "
                                          f"all-gather for the exact final GEPP, TSLU interior from 4 ranks",
                           "l2": "inputs larger than L2"},
                "gpu_launches": int(nl.item()),
                "clocks": {"sm_mhz": min(sm) if sm else None,
                           "sm_max_mhz": clks[0].get("sm_max_mhz") if clks[0] else None,
                           "reasons": reasons, "per_rank": clks},
                "roofline": None, "e2e": e2e, "cpu_baseline": None, "parity": parity, "comm": comm, "C5": c5,
                "note": "roofline and cpu_baseline are reported by the N=1 run"}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def torchrun_cmd(argv, nproc, port):
    """The driver's multi-GPU launch line for this script (one rank per GPU)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)


def _free_port():
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N`: start N ranks ourselves (same as the driver's torchrun)
        return subprocess.call(torchrun_cmd(sys.argv[1:], args.gpus, _free_port()))
    if os.environ.get("RLRA_B200_BENCH_DRYRUN") == "1" and int(os.environ.get("WORLD_SIZE", "1")) == 1:
        print(json.dumps({"dryrun": True, "arm": "single", "rank": 0, "world": 1}), flush=True)
        return 0
    return our_arm(args)


if __name__ == "__main__":
    sys.exit(main())
