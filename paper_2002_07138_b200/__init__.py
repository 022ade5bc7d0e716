"""B200-native PowerLU hot path (arXiv 2002.07138), drop-in for the reference
package ``rlra``'s PowerLU / PowerLU_FP / single-pass API.

All factorization arithmetic runs in hand-written sm_100a kernels in
librlra_b200.so called through its C ABI (include/rlra_b200.h): the pass
products as FP64 emulated on the int8 tensor cores (tcgen05 kind::i8,
Ozaki scheme II, with a dynamic-range guard that sends inputs outside its
DGEMM-class error bound to the FP64 DMMA GEMM), bit-exact GEPP, CholeskyQR2 /
Householder QR, TRSM, compensated reductions.  There is no CPU fallback:
without the library or a CUDA device every entry point raises
NativeUnavailable.  A ``ShardedMatrix`` (distributed.shard_rows) passed to the
same entry points runs the row-sharded multi-GPU algorithm (NCCL).
"""

from .backend import BACKEND, plu_inplace
from .core import gaussian, set_omega_cache
from .device import (
    DenseColumnStream,
    RlraFileColumnStream,
    DeviceColumnStream,
    DeviceMatrix,
    InstrumentedAccessor,
    SparseDeviceMatrix,
    as_accessor,
)
from .errors import (
    DeviceError,
    IllConditionedSolve,
    IllPosedPseudoinverse,
    NativeUnavailable,
    NotConverged,
    RankCollapse,
    RlraError,
    Unsatisfiable,
)
from .fixedprec import (
    AdaptiveOutcome,
    PrecisionParams,
    adaptive_rank,
    default_width,
    powerlu_fp,
    refine_rank,
    restart_policy,
)
from .fixedrank import (LowRankLU, LowRankSVD, lu_from_projection, powerlu, randlu, randlu_noreorth, randsvd,
                        range_agreement, reconstruct)
from .rangefinder import (PowerParams, RangeBasis, SketchLU, general_power_basis_v, power_basis_lu_l,
                          power_basis_q, power_basis_v)
from .singlepass import SketchPair, single_pass_lu, stream_sketch
from .distributed import ShardedMatrix, shard_rows
from .streams import read_rlra, read_rlra_header, write_rlra

__version__ = "0.1.0"

__all__ = [
    "BACKEND", "AdaptiveOutcome", "DenseColumnStream", "DeviceColumnStream", "DeviceError",
    "DeviceMatrix", "IllConditionedSolve", "IllPosedPseudoinverse", "InstrumentedAccessor",
    "LowRankLU", "NativeUnavailable", "NotConverged", "PrecisionParams", "RangeBasis",
    "RankCollapse", "RlraError", "SketchPair", "Unsatisfiable", "adaptive_rank", "as_accessor",
    "default_width", "gaussian", "general_power_basis_v", "lu_from_projection", "plu_inplace",
    "power_basis_v", "powerlu", "powerlu_fp", "reconstruct", "refine_rank", "restart_policy",
    "set_omega_cache", "single_pass_lu", "stream_sketch",
    # paper's comparison baselines
    "LowRankSVD", "PowerParams", "SketchLU", "power_basis_lu_l", "power_basis_q", "randlu",
    "randlu_noreorth", "randsvd", "range_agreement",
    # out-of-core streams
    "RlraFileColumnStream", "read_rlra", "read_rlra_header", "write_rlra",
    # sparse operands
    "SparseDeviceMatrix",
    # multi-GPU operands
    "ShardedMatrix", "shard_rows",
]
