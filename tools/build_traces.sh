# Trace builds of the GEPP paths (globaltimer stamps): tools/lu_trace (blocked
# cluster panels) and tools/lu_full_trace (one-launch cluster GEPP).
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_2002_07138_b200/csrc
SRC="$C/capi.cu $C/cholqr.cu $C/gemm.cu $C/gemm_tma.cu $C/getrf.cu $C/getrf_full.cu $C/geqrf.cu $C/misc.cu $C/ozaki.cu $C/rng.cu $C/svd.cu $C/trsm.cu"
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -DRLRA_LU_TRACE -diag-suppress 177"
# getrf_full.cu is built twice (256 and 384 threads per CTA, csrc/Makefile)
nvcc $F -DLUF_WIDE_CTA -c $C/getrf_full.cu -o /tmp/getrf_full_wide_trace.o
for t in ${@:-lu_full_trace}; do nvcc $F -o $R/tools/$t $R/tools/$t.cu $SRC /tmp/getrf_full_wide_trace.o; done
