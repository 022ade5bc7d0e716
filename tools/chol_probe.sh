# Phase-gated builds of the Cholesky kernel for tools/chol_probe.cu:
# tools/exp_chol_{base,NOTRAIL,NODIAG,NOBLKROW,NONEXT}.
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_2002_07138_b200/csrc
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -diag-suppress 177"
V="${VARIANTS:-base NOTRAIL NODIAG NOBLKROW NONEXT}"
mkdir -p $R/tools/vlib
for f in capi gemm gemm_tma getrf getrf_full geqrf misc ozaki rng svd trsm; do
  [ -f $R/tools/vlib/$f.o ] || nvcc $F -c $C/$f.cu -o $R/tools/vlib/$f.o &
done
for v in $V; do
  d=""; [ $v != base ] && d="-DCHOL_EXP_$v"
  nvcc $F $d -c $C/cholqr.cu -o $R/tools/vlib/cholqr_$v.o &
done
wait
O="$(ls $R/tools/vlib/*.o | grep -v cholqr_)"
for v in $V; do
  nvcc $F -o $R/tools/exp_chol_$v $R/tools/chol_probe.cu $R/tools/vlib/cholqr_$v.o $O -lcuda &
done
wait
# trace build: tools/exp_chol_trace (per-iteration globaltimer stamps)
nvcc $F -DCHOL_TRACE -c $C/cholqr.cu -o $R/tools/vlib/cholqr_trace.o
nvcc $F -DCHOL_TRACE -o $R/tools/exp_chol_trace $R/tools/chol_probe.cu $R/tools/vlib/cholqr_trace.o $O -lcuda
