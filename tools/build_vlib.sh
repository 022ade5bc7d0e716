# Variant build of librlra_b200.so for A/B runs: tools/build_vlib.sh NAME "-DFLAG ..." [file.cu ...]
# Recompiles only the listed sources (default ozaki.cu) with the extra flags, links
# against the regular objects, writes tools/vlib/NAME.so (use with RLRA_B200_LIB=...).
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_2002_07138_b200/csrc
O=$R/paper_2002_07138_b200/_lib/obj
NAME=$1; EXTRA=$2; shift 2 || true
FILES=${@:-ozaki.cu}
mkdir -p $R/tools/vlib/obj_$NAME
F="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr"
OBJS=""
for o in $O/*.o; do
  b=$(basename $o .o)
  if echo " $FILES " | grep -q " $b.cu "; then
    nvcc $F $EXTRA -c $C/$b.cu -o $R/tools/vlib/obj_$NAME/$b.o
    OBJS="$OBJS $R/tools/vlib/obj_$NAME/$b.o"
  else
    OBJS="$OBJS $o"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/tools/vlib/$NAME.so $OBJS -lcudart
echo built tools/vlib/$NAME.so
