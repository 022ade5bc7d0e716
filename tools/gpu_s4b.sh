for v in epinostore epinomath; do
RLRA_B200_LIB=$PWD/tools/vlib/$v.so python tools/oz_gemm_time.py 20000,10000,220 16384,16384,1024 50000,8192,720 > gpurun_out/gemm_$v.txt 2>&1; echo $v; cat gpurun_out/gemm_$v.txt
done
