# Round-2 final evidence (profiles/r02b_*): default bench (C2 + pass sweep + C5
# sub-record), reference arm, launch list of the same command, ncu full captures
# of the pass GEMM / residue / norms / CRT kernels, the Householder QR and the
# blocked GEPP kernels, every config, GEPP timings, the scaling model.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-c5 --no-sweep > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
for k in gemm_i8_kernel:4 residue_a_kernel:1 norms_partial_kernel:1 crt_kernel:4; do
  n=${k%%:*}; s=${k##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$n -s $s -c 1 \
    -o gpurun_out/ncu_$n python tools/run_powerlu.py C2 4 1 > gpurun_out/ncu_$n.log 2>&1; echo "ncu $n rc=$?"
done
# Householder QR (fallback path) kernels at the C3 sketch shape: launch list + the top kernel
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_geqrf.csv \
  python tools/qr_bench.py 16384 1024 > gpurun_out/ncu_geqrf_list.log 2>&1; echo "ncu geqrf list rc=$?"
# blocked GEPP (the path ncu can replay) at the C3 sketch shape: launch list
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_getrf.csv \
  python tools/time_getrf.py 16384,1024 > gpurun_out/ncu_getrf_list.log 2>&1; echo "ncu getrf list rc=$?"
timeout 300 python tools/time_getrf.py 20000,220 10000,220 20000,200 10000,200 16384,1024 16384,843 50000,720 32768,544 262144,512 > gpurun_out/time_getrf.txt 2>&1
timeout 300 python tools/oz_gemm_time.py > gpurun_out/oz_gemm_time.txt 2>&1
bash tools/all_configs.sh
timeout 1500 python tools/scale_model.py C5 > gpurun_out/scale_model_C5.json 2> gpurun_out/scale_model_C5.err; echo "scale rc=$?"
