# Round-2 evidence: default bench (C2 + C5 sub-record), reference arm, launch
# list of the same command, ncu full captures of the pass GEMM / residue /
# norms kernels, every config, the scaling model.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
lscpu | head -20 > gpurun_out/lscpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-c5 > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
for k in gemm_i8_kernel:4 residue_a_kernel:1 norms_partial_kernel:1; do
  n=${k%%:*}; s=${k##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$n -s $s -c 1 \
    -o gpurun_out/ncu_$n python tools/run_powerlu.py C2 4 1 > gpurun_out/ncu_$n.log 2>&1; echo "ncu $n rc=$?"
done
bash tools/all_configs.sh
