# End-of-round evidence: clean bench, reference arm, launch list of the same command,
# full ncu captures of the pass GEMM, the residue kernel and the CRT, all configs.
set -x
timeout 600 python bench.py --breakdown > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
for k in gemm_i8_kernel:4 residue_a_kernel:1 crt_kernel:2; do
  n=${k%%:*}; s=${k##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$n -s $s -c 1 \
    -o gpurun_out/ncu_$n python tools/run_powerlu.py C2 4 1 > gpurun_out/ncu_$n.log 2>&1; echo "ncu $n rc=$?"
done
bash tools/all_configs.sh
