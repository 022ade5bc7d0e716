# Round-1 final evidence: clean bench, reference arm, launch list of the same command, full capture of the top kernel
set -x
timeout 600 python bench.py --breakdown > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_i8_kernel -s 4 -c 1 \
  -o gpurun_out/oz_gemm python tools/run_powerlu.py C2 4 1 > gpurun_out/ncu_full1.log 2>&1; echo "ncu full1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:residue_a_kernel -s 1 -c 1 \
  -o gpurun_out/oz_residue_a python tools/run_powerlu.py C2 4 1 > gpurun_out/ncu_full2.log 2>&1; echo "ncu full2 rc=$?"
