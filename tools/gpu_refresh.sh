# Refresh of the headline evidence after the last kernel changes (profiles/r02b_*).
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-c5 --no-sweep > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 300 python tools/time_getrf.py 20000,220 10000,220 20000,200 10000,200 16384,1024 16384,843 50000,720 32768,544 262144,512 > gpurun_out/time_getrf.txt 2>&1
timeout 60 ./tools/lu_full_trace 10000 220 > gpurun_out/lu_trace.txt 2>&1
bash tools/all_configs.sh
