timeout 300 python tools/gap_probe.py 3 > gpurun_out/gap_r02.txt 2>&1; echo "gap rc=$?"; head -40 gpurun_out/gap_r02.txt
timeout 600 python bench.py --breakdown --no-c5 --no-cpu-baseline --no-e2e > gpurun_out/bench_bd.json 2> gpurun_out/bench_bd.err; echo "bench rc=$?"; cat gpurun_out/bench_bd.err | head -30
