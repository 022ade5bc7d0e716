timeout 300 python tools/gap_probe.py 3 > gpurun_out/gap_r02.txt 2>&1; echo "gap rc=$?"; head -12 gpurun_out/gap_r02.txt | tail -10
timeout 600 python bench.py --no-c5 --no-cpu-baseline > gpurun_out/bench_g14.json 2> gpurun_out/bench_g14.err; echo "bench rc=$?"; head -c 300 gpurun_out/bench_g14.json; echo
timeout 900 python -m pytest tests/test_guard_gpu.py tests/test_ozaki_gpu.py tests/test_drivers_gpu.py -q -p no:cacheprovider 2>&1 | tail -2
