nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_guard_gpu.py tests/test_ozaki_gpu.py tests/test_drivers_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_g1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g1.log
tail -30 gpurun_out/pytest_g1.log
timeout 600 python bench.py --breakdown > gpurun_out/bench_g1.json 2> gpurun_out/bench_g1.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_g1.json
