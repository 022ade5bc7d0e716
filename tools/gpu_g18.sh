timeout 1500 python -m pytest tests/test_configs_gpu.py tests/test_guard_gpu.py -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py --no-c5 --no-cpu-baseline --no-e2e > gpurun_out/bench_g18.json 2> gpurun_out/bench_g18.err; head -c 250 gpurun_out/bench_g18.json
