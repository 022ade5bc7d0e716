timeout 900 python -m pytest tests/test_qr_gpu.py tests/test_configs_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_g7.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g7.log
grep -E "passed|failed|^FAILED|^E  " gpurun_out/pytest_g7.log | head -30
for c in C3 C5; do BREAKDOWN=1 timeout 900 python tools/run_config.py $c 3 > gpurun_out/cfg_$c.log 2>&1; echo "$c rc=$?"; head -12 gpurun_out/cfg_$c.log; tail -1 gpurun_out/cfg_$c.log | cut -c1-300; done
timeout 600 python bench.py --no-c5 --no-cpu-baseline > gpurun_out/bench_g7.json 2> gpurun_out/bench_g7.err; echo "bench rc=$?"; head -c 400 gpurun_out/bench_g7.json
