timeout 1500 python -m pytest tests/test_streams_gpu.py tests/test_configs_gpu.py tests/test_drivers_gpu.py tests/test_reference_suite_gpu.py -q -p no:cacheprovider -x -k "not C5 and not c5" 2>&1 | tail -4
BREAKDOWN=1 timeout 900 python tools/run_config.py C4 5 > gpurun_out/cfg_C4.log 2>&1; echo "C4 rc=$?"; grep -E "^  " gpurun_out/cfg_C4.log | head -4; tail -1 gpurun_out/cfg_C4.log | cut -c1-330
timeout 600 python tools/oocore_bench.py > gpurun_out/oocore.txt 2>&1; tail -5 gpurun_out/oocore.txt
