timeout 600 python tools/timeline.py C4 100 > gpurun_out/timeline_C4.txt 2>&1; echo "C4 rc=$?"; head -1 gpurun_out/timeline_C4.txt; grep -A12 "per label" gpurun_out/timeline_C4.txt
timeout 1500 python -m pytest tests/test_configs_gpu.py -k "c4" tests/test_drivers_gpu.py tests/test_baselines_gpu.py tests/test_reference_suite_gpu.py -q -p no:cacheprovider 2>&1 | tail -3
