timeout 1200 python -m pytest tests/test_guard_gpu.py tests/test_ozaki_gpu.py tests/test_drivers_gpu.py tests/test_baselines_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_g3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g3.log
grep -E "passed|failed|^FAILED|^E  " gpurun_out/pytest_g3.log | head -30
