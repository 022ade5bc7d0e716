timeout 1800 python -m pytest tests/test_reference_suite_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_g5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g5.log
tail -80 gpurun_out/pytest_g5.log
