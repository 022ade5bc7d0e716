timeout 900 python -m pytest tests/test_ozaki_gpu.py tests/test_guard_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -5
python tools/oz_gemm_time.py > gpurun_out/gemm_new.txt 2>&1; cat gpurun_out/gemm_new.txt
