timeout 600 python -m pytest tests/test_qr_gpu.py -q -p no:cacheprovider -k "cholesky or scholqr" 2>&1 | tail -3
timeout 1500 python tools/scale_model.py C5 1 2 4 8 > gpurun_out/scale_model_C5.json 2> gpurun_out/scale_model_C5.err; echo "model rc=$?"; cat gpurun_out/scale_model_C5.err | tail -6
timeout 600 python tools/scale_model.py C2 1 2 4 8 > gpurun_out/scale_model_C2.json 2> gpurun_out/scale_model_C2.err; echo "model rc=$?"; tail -5 gpurun_out/scale_model_C2.err
