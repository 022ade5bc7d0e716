timeout 120 python tools/int8_peak.py > gpurun_out/int8_peak.json 2> gpurun_out/int8_peak.err; echo rc=$?; cat gpurun_out/int8_peak.json; tail -3 gpurun_out/int8_peak.err
python -c "import threadpoolctl, numpy; print(threadpoolctl.threadpool_info())"
