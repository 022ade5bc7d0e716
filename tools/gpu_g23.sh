timeout 900 python -m pytest tests/test_drivers_gpu.py -q -p no:cacheprovider -k "pipelined or upload or residues_built" 2>&1 | tail -15
timeout 600 python tools/e2e_loop.py 8 2>&1 | tail -3
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe_r02b.txt 2>&1; head -22 gpurun_out/e2e_probe_r02b.txt
