timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe_r02.txt 2>&1; echo rc=$?; head -60 gpurun_out/e2e_probe_r02.txt
