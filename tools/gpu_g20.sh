CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --leak-check no --print-limit 20 python tools/sanitize_probe.py > gpurun_out/sanitize_memcheck.txt 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/sanitize_memcheck.txt
timeout 1500 $CS --tool synccheck --print-limit 20 python tools/sanitize_probe.py > gpurun_out/sanitize_synccheck.txt 2>&1; echo "synccheck rc=$?"; tail -5 gpurun_out/sanitize_synccheck.txt
timeout 2400 $CS --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_probe.py > gpurun_out/sanitize_racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -5 gpurun_out/sanitize_racecheck.txt
