timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
grep -E "passed|failed|^FAILED|^E  " gpurun_out/pytest_full.log | head -20
for c in C3 C4 C5; do BREAKDOWN=1 timeout 900 python tools/run_config.py $c 3 > gpurun_out/cfg_$c.log 2>&1; echo "$c rc=$?"; head -8 gpurun_out/cfg_$c.log; tail -1 gpurun_out/cfg_$c.log | cut -c1-250; done
