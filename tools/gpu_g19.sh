for c in C3 C4; do timeout 600 python tools/timeline.py $c 100 > gpurun_out/timeline_$c.txt 2>&1; echo "$c rc=$?"; grep -A30 "per label" gpurun_out/timeline_$c.txt; done
