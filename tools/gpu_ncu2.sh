# full captures: chol_kernel, a mid-factorization 16-wide cluster GEPP panel
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chol_kernel -s 2 -c 1 \
  -o gpurun_out/chol python tools/run_powerlu.py C2 4 1 > gpurun_out/ncu_chol.log 2>&1; echo "ncu chol rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:lu_panel_cluster_kernel<16" -s 20 -c 1 \
  -o gpurun_out/lu_panel16 python tools/run_powerlu.py C2 4 1 > gpurun_out/ncu_lu16.log 2>&1; echo "ncu lu16 rc=$?"
