set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gen_0|k_direct_scan|k_table_clear" -c 12 -o gpurun_out/r2j_4b python scripts/probe_configs.py 4b --paths=auto > gpurun_out/r2j_ncu4b.log 2>&1; echo ncu_rc=$?; tail -2 gpurun_out/r2j_ncu4b.log
timeout 900 ncu --set full --clock-control none -k regex:"gen_0" -c 6 -o gpurun_out/r2j_4c python scripts/probe_configs.py 4c --paths=auto > gpurun_out/r2j_ncu4c.log 2>&1; echo ncu_rc=$?
