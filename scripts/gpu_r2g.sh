set -x
timeout 900 python -m pytest tests/test_gpu_guard.py -q > gpurun_out/r2g_guard.log 2>&1; echo g_rc=$?; tail -5 gpurun_out/r2g_guard.log
timeout 900 python scripts/probe_babycuda.py > gpurun_out/r2g_babycuda.jsonl 2>&1; echo pb_rc=$?; cat gpurun_out/r2g_babycuda.jsonl | cut -c1-400
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_0 -c 2 -o gpurun_out/r2g_unit3a python scripts/probe_configs.py 3a --paths=auto > gpurun_out/r2g_ncu.log 2>&1; echo ncu_rc=$?; tail -3 gpurun_out/r2g_ncu.log
