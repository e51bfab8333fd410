set -x
timeout 900 python -m pytest tests/test_gpu_babycuda.py tests/test_gpu_guard.py tests/test_gpu_unit.py -q -x > gpurun_out/r2h_tests.log 2>&1; echo t_rc=$?; tail -3 gpurun_out/r2h_tests.log
timeout 900 python scripts/probe_babycuda.py > gpurun_out/r2h_babycuda.jsonl 2>&1; echo pb_rc=$?; cat gpurun_out/r2h_babycuda.jsonl | cut -c1-300
timeout 600 python scripts/probe_configs.py 3a 3b --paths=auto > gpurun_out/r2h_configs.jsonl 2>&1; cut -c1-300 gpurun_out/r2h_configs.jsonl
