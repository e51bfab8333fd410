set -x
timeout 900 python scripts/probe_configs.py 4a 4b --paths=auto > gpurun_out/r2l_configs.jsonl 2>&1; cut -c1-250 gpurun_out/r2l_configs.jsonl
timeout 900 python scripts/probe_direct5a.py > gpurun_out/r2l_5a.jsonl 2>&1; cat gpurun_out/r2l_5a.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "jit or direct" > gpurun_out/r2l_parity.log 2>&1; echo p_rc=$?; tail -2 gpurun_out/r2l_parity.log
