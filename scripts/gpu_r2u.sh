timeout 900 python scripts/probe_configs.py 4a 4b 2b --paths=auto > gpurun_out/r2u_configs.jsonl 2>&1; cut -c1-250 gpurun_out/r2u_configs.jsonl
timeout 600 python scripts/probe_direct5a.py > gpurun_out/r2u_5a.jsonl 2>&1; cat gpurun_out/r2u_5a.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gaps.py -q -x -k "direct or jit or full_size or overlap or u32 or fuzz" > gpurun_out/r2u_parity.log 2>&1; echo p_rc=$?; tail -3 gpurun_out/r2u_parity.log
