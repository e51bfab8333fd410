timeout 900 python scripts/probe_configs.py 4a 4b 4c 4d 2b --paths=auto,direct > gpurun_out/r2v_configs.jsonl 2>&1; cut -c1-250 gpurun_out/r2v_configs.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gaps.py -q -x -k "direct or jit or full_size or overlap or u32 or fuzz" > gpurun_out/r2v_parity.log 2>&1; echo p_rc=$?; tail -3 gpurun_out/r2v_parity.log
