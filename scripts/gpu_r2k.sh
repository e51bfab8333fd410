set -x
timeout 900 python scripts/probe_configs.py 4a 4b 4c 4d --paths=auto > gpurun_out/r2k_configs.jsonl 2>&1; echo probe_rc=$?; cut -c1-330 gpurun_out/r2k_configs.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "jit or direct or full_size" > gpurun_out/r2k_parity.log 2>&1; echo p_rc=$?; tail -3 gpurun_out/r2k_parity.log
timeout 900 python -m pytest tests/test_gpu_gaps.py -q -x -k "rank_shards" > gpurun_out/r2k_shards.log 2>&1; echo s_rc=$?; tail -3 gpurun_out/r2k_shards.log
