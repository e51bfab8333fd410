set -x
timeout 1200 python -m pytest tests/test_gpu_unit.py -q -x > gpurun_out/r2m_unit.log 2>&1; echo u_rc=$?; tail -30 gpurun_out/r2m_unit.log | head -60
timeout 900 python scripts/probe_configs.py 4a 4b 4c 4d 3a 3b --paths=auto > gpurun_out/r2m_configs.jsonl 2>&1; cut -c1-300 gpurun_out/r2m_configs.jsonl
