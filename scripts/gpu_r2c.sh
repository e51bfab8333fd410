set -x
timeout 1200 python -m pytest tests/test_gpu_unit.py -q -x > gpurun_out/r2c_unit.log 2>&1; echo unit_rc=$?; tail -20 gpurun_out/r2c_unit.log
timeout 900 python scripts/probe_configs.py > gpurun_out/r2c_configs.jsonl 2> gpurun_out/r2c_configs.err; echo probe_rc=$?; cut -c1-400 gpurun_out/r2c_configs.jsonl; tail -3 gpurun_out/r2c_configs.err
