set -x
timeout 900 python -m pytest tests/test_gpu_unit.py tests/test_gpu_babycuda.py -q -x > gpurun_out/r2f_tests.log 2>&1; echo t_rc=$?; tail -3 gpurun_out/r2f_tests.log
timeout 600 python scripts/probe_configs.py 3a 3b --paths=auto > gpurun_out/r2f_configs.jsonl 2>&1; echo probe_rc=$?; cut -c1-300 gpurun_out/r2f_configs.jsonl
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/r2f_san_$tool.log 2>&1; echo ${tool}_rc=$?; tail -4 gpurun_out/r2f_san_$tool.log
done
