set -x
timeout 900 python -m pytest tests/test_gpu_unit.py tests/test_gpu_gaps.py -q -x > gpurun_out/r2d_tests.log 2>&1; echo t_rc=$?; tail -5 gpurun_out/r2d_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "direct or overlap or jit or full_size" > gpurun_out/r2d_parity.log 2>&1; echo p_rc=$?; tail -5 gpurun_out/r2d_parity.log
timeout 600 python scripts/probe_configs.py 3a 3b --paths=auto,direct > gpurun_out/r2d_configs.jsonl 2>&1; echo probe_rc=$?; cut -c1-300 gpurun_out/r2d_configs.jsonl
timeout 600 python bench.py --no-alt-path --no-cpu-baseline > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err; echo bench_rc=$?; cut -c1-300 gpurun_out/r2d_bench.json; python -c "
import json; d=json.load(open('gpurun_out/r2d_bench.json')); print(d['value'], d['roofline']['frac'], d['roofline'].get('solo'), d['kernels'])"
MAPC_RED_CACHE=0 timeout 600 python bench.py --no-alt-path --no-cpu-baseline --no-e2e > gpurun_out/r2d_bench_norc.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/r2d_bench_norc.json')); print('norc', d['value'], d['roofline']['frac'])"
