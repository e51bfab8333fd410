set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r1x.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_tests_r1x.log
python bench.py > gpurun_out/bench_r1x.json 2> gpurun_out/bench_r1x.err; echo bench_rc=$?; cat gpurun_out/bench_r1x.json
python scripts/probe_shard.py 5a > gpurun_out/r1x_shard.jsonl 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1x_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-alt-path > gpurun_out/ncu_ll_r1x.log 2>&1; echo ll_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gen_0|k_direct_scan|k_table_clear" -c 4 -o gpurun_out/r1x_ncu_full python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-alt-path > gpurun_out/ncu_full_r1x.log 2>&1; echo full_rc=$?
