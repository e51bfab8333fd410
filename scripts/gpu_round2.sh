set -x
bash scripts/box_info.sh > gpurun_out/${TAG:-r2}_box.txt 2>&1
python -m pytest tests -m gpu -q > gpurun_out/${TAG:-r2}_gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/${TAG:-r2}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG:-r2}_smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/${TAG:-r2}_smoke.log
python bench.py > gpurun_out/${TAG:-r2}_bench.json 2> gpurun_out/${TAG:-r2}_bench.err; echo bench_rc=$?; cut -c1-400 gpurun_out/${TAG:-r2}_bench.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG:-r2}_bench_ref.json 2>&1; echo ref_rc=$?; cut -c1-300 gpurun_out/${TAG:-r2}_bench_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG:-r2}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-alt-path --no-other-configs > gpurun_out/${TAG:-r2}_ncu_ll.log 2>&1; echo ll_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gen_0|k_direct_scan|k_table_clear" -c 5 -o gpurun_out/${TAG:-r2}_direct_ncu_full python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-alt-path --no-other-configs > gpurun_out/${TAG:-r2}_ncu_full.log 2>&1; echo full_rc=$?
