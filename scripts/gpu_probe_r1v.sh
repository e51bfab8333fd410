python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r1v.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_tests_r1v.log
python scripts/probe_configs.py > gpurun_out/r1v_configs.jsonl 2> gpurun_out/r1v_configs.err
MAPC_OVERLAP=0 python scripts/probe_direct.py 5a 3a 4b > gpurun_out/r1v_seq.jsonl 2>&1
bash scripts/sweep_overlap.sh > gpurun_out/r1v_overlap_sweep.jsonl 2>&1
