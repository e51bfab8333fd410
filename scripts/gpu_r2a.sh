set -x
python -m pytest tests/test_gpu_gaps.py -q > gpurun_out/r2a_gaps.log 2>&1; echo gaps_rc=$?; tail -15 gpurun_out/r2a_gaps.log
python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_gaps.py > gpurun_out/r2a_gpu_tests.log 2>&1; echo tests_rc=$?; tail -5 gpurun_out/r2a_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/r2a_smoke.log
python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo bench_rc=$?; cut -c1-600 gpurun_out/r2a_bench.json
