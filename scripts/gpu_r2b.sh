set -x
timeout 1500 python -m pytest tests/test_gpu_babycuda.py -q > gpurun_out/r2b_babycuda.log 2>&1; echo bc_rc=$?; tail -30 gpurun_out/r2b_babycuda.log
