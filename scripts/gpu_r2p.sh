set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "real_nccl" > gpurun_out/r2p_nccl.log 2>&1; echo n_rc=$?; tail -15 gpurun_out/r2p_nccl.log
timeout 900 python -m pytest tests/test_cli.py -q -x > gpurun_out/r2p_cli.log 2>&1; echo c_rc=$?; tail -15 gpurun_out/r2p_cli.log
