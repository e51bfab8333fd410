timeout 1500 python scripts/fuzz_all_paths.py 4100 5100 > gpurun_out/r2q_fuzz_all_paths.txt 2>&1; tail -3 gpurun_out/r2q_fuzz_all_paths.txt
timeout 900 python scripts/fuzz_all_paths.py 0 150 --big > gpurun_out/r2q_fuzz_all_paths_big.txt 2>&1; tail -3 gpurun_out/r2q_fuzz_all_paths_big.txt
timeout 1500 python scripts/fuzz_executor.py 1000 1600 > gpurun_out/r2q_fuzz_executor.txt 2>&1; tail -3 gpurun_out/r2q_fuzz_executor.txt
