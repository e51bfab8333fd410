# scan-free direct mode A/B (MAPC_DIRECT_ATOM), then its parity
for cfg in "MAPC_X=0" "MAPC_DIRECT_ATOM=1" "MAPC_X=0" "MAPC_DIRECT_ATOM=1"; do
  env $cfg timeout 300 python scripts/probe_direct5a.py 2>&1 | tail -1
done > gpurun_out/r2s_atom_ab.jsonl
cat gpurun_out/r2s_atom_ab.jsonl
MAPC_DIRECT_ATOM=1 timeout 900 python scripts/probe_configs.py 4a 4b 4c 4d --paths=auto,direct > gpurun_out/r2s_configs_atom.jsonl 2>&1; cut -c1-250 gpurun_out/r2s_configs_atom.jsonl
MAPC_DIRECT_ATOM=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "direct or jit or full_size or overlap" > gpurun_out/r2s_parity.log 2>&1; echo p_rc=$?; tail -3 gpurun_out/r2s_parity.log
