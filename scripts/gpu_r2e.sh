for cfg in "MAPC_RED_CACHE=0" "MAPC_RED_CACHE=1" "MAPC_JIT_MINB=8" "MAPC_JIT_MINB=6" "MAPC_JIT_MINB=12" "MAPC_RED_CACHE=0 MAPC_JIT_MINB=8"; do
  env $cfg timeout 300 python scripts/probe_direct5a.py 2>&1 | tail -1
done > gpurun_out/r2e_direct5a.jsonl
cat gpurun_out/r2e_direct5a.jsonl
