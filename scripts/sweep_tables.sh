# 5a, three tables: register cap of the generate (MAPC_JIT_MINB) x its CTAs per SM
bash scripts/box_info.sh | tail -1
for mb in 10 12 16; do for g in 10 12 14; do
  MAPC_JIT_MINB=$mb MAPC_OVL_GEN_CTAS=$g timeout 300 python scripts/probe_direct5a.py 2>&1 | grep '^{'
done; done
