# 5a with L2 eviction-priority hints on the table streams
for cfg in "MAPC_X=0" "MAPC_SCAN_EVICT_FIRST=1" "MAPC_GEN_EVICT_LAST=1" "MAPC_SCAN_EVICT_FIRST=1 MAPC_GEN_EVICT_LAST=1" "MAPC_X=0"; do
  env $cfg timeout 300 python scripts/probe_direct5a.py 2>&1 | tail -1
done
