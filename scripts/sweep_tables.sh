# 5a with three tables in rotation: scan depth x scan CTAs
bash scripts/box_info.sh | tail -1
for un in 2 4; do for sd in 6 8 10; do
  MAPC_SCAN_UNROLL=$un MAPC_OVL_SIDE_CTAS=$sd timeout 300 python scripts/probe_direct5a.py 2>&1 | grep '^{'
done; done
