# 5a with three tables in rotation (the default with the row-jammed generate): generate / clear CTAs
bash scripts/box_info.sh | tail -1
for rep in 1 2; do for g in 8 10; do for cl in 3 4; do
  MAPC_OVL_GEN_CTAS=$g MAPC_OVL_SIDE_CTAS=6 MAPC_OVL_CLEAR_CTAS=$cl timeout 300 python scripts/probe_direct5a.py 2>&1 | grep '^{'
done; done; done
