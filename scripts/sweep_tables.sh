# 5a with three tables in rotation (the default with the row-jammed generate): generate / scan / clear CTAs
for rep in 1 2; do for g in 6 8 10; do for sd in 6; do for cl in 3 4; do
  MAPC_OVL_GEN_CTAS=$g MAPC_OVL_SIDE_CTAS=$sd MAPC_OVL_CLEAR_CTAS=$cl timeout 300 python scripts/probe_direct5a.py 2>&1 | grep '^{'
done; done; done; done
