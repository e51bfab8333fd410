# 5a with three tables in rotation (the default with the row-jammed generate): scan CTAs x clear CTAs, 4-deep scan
for rep in 1 2; do for sd in 5 6 7; do for cl in 1 2 3; do
  MAPC_SCAN_UNROLL=4 MAPC_OVL_SIDE_CTAS=$sd MAPC_OVL_CLEAR_CTAS=$cl timeout 300 python scripts/probe_direct5a.py 2>&1 | grep '^{'
done; done; done
