# 5a direct path: side-stream CTAs/SM of the overlapped pipeline, and the
# sequential pipeline, one process per setting (the knobs are read once)
for sd in 2 3 4 6 8; do
  MAPC_OVL_SIDE_CTAS=$sd python scripts/probe_direct.py 5a | sed "s/^{/{\"side_ctas\": $sd, /"
done
MAPC_OVERLAP=0 python scripts/probe_direct.py 5a | sed "s/^{/{\"overlap\": 0, /"
