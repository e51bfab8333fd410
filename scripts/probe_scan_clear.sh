# fused scan + clear (MAPC_SCAN_CLEAR=1) vs separate passes, 5a/5b direct path, and
# parity of the fused variant on the GPU suite's direct-path and config tests
for sc in 0 1; do for sd in 2 3 4; do
  MAPC_SCAN_CLEAR=$sc MAPC_OVL_SIDE_CTAS=$sd python scripts/probe_direct.py 5a 5b | sed "s/^{/{\"scan_clear\": $sc, \"side_ctas\": $sd, /"
done; done
MAPC_SCAN_CLEAR=1 python -m pytest tests -m gpu -x -q -k "direct or configs or fuzz" 2>&1 | tail -2
