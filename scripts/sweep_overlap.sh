# 5a direct path: overlap CTA split (generate CTAs/SM x side-stream CTAs/SM) and
# the generate's register cap, one process per setting (the knobs are read once)
for g in 8 10 12 16; do for sd in 2 3 4 6; do
  MAPC_OVL_GEN_CTAS=$g MAPC_OVL_SIDE_CTAS=$sd python scripts/probe_direct.py 5a | sed "s/^{/{\"gen_ctas\": $g, \"side_ctas\": $sd, /"
done; done
for mb in 8 12 16; do
  MAPC_JIT_MINB=$mb python scripts/probe_direct.py 5a
done
