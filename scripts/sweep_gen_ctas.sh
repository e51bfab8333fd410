# 5a direct path after the SWAR scan: generate CTAs/SM x side CTAs/SM, and the
# generate's register cap at the default split (one process per setting)
for g in 6 8 12; do for sd in 3 4; do
  MAPC_OVL_GEN_CTAS=$g MAPC_OVL_SIDE_CTAS=$sd python scripts/probe_direct.py 5a | sed "s/^{/{\"gen_ctas\": $g, \"side_ctas\": $sd, /"
done; done
for mb in 8 12; do
  MAPC_JIT_MINB=$mb python scripts/probe_direct.py 5a | sed "s/^{/{\"minb_env\": $mb, /"
done
