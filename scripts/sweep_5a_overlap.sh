# 5a step time (graph replay) over the overlapped pipeline's CTA shares,
# scratch from map_scratch_alloc (compressible; PLAIN_SCRATCH=1 for torch.empty)
for g in 6 8 10 12; do for sd in 3 4 6 8; do
  MAPC_OVL_GEN_CTAS=$g MAPC_OVL_SIDE_CTAS=$sd timeout 300 python scripts/probe_direct5a.py 2>&1 | grep '^{'
done; done
