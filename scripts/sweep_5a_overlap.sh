# 5a step time (graph replay) over the overlapped pipeline's CTA shares,
# scratch from map_scratch_alloc (compressible; PLAIN_SCRATCH=1 for torch.empty)
for g in 10 12 14 16; do for sd in 2 3 4 6; do
  MAPC_OVL_GEN_CTAS=$g MAPC_OVL_SIDE_CTAS=$sd timeout 300 python scripts/probe_direct5a.py 2>&1 | tail -1
done; done
for mb in 8 12; do MAPC_JIT_MINB=$mb timeout 300 python scripts/probe_direct5a.py 2>&1 | tail -1; done
