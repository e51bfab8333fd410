"""One rank's share of the chunk-sharded run, timed on ONE GPU: rank 0 of
world W processes chunks c = 0, W, 2W, ....  The device time of
that share bounds what one GPU of a W-GPU run spends on its chunks -- a
projection of the per-rank work, not a multi-GPU measurement (no NCCL, no
concurrent ranks)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config

inst = config(sys.argv[1] if len(sys.argv) > 1 else "5a")
p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
scratch = torch.empty(p.scratch_bytes(), dtype=torch.uint8, device="cuda")
full = p.check_races(scratch=scratch)
for world in (1, 2, 4, 8):
    best = 1e9
    for _ in range(4):
        r = p.check_races(scratch=scratch, rank=0, world=world)
        best = min(best, r.device_ms)
    print(json.dumps({"cfg": inst.name, "world": world, "rank0_chunks": r.n_chunks, "rank0_ms": round(best, 3),
                      "projected_G_acc_s": round(full.n_accesses / best / 1e6, 1)}), flush=True)
