"""Device time of one call at several chunk capacities (direct path), full-size configs."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config

for name in (sys.argv[1:] or ["3a", "3b", "4a", "4b", "4c"]):
    inst = config(name)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    unit = p.info.max_unit_accesses
    total = p.info.max_accesses
    for cap in sorted({0, max(unit, total // 2), max(unit, total // 4), max(unit, total // 8)}):
        scratch = torch.empty(p.scratch_bytes(cap), dtype=torch.uint8, device="cuda")
        r = p.check_races(scratch=scratch, chunk_max_accesses=cap)
        best = min(p.check_races(scratch=scratch, chunk_max_accesses=cap).device_ms for _ in range(4))
        print(json.dumps({"cfg": name, "cap": cap, "chunks": r.n_chunks, "ms": round(best, 3),
                          "G_acc_s": round(r.n_accesses / best / 1e6, 1)}), flush=True)
        del scratch
