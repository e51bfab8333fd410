"""4c/4d (and 4a/4b) device time per call vs the chunk capacity (default, 1/2, 1/4, 1/8 of the plan)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config

for name in (sys.argv[1:] or ["4c", "4d", "4a", "4b"]):
    inst = config(name)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    out = {"cfg": name}
    for div in (0, 2, 4, 8):
        chunk = 0 if div == 0 else max(p.info.max_unit_accesses, p.info.max_accesses // div)
        scratch = torch.empty(p.scratch_bytes(chunk), dtype=torch.uint8, device="cuda")
        for _ in range(2):
            r = p.check_races(scratch=scratch, chunk_max_accesses=chunk)
        ms = min(p.check_races(scratch=scratch, chunk_max_accesses=chunk).device_ms for _ in range(5))
        out[f"div{div}"] = {"chunks": p.n_chunks(chunk), "ms": round(ms, 4), "G_acc_s": round(r.n_accesses / ms / 1e6, 1)}
        del scratch
    print(json.dumps(out), flush=True)
