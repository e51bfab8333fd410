"""Device time of one call, VM vs JIT generate (direct path), best of 3 after a warm-up."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config

for name in (sys.argv[1:] or ["3a", "3b", "4a", "4b", "4c", "4d"]):
    inst = config(name)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    scratch = torch.empty(p.scratch_bytes(), dtype=torch.uint8, device="cuda")
    out = {"cfg": name}
    for gen in ("vm", "jit"):
        r = p.check_races(scratch=scratch, gen=gen)
        best = min(p.check_races(scratch=scratch, gen=gen).device_ms for _ in range(3))
        out[gen] = {"ms": round(best, 3), "G_acc_s": round(r.n_accesses / best / 1e6, 1)}
    print(json.dumps(out), flush=True)
