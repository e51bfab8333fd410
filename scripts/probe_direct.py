"""Device time of the direct-address path on full-size configs (best of 3)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config

for name in (sys.argv[1:] or ["5a", "5b", "3a", "3b", "4a", "4b"]):
    inst = config(name)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    scratch = torch.empty(p.scratch_bytes(), dtype=torch.uint8, device="cuda")
    r = p.check_races(scratch=scratch, detect="direct", profile=True)
    best, rb = 1e9, None
    for _ in range(3):
        r = p.check_races(scratch=scratch, detect="direct", profile=True)
        if r.device_ms < best:
            best, rb = r.device_ms, r
    k = {c: round(v["ms"], 3) for c, v in rb.kernels.items() if v["launches"]}
    print(json.dumps({"cfg": name, "minb": os.environ.get("MAPC_JIT_MINB", "-"), "ms": round(best, 3),
                      "G_acc_s": round(rb.n_accesses / best / 1e6, 1), "kernels_ms": k}), flush=True)
