"""Device throughput of every config family at full size (every detect path)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config, CONFIG_NAMES

for name in CONFIG_NAMES:
    inst = config(name)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    scratch = torch.empty(p.scratch_bytes(), dtype=torch.uint8, device="cuda")
    out = {"cfg": name}
    for det in ("auto", "direct", "table", "sort"):
        p.check_races(scratch=scratch, detect=det)
        ms = []
        for _ in range(3):
            r = p.check_races(scratch=scratch, detect=det)
            ms.append(r.device_ms)
        best = min(ms)
        out[det] = {"ms": round(best, 3), "G_acc_s": round(r.n_accesses / best / 1e6, 2),
                    "res": [r.verdict, r.witness.as_tuple() if r.witness else None, r.racy_segments]}
    out["n"] = r.n_accesses
    out["verdict"] = r.verdict
    out["chunks"] = r.n_chunks
    print(json.dumps(out), flush=True)
