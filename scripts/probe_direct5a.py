"""5a direct generate alone and live: per-launch ms of the fused generate (gen_0,
mode direct) with the chunks sequential and overlapped, and the step's G acc/s."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config

inst = config("5a")
p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
CHUNK = int(os.environ.get("CHUNK", "0"))      # chunk_max_accesses (0 = library default)
scratch = (torch.empty(p.scratch_bytes(CHUNK), dtype=torch.uint8, device="cuda") if os.environ.get("PLAIN_SCRATCH")
           else mc.alloc_scratch(p.scratch_bytes(CHUNK)))
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("MAPC_") or k == "CHUNK"}}
for ovl in (False, True):
    p.check_races(scratch=scratch, overlap=ovl, chunk_max_accesses=CHUNK)
    r = p.check_races(scratch=scratch, overlap=ovl, profile=True, chunk_max_accesses=CHUNK)
    k = r.kernels["direct"]
    out["overlap" if ovl else "alone"] = {"gen_ms": round(k["ms"] / max(1, k["launches"]), 4),
                                          "step_ms": round(r.device_ms, 3),
                                          "G_acc_s": round(r.n_accesses / r.device_ms / 1e6, 1)}
    assert r.verdict == 0 and r.n_accesses == 2**34
ms = []
for _ in range(5):
    ms.append(p.check_races(scratch=scratch, chunk_max_accesses=CHUNK).device_ms)
out["graph_step_ms"] = round(min(ms), 3)
out["G_acc_s"] = round(2**34 / min(ms) / 1e6, 1)
print(json.dumps(out), flush=True)
