"""5a's stencil at smaller R (rows per thread): how fast is the direct path when a
chunk's table fits in L2?  One line per size: chunks, device ms, G acc/s."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config

sizes = [(256, 16), (128, 16), (64, 16), (32, 16), (16, 16), (8, 16), (4, 16)]
scratch = None
for R, T in sizes:
    inst = config("5a", R=R, T=T)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    need = p.scratch_bytes()
    if scratch is None or scratch.numel() < need:
        scratch = torch.empty(need, dtype=torch.uint8, device="cuda")
    r = p.check_races(scratch=scratch, profile=True, gen="jit")
    ms = []
    for _ in range(5):
        ms.append(p.check_races(scratch=scratch, gen="jit").device_ms)
    k = r.kernels.get("direct", {"ms": 0, "launches": 1})
    print(json.dumps({"R": R, "T": T, "accesses": r.n_accesses, "chunks": r.n_chunks,
                      "table_MiB": 2 * 2 * 1024 * R * 1024 / 2**20,
                      "gen_ms_per_launch": round(k["ms"] / max(1, k["launches"]), 4),
                      "ms": round(min(ms), 3), "G_acc_s": round(r.n_accesses / min(ms) / 1e6, 1),
                      "verdict": r.verdict}), flush=True)
