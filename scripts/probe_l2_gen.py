"""Direct generate rate when the chunk's table is L2-resident: 5a's stencil at R rows
per thread (table 2 * 2 * 1024 * R * 1024 B), chunks run one after another (the
clear just before each generate leaves the table's zeroed lines in L2), vs R=256."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config

scratch = None
for R in (256, 64, 32, 16, 8):
    inst = config("5a", R=R, T=16)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    need = p.scratch_bytes()
    if scratch is None or scratch.numel() < need:
        scratch = None
        torch.cuda.empty_cache()
        scratch = torch.empty(need, dtype=torch.uint8, device="cuda")
    out = {"R": R, "table_MiB": 4 * R}
    for ovl in (False, True):
        p.check_races(scratch=scratch, overlap=ovl, gen="jit")
        r = p.check_races(scratch=scratch, overlap=ovl, gen="jit", profile=True)
        ks = {k: round(v["ms"] / max(1, v["launches"]), 4) for k, v in r.kernels.items()}
        out["overlap" if ovl else "alone"] = {"per_launch_ms": ks, "step_ms": round(r.device_ms, 3),
                                              "gen_G_acc_s": round(r.n_accesses / 16 / ks["direct"] / 1e6, 1)}
    print(json.dumps(out), flush=True)
