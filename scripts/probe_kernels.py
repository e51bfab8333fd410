"""Per-kernel-class timings of config 5a scaled to T phases (default 4), live CUDA events."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config

T = int(sys.argv[1]) if len(sys.argv) > 1 else 4
name = sys.argv[2] if len(sys.argv) > 2 else "5a"
detect = sys.argv[3] if len(sys.argv) > 3 else "auto"
inst = config(name, T=T) if name[0] == "5" else config(name)
p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
scratch = torch.empty(p.scratch_bytes(), dtype=torch.uint8, device="cuda")
p.check_races(scratch=scratch, detect=detect)
r = p.check_races(scratch=scratch, profile=True, detect=detect)
out = {"detect": detect, "cfg": name, "T": T, "ms": round(r.device_ms, 2),
       "gacc": round(r.n_accesses / r.device_ms / 1e6, 2), "verdict": r.verdict, "n": r.n_accesses}
for k, v in r.kernels.items():
    if v["ms"] > 0.05:
        out[k] = (round(v["ms"], 2), round(v["bytes"] / v["ms"] / 1e6, 0) if v["bytes"] else None)
print(json.dumps(out), flush=True)
