import json, sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2203_12878_b200 as mc
from workloads import config
for R, T in [(32, 128), (16, 256), (8, 512), (4, 1024)]:
    inst = config("5a", R=R, T=T)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    s = torch.empty(p.scratch_bytes(), dtype=torch.uint8, device="cuda")
    import time; t0 = time.time(); p.check_races(scratch=s); first = time.time() - t0
    ms = min(p.check_races(scratch=s).device_ms for _ in range(4))
    print(json.dumps({"R": R, "T": T, "chunks": p.n_chunks(), "first_call_s": round(first, 2), "ms": round(ms, 3),
                      "G_acc_s": round(2**34 / ms / 1e6, 1)}), flush=True)
    del s
