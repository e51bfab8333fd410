import json, os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2203_12878_b200 as mc
from workloads import config
inst = config("5b")
p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
s = mc.alloc_scratch(p.scratch_bytes())
r = p.check_races(scratch=s)
ms = min(p.check_races(scratch=s).device_ms for _ in range(4))
print(json.dumps({"cfg": "5b", "ms": round(ms, 3), "G_acc_s": round(2**34 / ms / 1e6, 1), "racy": r.racy_segments,
                  "witness": list(r.witness.as_tuple())}))
