import json, os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2203_12878_b200 as mc
from workloads import config
for name in ("4a", "4b", "4c"):
    inst = config(name)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    s = mc.alloc_scratch(p.scratch_bytes())
    for ovl in (True, False):
        for _ in range(3): p.check_races(scratch=s, overlap=ovl)
        r = p.check_races(scratch=s, profile=True, overlap=ovl)
        ms = min(p.check_races(scratch=s, overlap=ovl).device_ms for _ in range(4))
        print(json.dumps({"cfg": name, "overlap": ovl, "ms": round(ms, 4), "chunks": r.n_chunks,
                          "k": {k: (round(v["ms"], 4), v["launches"]) for k, v in r.kernels.items() if v["launches"]}}))
    for i in range(p.n_chunks()):
        print(json.dumps({"chunk": i, **p.chunk_info(i)}))
