"""Device throughput of every config family at full size (every detect path).

Usage: python scripts/probe_configs.py [names...] [--paths=auto,unit,direct,table,sort] [--compressible]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config, CONFIG_NAMES

args = [a for a in sys.argv[1:] if not a.startswith("--")]
paths = ("auto", "unit", "direct", "table", "sort")
for a in sys.argv[1:]:
    if a.startswith("--paths="):
        paths = tuple(a.split("=", 1)[1].split(","))
for name in (args or CONFIG_NAMES):
    if name.startswith("5"):
        continue
    inst = config(name)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    scratch = (mc.alloc_scratch(p.scratch_bytes()) if "--compressible" in sys.argv
               else torch.empty(p.scratch_bytes(), dtype=torch.uint8, device="cuda"))
    out = {"cfg": name}
    for det in paths:
        gen = "jit" if det == "unit" else "auto"
        p.check_races(scratch=scratch, detect=det, gen=gen)
        ms = []
        for _ in range(5):
            r = p.check_races(scratch=scratch, detect=det, gen=gen)
            ms.append(r.device_ms)
        best = min(ms)
        k = p.check_races(scratch=scratch, detect=det, gen=gen, profile=True).kernels
        out[det] = {"ms": round(best, 4), "G_acc_s": round(r.n_accesses / best / 1e6, 2),
                    "res": [r.verdict, r.witness.as_tuple() if r.witness else None, r.racy_segments],
                    "top": sorted(((v["ms"], c) for c, v in k.items() if v["launches"]), reverse=True)[:3]}
    out["n"] = r.n_accesses
    out["chunks"] = r.n_chunks
    print(json.dumps(out), flush=True)
