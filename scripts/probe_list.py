"""Time the full race listing (NEXT-4) against map_check_races on one config."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config

name = sys.argv[1] if len(sys.argv) > 1 else "3b"
kw = {"T": int(sys.argv[2])} if len(sys.argv) > 2 else {}
inst = config(name, **kw)
p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
scratch = torch.empty(p.scratch_bytes(), dtype=torch.uint8, device="cuda")
r = p.check_races(scratch=scratch)
out = {"cfg": name, **kw, "n": r.n_accesses, "racy_segments": r.racy_segments, "check_ms": r.device_ms}
for cap in (1000, 1 << 20):
    p.list_races(cap=cap, scratch=scratch)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    total, got = p.list_races(cap=cap, scratch=scratch)
    torch.cuda.synchronize()
    out[f"list_cap{cap}_s"] = round(time.perf_counter() - t0, 4)
    assert total == r.racy_segments and got[0].as_tuple() == r.witness.as_tuple()
print(json.dumps(out))
