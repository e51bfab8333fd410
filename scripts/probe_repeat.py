"""Repeated calls on one program (graph replay from the third call): device time
and host wall time per call, results checked against the first call."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config

for name in (sys.argv[1:] or ["1a", "1b", "2a", "2b", "4c", "3a", "5a"]):
    inst = config(name)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    scratch = torch.empty(p.scratch_bytes(), dtype=torch.uint8, device="cuda")
    ref = p.check_races(scratch=scratch)
    key = lambda r: (r.verdict, r.witness.as_tuple() if r.witness else None, r.n_accesses, r.racy_segments)
    dev, wall, ok = [], [], True
    for i in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = p.check_races(scratch=scratch)
        wall.append((time.perf_counter() - t0) * 1e3)
        dev.append(r.device_ms)
        ok = ok and key(r) == key(ref)
    print(json.dumps({"cfg": name, "same_results": ok, "device_ms": [round(x, 3) for x in dev[:3]] + [round(min(dev[3:]), 3)],
                      "wall_ms": [round(x, 3) for x in wall[:3]] + [round(min(wall[3:]), 3)]}), flush=True)
