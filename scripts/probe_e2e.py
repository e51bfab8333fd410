"""Where the e2e path's time goes (5a): per step a new MapProgram from the MAP text
(map_compile) and one map_check_races, as bench.py's e2e leg; host wall time of the
compile, of the call, and the call's device time."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config

inst = config("5a")
p0 = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
scratch = mc.alloc_scratch(p0.scratch_bytes())
stream = torch.cuda.current_stream()
for _ in range(3):
    p0.check_races(scratch=scratch, stream=stream)
rows = []
for i in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    t1 = time.perf_counter()
    r = p.check_races(scratch=scratch, stream=stream)
    t2 = time.perf_counter()
    rows.append({"compile_ms": round((t1 - t0) * 1e3, 3), "call_ms": round((t2 - t1) * 1e3, 3),
                 "device_ms": round(r.device_ms, 3)})
    del p
print(json.dumps({"steps": rows}), flush=True)
