"""Host turnaround of one blocking map_check_races call (5a): wall time per call vs the
call's device time, with and without per-kernel profiling, and back-to-back steps timed
with CUDA events around the whole loop (as bench.py does)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config

inst = config("5a")
p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
scratch = mc.alloc_scratch(p.scratch_bytes())
stream = torch.cuda.current_stream()
for prof in (False, True):
    for _ in range(3):
        p.check_races(scratch=scratch, stream=stream, profile=prof)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    walls, devs = [], []
    e0.record(stream)
    for _ in range(10):
        t0 = time.perf_counter()
        r = p.check_races(scratch=scratch, stream=stream, profile=prof)
        walls.append((time.perf_counter() - t0) * 1e3)
        devs.append(r.device_ms)
    e1.record(stream)
    torch.cuda.synchronize()
    loop = e0.elapsed_time(e1) / 10
    print(json.dumps({"profile": prof, "loop_ms_per_step": round(loop, 3), "wall_ms": round(sum(walls) / 10, 3),
                      "device_ms": round(sum(devs) / 10, 3), "gap_ms": round(loop - sum(devs) / 10, 3),
                      "G_acc_s_loop": round(2**34 / loop / 1e6, 1)}), flush=True)
