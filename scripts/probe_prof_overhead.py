"""Cost of the bench's per-launch timing events on 5a: graph-replayed steps with no
timing, with CUDA events around the generate launches only (bench.py's timed steps),
and around every launch."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config

inst = config("5a")
p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
scratch = mc.alloc_scratch(p.scratch_bytes())
stream = torch.cuda.current_stream()
out = {}
for mode in (False, "generate", True, False):
    for _ in range(3):
        p.check_races(scratch=scratch, stream=stream, profile=mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        p.check_races(scratch=scratch, stream=stream, profile=mode)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    out.setdefault(str(mode), []).append(round(ms, 3))
print(json.dumps(out), flush=True)
