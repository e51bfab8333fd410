"""ncu target for the direct-address path: config 5a at full size (2^34
accesses, 16 one-phase chunks of 2^30), exactly the bench's workload and
launch configuration; one check_races call (capture with -c to limit replays)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config

inst = config(sys.argv[1] if len(sys.argv) > 1 else "5a")
p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
r = p.check_races(detect="direct")
print(r.n_accesses, r.verdict, r.device_ms)
