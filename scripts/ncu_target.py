"""ncu target: config 5a scaled to T=2 phases, R=32 rows/thread (2^27 keys per
phase chunk) -- same kernels, same launch configuration as the bench, small
enough for ~40 replays per kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import config

inst = config("5a", T=2, R=32)
p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
r = p.check_races()
print(r.n_accesses, r.verdict, r.device_ms)
assert r.n_accesses == 4 * 2 * 32 * 1024 * 1024 and r.verdict == 0
