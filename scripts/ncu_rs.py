import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_12878_b200 as mc
from workloads import config
inst = config("5a", T=1, R=64)
r = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params).check_races()
print(r.n_accesses, r.verdict, r.device_ms)
