import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_12878_b200 as mc
from workloads import config
inst = config("3b")
p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
a = p.check_races(detect="sort")
b = p.check_races(detect="table")
print(json.dumps({"G": os.environ.get("MAPC_TABLE_G"), "sort": [a.racy_segments, a.n_accesses], "table": [b.racy_segments, b.n_accesses]}))
