import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MAPC_OS_VARIANT"] = "39"
import torch
import paper_2203_12878_b200 as mc
from workloads import config
inst = config("5a", T=1, R=256)
p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
scratch = torch.empty(p.scratch_bytes(), dtype=torch.uint8, device="cuda")
p.check_races(scratch=scratch)
buf = (ctypes.c_ulonglong * 16)()
mc._lib.mapc_os_debug(buf, 1)
r = p.check_races(scratch=scratch, profile=True)
mc._lib.mapc_os_debug(buf, 0)
names = ["ticket+zero+sync", "load+early", "sync", "prefix+publish+scan+sync", "lookback(t0)", "rank", "sync", "writeout+sync"]
tot0 = sum(buf[0:8]); tot1 = sum(buf[8:16])
print(json.dumps({"onesweep_ms": r.kernels["onesweep"]["ms"], "t0": {n: round(100 * buf[i] / tot0, 1) for i, n in enumerate(names)},
                  "tlast": {n: round(100 * buf[8 + i] / tot1, 1) for i, n in enumerate(names)}, "cycles_t0": tot0}))
