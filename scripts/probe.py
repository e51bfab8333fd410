"""Quick timing probe (not the bench): run a config N times, print device ms."""
import sys, time, json
import torch
import paper_2203_12878_b200 as mc
from workloads import config

name = sys.argv[1] if len(sys.argv) > 1 else "5a"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
inst = config(name)
p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
need = p.scratch_bytes()
scratch = torch.empty(need, dtype=torch.uint8, device="cuda")
for i in range(reps):
    t = time.time()
    r = p.check_races(scratch=scratch)
    dt = time.time() - t
    print(json.dumps(dict(cfg=name, ms=r.device_ms, wall=dt, n=r.n_accesses, verdict=r.verdict,
                          witness=r.witness.as_tuple() if r.witness else None, racy=r.racy_segments,
                          chunks=r.n_chunks, launches=r.gpu_launches,
                          gacc=r.n_accesses / r.device_ms / 1e6)), flush=True)
