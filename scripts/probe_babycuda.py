"""NEXT-2 executor throughput: BabyCUDA kernels of the workload families at
config scale, executed with data on the GPU (map_execute: run + sort + race
check) and checked against their inferred MAP (map_theorem1_diff)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_12878_b200 as mc
from workloads import babycuda as wb

cases = [("transpose", dict(ts=32, rw=8, grid=65536)), ("transpose_racy", dict(ts=32, rw=8, grid=65536)),
         ("reduce", dict(block=1024, grid=4096)), ("hillis", dict(n=1 << 16, bs=1024)),
         ("stencil", dict(block=1024, T=4, R=16, C=256))]
for name, kw in cases:
    inst = wb.kernel(name, **kw)
    k = mc.Kernel(inst.src, inst.grid, inst.block, inst.params)
    r = k.execute()
    ms = []
    for _ in range(3):
        r = k.execute()
        ms.append(r.device_ms)
    best = min(ms)
    prog = mc.MapProgram(mc.infer(inst.src).map_text, inst.grid, inst.block, inst.params)
    t0 = time.perf_counter()
    d = k.theorem1_diff(prog)
    dt = time.perf_counter() - t0
    m = prog.check_races()
    print(json.dumps({"kernel": name, "sizes": kw, "n_events": r.n_events, "exec_ms": round(best, 3),
                      "G_events_s": round(r.n_events / best / 1e6, 2), "verdict": r.verdict,
                      "witness": r.witness.as_tuple() if r.witness else None,
                      "map_verdict": m.verdict, "map_witness": m.witness.as_tuple() if m.witness else None,
                      "theorem1_equal": d.equal, "n_alpha": d.n_alpha, "n_lambda": d.n_lambda,
                      "diff_wall_s": round(dt, 3)}), flush=True)
