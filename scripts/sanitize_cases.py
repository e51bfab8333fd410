"""Small invocations of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): the MAP paths (VM and JIT
generate; unit, direct, table and sort detect; listing; key exchange stages)
on scaled configs 1a, 2b, 3b, 4b, 5b, and the BabyCUDA executor + Theorem-1 diff.
Prints one line per case; exits non-zero on a result mismatch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_12878_b200 as mc  # noqa: E402
from workloads import config  # noqa: E402
from workloads import babycuda as wb  # noqa: E402

cases = [config("1a"), config("2b"), config("3b", ts=32, rw=8, grid=16), config("4b", n=4096, bs=256),
         config("5b", block=64, T=2, R=4, C=16)]
bad = 0
for inst in cases:
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    ref = None
    for gen, det in [("vm", "sort"), ("vm", "table"), ("vm", "direct"), ("jit", "direct"), ("jit", "unit"),
                     ("jit", "sort")]:
        r = p.check_races(gen=gen, detect=det)
        got = (r.verdict, r.witness.as_tuple() if r.witness else None, r.n_accesses, r.racy_segments)
        ref = ref or got
        bad += got != ref
        print(inst.name, gen, det, got, flush=True)
    total, lst = p.list_races(cap=16)
    print(inst.name, "list", total, len(lst), flush=True)
    scratch = torch.empty(p.scratch_bytes(), dtype=torch.uint8, device="cuda")
    keys = torch.empty(max(1, p.chunk_info(0)["bound"]), dtype=torch.int64, device="cuda")
    counts = p.generate_bucketed(0, 0, 2, keys, scratch)
    print(inst.name, "bucketed", counts, flush=True)
for name in ("reduce", "transpose_racy", "hillis_inplace"):
    inst = wb.kernel(name)
    k = mc.Kernel(inst.src, inst.grid, inst.block, inst.params)
    r = k.execute(keep_memory=True)
    d = k.theorem1_diff(mc.MapProgram(mc.infer(inst.src).map_text, inst.grid, inst.block, inst.params))
    bad += not d.equal
    print(name, "exec", r.verdict, r.n_events, "theorem1", d.equal, flush=True)
sys.exit(1 if bad else 0)
