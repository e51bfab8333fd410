"""Extended differential check of the stride-compressed direct table: random strided
MAPs (workloads.fuzz.random_strided_instance, seeds [a, b)) on the direct path with the
specialised generate (overlapped and sequential) vs the CPU oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_2203_12878_b200 as mc
from workloads import fuzz

a, b = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (0, 1000)
t0, runs, bad, comp = time.time(), 0, 0, 0
for seed in range(a, b):
    inst = fuzz.random_strided_instance(seed)
    o = oracle.check_instance(inst)
    if o.status != 0:
        continue
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    comp += any("cbase_" in p.jit_source(c, 1) for c in range(p.n_chunks()))
    want = (o.verdict, o.witness, o.n_accesses, o.n_racy_segments)
    for ovl in (True, False):
        r = p.check_races(detect="direct", gen="jit", overlap=ovl)
        runs += 1
        got = (r.verdict, r.witness.as_tuple() if r.witness else None, r.n_accesses, r.racy_segments)
        if got != want:
            bad += 1
            print("MISMATCH", seed, ovl, got, want, inst.src, flush=True)
print(f"seeds {a}..{b}: {runs} runs ({comp} compressed programs), {bad} mismatches, {time.time() - t0:.0f} s")
