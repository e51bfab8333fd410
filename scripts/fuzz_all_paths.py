"""Extended differential check (not part of the test suite's time budget):
every detect path x generate path vs the CPU oracle on fuzz seeds [a, b),
with the plan's default chunks and with unit chunks.  Prints mismatches and a
summary line."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_2203_12878_b200 as mc
from workloads import fuzz

args = [x for x in sys.argv[1:] if not x.startswith("--")]
a, b = (int(args[0]), int(args[1])) if len(args) > 1 else (0, 1000)
combos = [("auto", "auto"), ("direct", "vm"), ("direct", "jit"), ("unit", "jit"), ("table", "vm"), ("sort", "vm")]
big = "--big" in sys.argv          # blockDim 1025..2048 (u32 cells)
bad, n, t0 = 0, 0, time.time()
for seed in range(a, b):
    inst, _ = fuzz.random_instance(seed, big_block=big)
    o = oracle.check_instance(inst, threads=1)
    if o.status != 0:
        continue
    want = (o.verdict, o.witness, o.n_accesses, o.n_racy_segments)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    unit = max(1, p.info.max_unit_accesses)
    for det, gen in combos:
        for chunk in (0, unit):
            if gen == "jit" and chunk and p.n_chunks(chunk) > 16:
                continue
            r = p.check_races(detect=det, gen=gen, chunk_max_accesses=chunk)
            got = (r.verdict, r.witness.as_tuple() if r.witness else None, r.n_accesses, r.racy_segments)
            n += 1
            if got != want:
                bad += 1
                print("MISMATCH", seed, det, gen, chunk, got, want, inst.src, flush=True)
print(f"seeds {a}..{b}: {n} runs, {bad} mismatches, {time.time() - t0:.0f} s", flush=True)
