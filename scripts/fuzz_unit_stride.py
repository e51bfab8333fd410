"""Differential check of the compile-time unit-stride sites: among
fuzz seeds [a, b), every instance whose direct-mode JIT source marks a site
unit-stride (US_ true) is run on the direct path with the JIT generate, default
and unit chunks, and compared with the CPU oracle.  Prints mismatches and a summary."""
import os, re, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_2203_12878_b200 as mc
from workloads import fuzz

a, b = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (0, 4000)
n = bad = picked = 0
t0 = time.time()
for seed in range(a, b):
    inst, _ = fuzz.random_instance(seed)
    try:
        p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    except Exception:
        continue
    if not any("true" in x for c in range(min(p.n_chunks(0), 4))
               for x in re.findall(r"US_\[\d+\] = \{([^}]*)\}", p.jit_source(c, 1))):
        continue
    o = oracle.check_instance(inst, threads=1)
    if o.status != 0:
        continue
    picked += 1
    want = (o.verdict, o.witness, o.n_accesses, o.n_racy_segments)
    unit = max(1, p.info.max_unit_accesses)
    for chunk in (0, unit):
        if chunk and p.n_chunks(chunk) > 16:
            continue
        r = p.check_races(detect="direct", gen="jit", chunk_max_accesses=chunk)
        got = (r.verdict, r.witness.as_tuple() if r.witness else None, r.n_accesses, r.racy_segments)
        n += 1
        if got != want:
            bad += 1
            print("MISMATCH", seed, chunk, got, want, flush=True)
print(f"seeds [{a},{b}): {picked} instances with unit-stride sites, {n} runs, {bad} mismatches, "
      f"{time.time() - t0:.0f} s", flush=True)
