"""Extended differential check of the BabyCUDA executor (NEXT-2) outside the
test budget: random typable and ill-typed kernels, seeds [a, b): the GPU
execution vs the oracle's Fig. 5 interpreter (verdict, witness, racy cells,
executed accesses, |alpha|, bottom / ambiguous reads, final arrays), and for
typable kernels Theorem 1 on the GPU (alpha == Lambda)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_12878_b200 as mc
from oracle import babycuda as bc
from workloads import babycuda as wb

a, b = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (0, 500)
bad, n, nt, t0 = 0, 0, 0, time.time()
for seed in range(a, b):
    for ill in (False, True):
        inst, planted = wb.random_kernel(seed, ill_typed=ill)
        o = bc.execute(inst.src, inst.grid, inst.block, inst.params, keep_memory=True)
        try:
            k = mc.Kernel(inst.src, inst.grid, inst.block, inst.params)
            r = k.execute(keep_memory=True)
        except mc.MapError as e:
            n += 1
            if e.status != o.status:
                bad += 1
                print("MISMATCH status", seed, ill, e.status, o.status, inst.src, flush=True)
            continue
        n += 1
        got = (0, r.verdict, r.witness.as_tuple() if r.witness else None, r.racy_segments, r.n_events, r.n_alpha,
               r.uninit_reads, r.ambiguous_reads)
        want = (o.status, o.verdict, o.witness, o.racy_segments, o.n_events, len(o.alpha), o.uninit_reads,
                o.ambiguous_reads)
        mem_ok = all({i: v for i, v in enumerate(k.memory(blk, arr, k.extents[arr])) if v is not None}
                     == o.memory[blk][arr] for blk in range(inst.n_blocks) for arr in range(len(k.extents)))
        if got != want or not mem_ok:
            bad += 1
            print("MISMATCH", seed, ill, got, want, mem_ok, inst.src, flush=True)
        if not ill:
            inf = mc.infer(inst.src)
            d = k.theorem1_diff(mc.MapProgram(inf.map_text, inst.grid, inst.block, inst.params))
            nt += 1
            if not d.equal:
                bad += 1
                print("THEOREM1", seed, d, inst.src, flush=True)
print(f"seeds {a}..{b}: {n} executions, {nt} Theorem-1 checks, {bad} mismatches, {time.time() - t0:.0f} s", flush=True)
