"""Memory-safety checks of our own (compute-sanitizer is closed on this pool:
profiles/r2f_compute_sanitizer_closed.txt).

* initcheck substitute: the scratch buffer is poisoned (all 0x00, all 0xFF, random
  bytes) before every run; a kernel that read scratch it had not written first would
  change the result -- every path must give the oracle's result regardless.
* memcheck substitute (scratch overruns): the scratch is a view into a larger buffer
  with 1 MiB canary bands of 0xA5 before and after it; no run may touch them.
"""
import pytest

import oracle
import paper_2203_12878_b200 as mc
from workloads import babycuda as wb
from workloads import config

pytestmark = pytest.mark.gpu
BAND = 1 << 20
PATHS = [("vm", "sort"), ("vm", "table"), ("vm", "direct"), ("jit", "direct"), ("jit", "unit"), ("jit", "auto")]
CASES = [config("1a"), config("2b"), config("3b", ts=32, rw=8, grid=64), config("4b", n=4096, bs=256),
         config("4d", n=4096, bs=256), config("5a", block=64, T=3, R=4, C=64), config("5b", block=64, T=2, R=4, C=16)]


def _guarded(n):
    import torch
    buf = torch.full((n + 2 * BAND,), 0xA5, dtype=torch.uint8, device="cuda")
    return buf, buf[BAND:BAND + n]


def _bands_intact(buf, n):
    import torch
    return bool(torch.all(buf[:BAND] == 0xA5)) and bool(torch.all(buf[BAND + n:] == 0xA5))


@pytest.mark.parametrize("inst", CASES, ids=[c.name for c in CASES])
def test_poisoned_and_guarded_scratch(inst):
    import torch
    o = oracle.check_instance(inst)
    want = (o.verdict, o.witness, o.n_accesses, o.n_racy_segments)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    unit = max(1, p.info.max_unit_accesses)
    for chunk in (0, unit):
        if chunk and p.n_chunks(chunk) > 64:
            continue
        n = p.scratch_bytes(chunk)
        buf, scratch = _guarded(n)
        g = torch.Generator(device="cuda").manual_seed(1)
        for poison in ("zero", "ones", "random"):
            for gen, det in PATHS:
                if poison == "zero":
                    scratch.zero_()
                elif poison == "ones":
                    scratch.fill_(0xFF)
                else:
                    scratch.copy_(torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda", generator=g))
                r = p.check_races(scratch=scratch, chunk_max_accesses=chunk, gen=gen, detect=det)
                got = (r.verdict, r.witness.as_tuple() if r.witness else None, r.n_accesses, r.racy_segments)
                assert got == want, (inst.name, chunk, poison, gen, det)
        torch.cuda.synchronize()
        assert _bands_intact(buf, n), (inst.name, chunk)


@pytest.mark.parametrize("name", ["reduce", "transpose_racy", "hillis_inplace", "stencil"])
def test_executor_poisoned_and_guarded_scratch(name):
    import torch
    inst = wb.kernel(name)
    k = mc.Kernel(inst.src, inst.grid, inst.block, inst.params)
    ref = k.execute(keep_memory=True)
    cap = max(1, k.info["max_events"])
    n = mc._lib.map_kernel_scratch_bytes(k._h, cap, 0, mc.EXEC_KEEP_MEMORY)
    buf, scratch = _guarded(n)
    for fill in (0x00, 0xFF, 0x5A):
        scratch.fill_(fill)
        r = k.execute(keep_memory=True, scratch=scratch)
        assert (r.verdict, r.witness, r.n_events, r.n_alpha, r.uninit_reads, r.ambiguous_reads) == \
               (ref.verdict, ref.witness, ref.n_events, ref.n_alpha, ref.uninit_reads, ref.ambiguous_reads)
    torch.cuda.synchronize()
    assert _bands_intact(buf, n)
