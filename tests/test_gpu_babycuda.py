"""GPU parity of NEXT-1/NEXT-2: the BabyCUDA executor (map_execute)
against the oracle's Fig. 5 interpreter (oracle/babycuda.py) -- executed access
values, race verdict and witness, bottom / ambiguous read counts and the final
array CONTENTS, bit-exact -- and the Theorem-1 differential check
(map_theorem1_diff): for typable kernels the executed access set equals the
inferred MAP's Lambda; for the paper's ill-typed kernel (Eq. 1) it does not,
and the abstracted MAP's race is a false alarm."""
import pytest

import oracle
import paper_2203_12878_b200 as mc
from oracle import babycuda as bc
from workloads import babycuda as wb

pytestmark = pytest.mark.gpu


def compare(inst, keep_memory=True):
    o = bc.execute(inst.src, inst.grid, inst.block, inst.params, keep_memory=keep_memory)
    try:
        k = mc.Kernel(inst.src, inst.grid, inst.block, inst.params)
        r = k.execute(keep_memory=keep_memory)
    except mc.MapError as e:
        assert o.status == e.status, (inst.src, o.diag, str(e))
        return None
    assert o.status == 0, (inst.src, o.diag)
    got = (r.verdict, r.witness.as_tuple() if r.witness else None, r.racy_segments, r.n_events, r.n_alpha,
           r.uninit_reads, r.ambiguous_reads)
    want = (o.verdict, o.witness, o.racy_segments, o.n_events, len(o.alpha), o.uninit_reads, o.ambiguous_reads)
    assert got == want, (inst.src, got, want)
    if keep_memory:
        bk = bc.parse(inst.src)
        ext = k.extents
        for b in range(inst.n_blocks):
            for a in range(len(bk.arrays)):
                vals = k.memory(b, a, ext[a])
                gpu = {i: v for i, v in enumerate(vals) if v is not None}
                assert gpu == o.memory[b][a], (inst.src, b, a)
    return r


@pytest.mark.parametrize("name", wb.KERNELS)
def test_executor_workload_kernels(name):
    compare(wb.kernel(name))


@pytest.mark.parametrize("name", list(wb.PAPER))
def test_executor_paper_kernels(name):
    src = wb.PAPER[name] if name != "eq1_ill_typed" else "shared A[8]; " + wb.PAPER[name]
    for blk in (1, 2, 8):
        compare(wb.Instance(name, src, block=(blk, 1, 1), params={"M": 3} if "M" in src else {}))


def test_executor_data_closed_forms():
    # the reduction sums, the transpose transposes (as the oracle's pins)
    inst = wb.kernel("reduce", block=256, grid=3)
    k = mc.Kernel(inst.src, inst.grid, inst.block, inst.params)
    r = k.execute(keep_memory=True)
    assert r.verdict == 0 and r.uninit_reads == 0
    for b in range(3):
        assert k.memory(b, 0, 1) == [256 * 257 // 2]
    inst = wb.kernel("transpose", ts=32, rw=8, grid=5)
    k = mc.Kernel(inst.src, inst.grid, inst.block, inst.params)
    assert k.execute(keep_memory=True).verdict == 0
    for b in range(5):
        out = k.memory(b, 1, 1024)
        assert out == [b * 1024 + (i % 32) * 32 + i // 32 for i in range(1024)]


def test_executor_fuzz():
    bad = []
    for seed in range(0, 240, 2):
        for ill in (False, True):
            inst, _ = wb.random_kernel(seed, ill_typed=ill)
            try:
                compare(inst)
            except AssertionError as e:
                bad.append((seed, ill, str(e)[:300]))
    assert not bad, bad[:3]


def test_executor_thread_conflicts_commit_smallest_tid():
    # every thread writes the same cells in one phase (write-write races): the
    # commit keeps the smallest writer's value, later reads count as ambiguous
    src = "shared A[4], B[64]; for x in 0..4 { A[x] := tid * 10 + x }; sync; let y = A[2] in B[tid] := y"
    for blk in (2, 32, 64):
        compare(wb.Instance("conflict", src, block=(blk, 1, 1)))


def test_executor_errors():
    for src, status in [("shared A[4]; A[1 / (tid - tid)] := 0", 5), ("shared A[4]; let y = A[0] in A[1] := y / 0", 5),
                        ("shared A[4]; A[0] := 18446744073709551615 + tid", 4), ("shared A[4]; A[tid] := 1", 4)]:
        o = bc.execute(src, block=(5, 1, 1))
        assert o.status == status
        with pytest.raises(mc.MapError) as e:
            mc.Kernel(src, block=(5, 1, 1)).execute()
        assert e.value.status == status


# ---- Theorem 1, checked on the GPU ---------------------------------------------

def _diff(inst, domain=0):
    inf = mc.infer(inst.src, data_domain=domain)
    prog = mc.MapProgram(inf.map_text, inst.grid, inst.block, inst.params)
    k = mc.Kernel(inst.src, inst.grid, inst.block, inst.params)
    return inf, prog, k.theorem1_diff(prog)


@pytest.mark.parametrize("name", wb.KERNELS)
def test_theorem1_workload_kernels(name):
    inst = wb.kernel(name)
    inf, prog, d = _diff(inst)
    assert inf.typable and d.equal and d.only_alpha == 0 and d.only_lambda == 0
    m = prog.check_races()
    assert d.n_alpha == d.n_lambda and d.exec.n_events == m.n_accesses
    assert (d.exec.verdict, d.exec.witness.as_tuple() if d.exec.witness else None, d.exec.racy_segments) == \
           (m.verdict, m.witness.as_tuple() if m.witness else None, m.racy_segments)


def test_theorem1_fuzz_typable():
    bad = []
    for seed in range(0, 300, 3):
        inst, _ = wb.random_kernel(seed)
        if bc.execute(inst.src, inst.grid, inst.block, inst.params).status != 0:
            continue
        inf, prog, d = _diff(inst)
        if not (inf.typable and d.equal):
            bad.append((seed, inst.src, d))
    assert not bad, bad[:2]


def test_theorem1_eq1_mismatch_and_false_alarm():
    # ill-typed; the execution is DRF (each thread reads back its own
    # write, x = tid), the data-abstracted MAP is racy: alpha is a strict subset of Lambda
    src = "shared A[8]; " + wb.PAPER["eq1_ill_typed"]
    inst = wb.Instance("eq1", src, block=(8, 1, 1))
    inf, prog, d = _diff(inst, domain=8)
    assert not inf.typable
    assert not d.equal and d.only_alpha == 0 and d.only_lambda > 0
    assert d.exec.verdict == 0 and prog.check_races().verdict == 1
    # the smallest access value only the abstraction has: thread 1 writing A[0] (x = 0)
    assert d.first_lambda == (0, 0, 0, 0, 1, 1)
    rep = mc.check_kernel(src, block=(8, 1, 1), data_domain=8)
    assert rep["typable"] is False and rep["result"].verdict == 1 and rep["true_alarm"] is False


def test_theorem1_ill_typed_fuzz_subset():
    checked = 0
    for seed in range(0, 300, 3):
        inst, planted = wb.random_kernel(seed, ill_typed=True)
        if not planted or bc.execute(inst.src, inst.grid, inst.block, inst.params).status != 0:
            continue
        inf = mc.infer(inst.src, data_domain=8)
        try:
            prog = mc.MapProgram(inf.map_text, inst.grid, inst.block, inst.params)
        except mc.MapError:
            continue                 # e.g. an abstracted read around a sync
        d = mc.Kernel(inst.src, inst.grid, inst.block, inst.params).theorem1_diff(prog)
        assert d.only_alpha == 0, (seed, inst.src)          # the abstraction is sound
        checked += 1
    assert checked >= 20


def test_theorem1_config_scale():
    # config-3 shaped transpose (2^12 blocks x 256 threads) and a 1024-thread stencil
    for inst in [wb.kernel("transpose", ts=32, rw=8, grid=4096), wb.kernel("transpose_racy", ts=32, rw=8, grid=4096),
                 wb.kernel("stencil", block=1024, T=4, R=4, C=64), wb.kernel("stencil_racy", block=1024, T=2, R=4, C=64)]:
        inf, prog, d = _diff(inst)
        assert inf.typable and d.equal, inst.name
        m = prog.check_races()
        assert (d.exec.verdict, d.exec.witness.as_tuple() if d.exec.witness else None) == \
               (m.verdict, m.witness.as_tuple() if m.witness else None)


def test_check_kernel_labels_true_alarms():
    for name in ("reduce_racy", "transpose_racy", "stencil_racy"):
        inst = wb.kernel(name)
        rep = mc.check_kernel(inst.src, inst.grid, inst.block, inst.params)
        o = oracle.check(rep["map"], inst.grid, inst.block, inst.params)
        assert rep["typable"] and rep["result"].verdict == o.verdict == 1 and rep["true_alarm"] is True
