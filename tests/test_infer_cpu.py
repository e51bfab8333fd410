"""NEXT-1 on the CPU: the product's BabyCUDA front end (map_infer, C++) against
the oracle (oracle/babycuda.py): same typability verdict, same first failing
premise (kind, variable, line:col), and MAP texts with the same meaning (the
C++ MAP oracle enumerates identical access multisets from both), accepted by
the product's own MAP compiler."""
import random

import pytest

import oracle
import paper_2203_12878_b200 as mc
from oracle import babycuda as bc
from workloads import babycuda as wb

KIND = {bc.T_OK: "ok", bc.T_DATA_INDEX: "data_dependent_index", bc.T_DATA_CONTROL: "data_dependent_control"}


def _records(map_src, inst):
    o = oracle.check(map_src, inst.grid, inst.block, inst.params)
    if o.status != 0:
        return ("status", o.status)
    recs = oracle.enumerate_accesses(map_src, inst.grid, inst.block, inst.params)
    return sorted(tuple(int(x) for x in r) for r in recs)


def _agree(inst, domain):
    st, ty, m = bc.infer_text(inst.src, domain=domain)
    got = mc.infer(inst.src, data_domain=domain)
    assert got.typable == ty.typable, inst.src
    if not ty.typable:
        assert (got.kind, got.var, got.line, got.col) == (KIND[ty.kind], ty.var, ty.line, ty.col), inst.src
    if st == 0:
        assert got.map_text is not None
        want = _records(m, inst)
        assert _records(got.map_text, inst) == want, (inst.src, got.map_text, m)
        if isinstance(want, tuple):      # e.g. an abstracted read around a sync: forU over a barrier
            with pytest.raises(mc.MapError) as e:
                mc.MapProgram(got.map_text, inst.grid, inst.block, inst.params)
            assert e.value.status == want[1]
        else:
            mc.MapProgram(got.map_text, inst.grid, inst.block, inst.params)     # the product compiler accepts it
    else:
        assert got.map_text is None


@pytest.mark.parametrize("name", list(wb.PAPER))
def test_paper_kernels(name):
    for domain in (0, 8):
        _agree(wb.Instance(name, wb.PAPER[name], block=(4, 1, 1), params={"M": 3} if "M" in wb.PAPER[name] else {}),
               domain)


def test_paper_derivation_texts():
    # the displayed results, as MAP text
    assert mc.infer(wb.PAPER["fig3_racy"]).map_text == "params M; shared A; forU x in 0..M { rd A[x]; wr A[x] }"
    assert mc.infer(wb.PAPER["fig4_drf"]).map_text == "shared A; if (tid = 0) { wr A[0] } else { skip }"
    e = mc.infer(wb.PAPER["eq1_ill_typed"])
    assert not e.typable and e.kind == "data_dependent_index" and e.var == "x" and e.map_text is None


@pytest.mark.parametrize("name", wb.KERNELS)
def test_workload_kernels(name):
    _agree(wb.kernel(name), 0)


def test_fuzz_typable_and_ill_typed():
    for seed in range(250):
        for ill in (False, True):
            inst, _ = wb.random_kernel(seed, ill_typed=ill)
            for domain in ((0, 6) if ill else (0,)):
                _agree(inst, domain)


@pytest.mark.parametrize("src,status", [
    ("if (tid = 0) { sync } else { skip }", 3),
    ("for x in 0..tid { A[x] := 1; sync }", 3),
    ("let y = A[0] in for x in 0..y { sync }", 3),
    ("A[q] := 1", 2),
    ("Q[0] := 1", 2),
    ("for x in 0..2 { for x in 0..2 { A[x] := 1 } }", 2),
    ("let z = A[0] in let z = A[1] in skip", 2),
    ("if (tid = 0) { A[0] := 1 }", 1),
    ("A[0] = 1", 1),
    ("A[0] := 1 $", 1),
    ("A[18446744073709551616] := 1", 4),
])
def test_static_errors_match_oracle(src, status):
    with pytest.raises(bc.BcError) as e:
        bc.parse(src)
    assert e.value.status == status
    with pytest.raises(mc.MapError) as e2:
        mc.infer(src)
    assert e2.value.status == status


def test_mutated_texts_same_status_class():
    # random token deletions / swaps of valid kernels: both front ends accept or
    # reject them alike (status only; diagnostics may word the position differently)
    rng = random.Random(3)
    for seed in range(150):
        inst, _ = wb.random_kernel(seed)
        toks = inst.src.split(" ")
        for _ in range(3):
            t = list(toks)
            i = rng.randrange(len(t))
            if rng.random() < 0.5:
                del t[i]
            else:
                j = rng.randrange(len(t))
                t[i], t[j] = t[j], t[i]
            src = " ".join(t)
            try:
                bc.parse(src)
                want = 0
            except bc.BcError as e:
                want = e.status
            try:
                mc.infer(src, data_domain=4)
                got = 0
            except mc.MapError as e:
                got = e.status
            assert got == want, (src, got, want)


# ---- NEXT-2 executor planning on the CPU (no GPU: NVRTC compiles without one) --

def test_executor_sources_compile():
    bad = []
    kernels = [wb.kernel(n) for n in wb.KERNELS] + [wb.random_kernel(s, ill_typed=ill)[0]
                                                    for s in range(0, 60, 3) for ill in (False, True)]
    for inst in kernels:
        try:
            k = mc.Kernel(inst.src, inst.grid, inst.block, inst.params)
        except mc.MapError as e:
            bad.append((inst.src, str(e)))
            continue
        log = k.jit_check()
        if log:
            bad.append((inst.src, log[:500]))
    assert not bad, bad[:2]


def test_executor_plan_facts():
    inst = wb.kernel("transpose", ts=8, rw=4, grid=4)
    k = mc.Kernel(inst.src, inst.grid, inst.block, inst.params)
    i = k.info
    assert i["typable"] == 1 and i["n_phases"] == 2 and i["n_arrays"] == 2 and i["cells_per_block"] == 128
    assert i["max_events"] == 4 * 32 * 6      # 2 rows per thread: tile write, tile read, out write
    # ill-typed kernels must declare their extents; blockDim is CUDA's (<= 1024)
    with pytest.raises(mc.MapError) as e:
        mc.Kernel("A[tid] := tid; let x = A[tid] in A[x] := 9", block=(8, 1, 1))
    assert e.value.status == 8
    mc.Kernel("shared A[8]; A[tid] := tid; let x = A[tid] in A[x] := 9", block=(8, 1, 1))
    with pytest.raises(mc.MapError) as e:
        mc.Kernel("shared A[8]; A[0] := 1", block=(1025, 1, 1))
    assert e.value.status == 8
