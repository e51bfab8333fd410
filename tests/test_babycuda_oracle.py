"""Pins for the BabyCUDA oracle (oracle/babycuda.py) against things other than itself.

* the paper's displayed typing derivations and its ill-typed
  kernel (Eq. 1);
* the lastwrite / thread / par examples SPEC.md derives by hand from the rules
  of Fig. 5 (each marked [PAPER] or [DERIVED] there);
* closed forms of what the data-carrying workload kernels compute (a tree
  reduction sums, a transpose transposes, a scan prefix-sums);
* Theorem 1 as an executable property: for typable kernels
  the executed access values alpha equal the MAP's Lambda, where Lambda comes
  from the INDEPENDENT C++ MAP oracle (oracle/oracle.cpp) run on the inferred
  MAP text -- two implementations that share nothing but the paper;
* invariants: thread-order independence (rule par has no inter-thread
  premise), own-write visibility, context monotonicity, read-binder exclusion.
"""
import random

import pytest

import oracle
from oracle import babycuda as bc
from workloads import babycuda as wb

RD, WR = bc.RD, bc.WR


def strip(e):
    """An AST without source positions (tuples of strings/ints/lists only)."""
    if isinstance(e, tuple):
        return tuple(strip(x) for x in e if not (isinstance(x, tuple) and len(x) == 2 and
                                                  all(isinstance(v, int) for v in x)))
    if isinstance(e, list):
        return [strip(x) for x in e]
    return e


def lam(map_src, inst):
    recs = oracle.enumerate_accesses(map_src, inst.grid, inst.block, inst.params)
    return {tuple(int(x) for x in r) for r in recs}


# ------------------------------------------- the paper's derivations ------
def test_displayed_derivation_racy_loop():
    # {M, tid} |- for x in 0..M { rd y = A[x]; wr A[x] := y + 1 }
    #                   => forU x in 0..M { rd[x]; wr[x] }
    k = bc.parse(wb.PAPER["fig3_racy"])
    ty = bc.infer(k)
    assert ty.typable
    want = ("forU", "x", ("nat", 0), ("var", "M"), ("nat", 1),
            ("seq", [("acc", RD, "A", ("var", "x")), ("acc", WR, "A", ("var", "x"))]))
    assert strip(ty.protocol) == want


def test_displayed_derivation_drf_conditional():
    # {tid} |- if (tid = 0) { wr A[0] := tid } else { skip }
    #                   => if (tid = 0) { wr[0] } else { skip }
    ty = bc.infer(bc.parse(wb.PAPER["fig4_drf"]))
    assert ty.typable
    assert strip(ty.protocol) == ("if", ("rel", "=", ("tid",), ("nat", 0)), ("acc", WR, "A", ("nat", 0)), ("skip",))


def test_eq1_is_ill_typed_at_the_data_indexed_write():
    # wr A[tid] := tid; rd x = A[tid]; wr A[x] := 9 is NOT typable:
    # x, read from the array, indexes the write (the premise V |- n of t-write fails)
    ty = bc.infer(bc.parse(wb.PAPER["eq1_ill_typed"]))
    assert not ty.typable and ty.kind == bc.T_DATA_INDEX and ty.var == "x"
    src = wb.PAPER["eq1_ill_typed"]
    assert src[ty.col - 1:].startswith("x] := 9")
    st, _, _ = bc.infer_text(src)
    assert st == bc.S_TYPE


def test_eq1_false_alarm():
    # the data-abstracted MAP (read values arbitrary, Faial's view PAPER.md:880-885)
    # reports a race; the execution has none: each thread reads back its own write
    # (x = tid) and writes A[tid] -- the "dotted area" of PAPER.md:886
    src = wb.PAPER["eq1_ill_typed"]
    st, ty, m = bc.infer_text(src, domain=8)
    assert st == 0 and not ty.typable
    o = oracle.check(m, block=(8, 1, 1))
    assert o.status == 0 and o.verdict == 1
    r = bc.execute(src, block=(8, 1, 1), keep_memory=True)
    assert r.status == 0 and r.verdict == 0
    assert r.memory[0][0] == {i: 9 for i in range(8)}
    # soundness of the abstraction: every executed access value is in the abstract Lambda
    inst = wb.Instance("eq1", src, block=(8, 1, 1))
    assert r.alpha <= lam(m, inst)


def test_control_dependence_is_ill_typed():
    ty = bc.infer(bc.parse("let y = A[0] in if (y < 2) { A[1] := 0 } else { skip }"))
    assert not ty.typable and ty.kind == bc.T_DATA_CONTROL and ty.var == "y"
    ty = bc.infer(bc.parse("let y = A[0] in for x in 0..y { A[x] := 1 }"))
    assert not ty.typable and ty.kind == bc.T_DATA_CONTROL and ty.var == "y"
    # a read value in a payload is fine (t-write erases the payload)
    assert bc.infer(bc.parse("let y = A[0] in A[tid] := y * 2")).typable


# ------------------------------------------------ Fig. 5 rules (SPEC) -----
def test_lastwrite_rules():
    # lastwrite-undef, -curr, -prev (SPEC.md lastwrite examples)
    assert bc.lastwrite(("A", 0), []) is None
    assert bc.lastwrite(("A", 0), [{0: (set(), {("A", 0): 7})}]) == 7
    newest_first = [{1: (set(), {("A", 1): 9})}, {0: (set(), {("A", 0): 7})}]
    assert bc.lastwrite(("A", 0), newest_first) == 7          # prev, then curr
    assert bc.lastwrite(("A", 1), newest_first) == 9


def test_thread_records_drf_example():
    # SPEC.md eval_thread: Fig. 4 kernel, thread 0 -> (empty, {0 -> 0}); thread 1 -> (empty, empty)
    r = bc.execute(wb.PAPER["fig4_drf"], block=(2, 1, 1), keep_history=True)
    (P,) = r.history[0]
    assert P[0] == (set(), {("A", 0): 0})
    assert P[1] == (set(), {})


def test_par_racy_example_m1():
    # SPEC.md run: T = {0, 1}, M = 1, zero-initialised A: Q(0) = Q(1) = ({0}, {0 -> 1})
    r = bc.execute(wb.PAPER["fig3_racy"], block=(2, 1, 1), params={"M": 1}, keep_history=True)
    (P,) = r.history[0]
    assert P[0] == ({("A", 0)}, {("A", 0): 1}) and P[1] == ({("A", 0)}, {("A", 0): 1})
    assert r.uninit_reads == 2                  # both read bottom (R20: as 0)
    assert r.alpha == {(0, 0, 0, 0, t, o) for t in (0, 1) for o in (RD, WR)}
    assert r.witness == (0, 0, 0, 0, 0, 1, RD, WR)


def test_own_write_visibility():
    # rule read consults {i : (R, W)} :: H -- the thread's OWN current record, not the
    # other threads': each thread reads back its own tid + 1
    src = "shared A[4], B[8]; A[0] := tid + 1; let y = A[0] in B[tid] := y"
    r = bc.execute(src, block=(8, 1, 1), keep_memory=True)
    assert r.memory[0][1] == {i: i + 1 for i in range(8)}
    assert r.memory[0][0] == {0: 1}              # final lastwrite: smallest writer tid (R21)
    # another thread's write of the same phase is invisible: bottom (0), counted
    src2 = "shared A[8], B[8]; A[tid] := tid + 5; let y = A[(tid + 1) % 8] in B[tid] := y"
    r2 = bc.execute(src2, block=(8, 1, 1), keep_memory=True)
    assert r2.memory[0][1] == {i: 0 for i in range(8)} and r2.uninit_reads == 8
    # ... but visible after a barrier (lastwrite-prev then -curr)
    src3 = "shared A[8], B[8]; A[tid] := tid * 10; sync; let y = A[(tid + 1) % 8] in B[tid] := y"
    r3 = bc.execute(src3, block=(8, 1, 1), keep_memory=True)
    assert r3.memory[0][1] == {i: ((i + 1) % 8) * 10 for i in range(8)} and r3.uninit_reads == 0
    # an index written by two threads in the consulted phase: smallest tid, counted
    src4 = "shared A[8], B[8]; A[0] := tid + 3; sync; let y = A[0] in B[tid] := y"
    r4 = bc.execute(src4, block=(4, 1, 1), keep_memory=True)
    assert r4.memory[0][1] == {i: 3 for i in range(4)} and r4.ambiguous_reads == 4


# ---------------------------------------- closed forms of the data --------
@pytest.mark.parametrize("B", [2, 8, 64])
def test_reduction_sums(B):
    inst = wb.kernel("reduce", block=B, grid=2)
    r = bc.execute(inst.src, inst.grid, inst.block, inst.params, keep_memory=True)
    assert r.status == 0 and r.verdict == 0 and r.uninit_reads == 0
    for blk in range(2):
        assert r.memory[blk][0][0] == B * (B + 1) // 2


def test_transpose_transposes():
    inst = wb.kernel("transpose", ts=8, rw=4, grid=3)
    r = bc.execute(inst.src, inst.grid, inst.block, inst.params, keep_memory=True)
    assert r.status == 0 and r.verdict == 0
    for b in range(3):
        out = r.memory[b][1]
        assert out == {i * 8 + j: b * 64 + j * 8 + i for i in range(8) for j in range(8)}


@pytest.mark.parametrize("name,bs", [("hillis", 16), ("hillis", 64), ("hillis_inplace", 64)])
def test_scan_prefix_sums(name, bs):
    # all-ones input: the inclusive scan is i + 1.  In place (one element per thread) the
    # kernel is racy, yet the formal semantics -- other threads' in-phase writes are
    # invisible to a read -- still computes it
    inst = wb.kernel(name, n=64, bs=bs)
    r = bc.execute(inst.src, inst.grid, inst.block, inst.params, keep_memory=True)
    assert r.status == 0 and r.verdict == (1 if name == "hillis_inplace" else 0)
    N, D = 64, 6
    base = (D % 2) * N if name == "hillis" else 0
    mem = r.memory[0][0]
    assert [mem[base + i] for i in range(N)] == [i + 1 for i in range(N)]


# ------------------------------------------- Theorem 1 (executable) -------
def _theorem1(inst):
    st, ty, m = bc.infer_text(inst.src)
    assert st == 0 and ty.typable, (inst.src, ty)
    r = bc.execute(inst.src, inst.grid, inst.block, inst.params)
    o = oracle.check(m, inst.grid, inst.block, inst.params)
    return r, o, m


@pytest.mark.parametrize("name", wb.KERNELS)
def test_theorem1_workload_kernels(name):
    inst = wb.kernel(name)
    r, o, m = _theorem1(inst)
    assert r.status == 0 and o.status == 0
    assert r.alpha == lam(m, inst)                    # alpha in^ P  <=>  alpha in Lambda
    assert r.n_events == o.n_accesses                 # t-rules are homomorphic: same multiset size
    assert (r.verdict, r.witness, r.racy_segments) == (o.verdict, o.witness, o.n_racy_segments)


def test_theorem1_fuzz_typable():
    ran = 0
    for seed in range(300):
        inst, _ = wb.random_kernel(seed)
        st, ty, m = bc.infer_text(inst.src)
        assert st == 0 and ty.typable, (seed, inst.src)
        r = bc.execute(inst.src, inst.grid, inst.block, inst.params)
        o = oracle.check(m, inst.grid, inst.block, inst.params)
        if r.status != 0:                       # e.g. a payload overflow: no derivation to compare
            assert r.status in (bc.S_RANGE, bc.S_ARITH)
            continue
        assert o.status == 0, (seed, o.diag)
        ran += 1
        assert r.alpha == lam(m, inst), (seed, inst.src)
        assert r.n_events == o.n_accesses
        assert (r.verdict, r.witness, r.racy_segments) == (o.verdict, o.witness, o.n_racy_segments), seed
    assert ran >= 250


def test_ill_typed_fuzz_abstraction_is_sound():
    planted = 0
    for seed in range(300):
        inst, pl = wb.random_kernel(seed, ill_typed=True)
        st, ty, m = bc.infer_text(inst.src, domain=8)
        assert st == 0
        assert ty.typable == (not pl), (seed, inst.src)
        if not pl:
            continue
        planted += 1
        r = bc.execute(inst.src, inst.grid, inst.block, inst.params)
        o = oracle.check(m, inst.grid, inst.block, inst.params)
        if r.status != 0 or o.status != 0:
            continue
        assert r.alpha <= lam(m, inst), (seed, inst.src)
        assert r.verdict <= o.verdict                  # racy execution => racy abstraction
    assert planted >= 100


# ------------------------------------------------------- invariants -------
def test_thread_order_independence():
    rng = random.Random(7)
    for seed in range(0, 120, 3):
        for ill in (False, True):
            inst, _ = wb.random_kernel(seed, ill_typed=ill)
            a = bc.execute(inst.src, inst.grid, inst.block, inst.params, keep_memory=True)
            order = list(range(inst.n_threads))
            rng.shuffle(order)
            b = bc.execute(inst.src, inst.grid, inst.block, inst.params, thread_order=order, keep_memory=True)
            assert (a.status, a.alpha, a.memory, a.uninit_reads, a.ambiguous_reads) == \
                   (b.status, b.alpha, b.memory, b.uninit_reads, b.ambiguous_reads), seed


def test_context_monotonicity_and_binder_exclusion():
    for seed in range(100):
        inst, _ = wb.random_kernel(seed)
        k = bc.parse(inst.src)
        u = bc.infer(k).protocol
        k2 = bc.parse("params ZZ9; " + inst.src) if not inst.params else None
        if k2 is not None:
            assert strip(bc.infer(k2).protocol) == strip(u)
        # no read binder occurs in an index or condition of the inferred MAP
        binders = set()

        def walk_k(s):
            if s[0] == "let":
                binders.add(s[1])
                walk_k(s[4])
            elif s[0] == "seq":
                for x in s[1]:
                    walk_k(x)
            elif s[0] == "if":
                walk_k(s[2])
                walk_k(s[3])
            elif s[0] == "for":
                walk_k(s[5])
        walk_k(k.body)
        text = bc.map_text(k, u)
        assert not any(f" {y}" in text or f"[{y}" in text or f"({y}" in text for y in binders), (seed, text)


@pytest.mark.parametrize("src,status", [
    ("if (tid = 0) { sync } else { skip }", bc.S_BARRIER),
    ("for x in 0..tid { A[x] := 1; sync }", bc.S_BARRIER),
    ("let y = A[0] in for x in 0..y { sync }", bc.S_BARRIER),
    ("A[q] := 1", bc.S_SCOPE),
    ("for x in 0..2 { for x in 0..2 { A[x] := 1 } }", bc.S_SCOPE),
    ("let tid2 = A[0] in let tid2 = A[1] in skip", bc.S_SCOPE),
    ("if (tid = 0) { A[0] := 1 }", bc.S_PARSE),
    ("A[0] = 1", bc.S_PARSE),
    ("A[18446744073709551616] := 1", bc.S_RANGE),
])
def test_static_errors(src, status):
    with pytest.raises(bc.BcError) as e:
        bc.parse(src)
    assert e.value.status == status


def test_runtime_errors():
    assert bc.execute("A[1 / (tid - tid)] := 0", block=(2, 1, 1)).status == bc.S_ARITH
    assert bc.execute("let y = A[0] in A[1] := y / 0", block=(2, 1, 1)).status == bc.S_ARITH
    assert bc.execute("A[0] := 18446744073709551615 + tid", block=(2, 1, 1)).status == bc.S_RANGE
    assert bc.execute("shared A[4]; A[tid] := 1", block=(5, 1, 1)).status == bc.S_RANGE
    assert bc.execute("shared A[4]; A[tid] := 1", block=(4, 1, 1)).status == 0


def test_inplace_scan_sees_own_writes():
    # with 4 elements per thread, element 32 + t reads element t at d = 5, which thread t
    # itself wrote earlier in the same phase: own writes ARE visible (rule read), so the
    # racy in-place scan diverges from the prefix sums exactly there
    inst = wb.kernel("hillis_inplace", n=64, bs=16)
    r = bc.execute(inst.src, inst.grid, inst.block, inst.params, keep_memory=True)
    mem = r.memory[0][0]
    assert [mem[i] for i in range(32)] == [i + 1 for i in range(32)]
    assert mem[32] == 34 and r.verdict == 1
