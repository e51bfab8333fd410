"""Pins for the CPU oracle (oracle/oracle.cpp) against things other than itself.

* the paper's worked examples and the values SPEC.md prints for them
  (tests/golden/paper_examples.json, each entry cited);
* closed forms of the access counts and of the canonical witnesses of the five
  BASELINE.json configs (derivations in DESIGN.md §6);
* the L0 brute force (tests/brute.py): configs hand-written as Python loops and
  a direct evaluator of the fuzz AST, with the race test done over all pairs;
* invariants (thread-count independence, monotonicity, one thread => DRF).
"""
import json
import os

import numpy as np
import pytest

import oracle
from tests import brute
from workloads import config, fuzz

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
RD, WR = 0, 1


def _check(inst, threads=2):
    r = oracle.check_instance(inst, threads=threads)
    assert r.status == 0, r.diag
    return r


# ---------------------------------------------------------------- golden ----
with open(os.path.join(GOLDEN, "paper_examples.json")) as f:
    PAPER_EXAMPLES = json.load(f)


@pytest.mark.parametrize("ex", PAPER_EXAMPLES, ids=[e["name"] for e in PAPER_EXAMPLES])
def test_paper_examples(ex):
    r = oracle.check(ex["src"], ex["grid"], ex["block"], ex["params"], threads=1)
    assert r.status == 0, r.diag
    assert r.verdict == (1 if ex["verdict"] == "racy" else 0)
    recs = oracle.enumerate_accesses(ex["src"], ex["grid"], ex["block"], ex["params"])
    values = {(int(t), "wr" if k else "rd", int(ix)) for (_, _, _, ix, t, k) in recs}
    if "accesses" in ex:
        assert values == {tuple(a) for a in ex["accesses"]}
    if "n_access_values" in ex:
        assert len(values) == ex["n_access_values"]


def test_fig3_racy_pair_wr_wr_at_index0():
    # races_of(Lambda of Fig. 3, T={0,1}, M=1) includes the wr/wr
    # pair at index 0; the canonical witness is the smallest pair, (0 rd, 1 wr).
    r = oracle.check("params M; forU x in 0..M { rd[x]; wr[x] }", block=(2, 1, 1), params={"M": 1})
    assert r.witness == (0, 0, 0, 0, 0, 1, RD, WR)
    assert r.n_racy_segments == 1


# --------------------------------------------------- closed-form counts -----
def n_closed(name, inst):
    p, B, G = inst.params, inst.n_threads, inst.n_blocks
    if name == "1a":
        return 2 * B * p["M"]
    if name == "1b":
        return 1
    if name[0] == "2":
        return B + 3 * (B - 1)
    if name[0] == "3":
        return G * p["TS"] * p["TS"] * 2
    n, L = p.get("N"), p.get("D")
    if name == "4a":
        return 3 * n * L - (n - 1)
    if name == "4b":
        return 3 * n * L - 3 * (n - 1)
    if name in ("4c", "4d"):
        return 9 * n - 7
    if name[0] == "5":
        return 4 * p["T"] * p["R"] * p["C"] * B


SCALED = {
    "1a": [dict(block=8, M=8), dict(block=3, M=5), dict(block=1, M=4), dict(block=4, M=0)],
    "1b": [dict(block=8), dict(block=1)],
    "2a": [dict(block=1024), dict(block=16), dict(block=2)],
    "2b": [dict(block=1024), dict(block=16), dict(block=4), dict(block=2)],
    "2c": [dict(block=1024), dict(block=16), dict(block=2)],
    "3a": [dict(ts=32, rw=8, grid=64), dict(ts=8, rw=2, grid=3)],
    "3b": [dict(ts=32, rw=8, grid=64), dict(ts=8, rw=2, grid=3), dict(ts=2, rw=1, grid=1)],
    "4a": [dict(n=1 << 14, bs=1024), dict(n=64, bs=8)],
    "4b": [dict(n=1 << 14, bs=1024), dict(n=64, bs=8)],
    "4c": [dict(n=1 << 14, bs=1024), dict(n=64, bs=8), dict(n=4, bs=2)],
    "4d": [dict(n=1 << 14, bs=1024), dict(n=64, bs=8), dict(n=4, bs=2)],
    "5a": [dict(block=64, T=3, R=4, C=8), dict(block=8, T=2, R=1, C=3)],
    "5b": [dict(block=64, T=3, R=4, C=8), dict(block=8, T=2, R=1, C=3), dict(block=2, T=1, R=2, C=2)],
}
CASES = [(n, s) for n, ss in SCALED.items() for s in ss]


def witness_closed(name, inst):
    """Canonical witness (phase, array, block, index, t_lo, t_hi, k_lo, k_hi) or None."""
    p, B = inst.params, inst.n_threads
    if name == "1a":
        return (0, 0, 0, 0, 0, 1, RD, WR) if B >= 2 and p["M"] >= 1 else None
    if name in ("1b", "2a", "3a", "4a", "4c", "5a"):
        return None
    if name == "2b":
        return (1, 0, 0, 1, 0, 1, RD, WR) if B >= 4 else None
    if name == "2c":
        return (0, 0, 0, B // 2, 0, B // 2, RD, WR) if B >= 2 else None
    if name == "3b":
        # index 1 is written by tid 1 (j=0) and read by the thread with
        # tid%TS = 0, tid/TS + j = 1: tid TS (j=0) when RW >= 2, else tid 0 (j=1)
        return (0, 0, 0, 1, 1, p["TS"], WR, RD) if p["RW"] >= 2 else (0, 0, 0, 1, 0, 1, RD, WR)
    if name == "4b":
        return (0, 0, 0, 1, 1, 2, WR, RD)
    if name == "4d":
        return (p["D"] + 2, 0, 0, 3, 0, 1, RD, WR)
    if name == "5b":
        return (0, 0, 0, 0, 0, 1 if p["R"] == 1 else B - 1, WR, RD)


def racy_closed(name, inst):
    """Racy (phase, array, block, index) cells of the stencil configs.  5a: none
    (ping-pong halves; each cell of the write half has one writer and no reader).
    5b (in place): row tid*R is read by the owner of row tid*R - 1 (its r+1
    neighbour) and row tid*R + R - 1 by the owner of row tid*R + R (its r-1
    neighbour); every other row is touched by its owner only.  So min(R, 2)
    racy rows of C cells per thread per phase, when there are >= 2 threads."""
    p, B = inst.params, inst.n_threads
    if name == "5a":
        return 0
    if name == "5b":
        return p["T"] * B * p["C"] * min(p["R"], 2) if B >= 2 else 0
    raise KeyError(name)


@pytest.mark.parametrize("sizes", [dict(block=2, T=1, R=1, C=3), dict(block=4, T=2, R=3, C=5),
                                   dict(block=8, T=3, R=2, C=4), dict(block=1, T=2, R=3, C=2),
                                   dict(block=16, T=1, R=5, C=7)])
@pytest.mark.parametrize("name", ["5a", "5b"])
def test_stencil_racy_count_closed_form(name, sizes):
    # pinned against the L0 brute force's all-pairs count and the oracle
    inst = config(name, **sizes)
    r = _check(inst)
    assert r.n_racy_segments == racy_closed(name, inst)
    assert len(brute.race_list(brute.config_records(inst))) == racy_closed(name, inst)


def test_and_or_evaluate_both_operands():
    # DESIGN.md R2 (P:201 leaves the boolean operators unspecified): both operands
    # of and/or are evaluated, so the division by zero in the right operand is
    # reached even though the left one already decides the condition
    for src in ["if (tid = 9 and 1 / (tid - tid) = 0) { wr[0] } else { skip }",
                "if (tid < 9 or 1 % (tid - tid) = 0) { wr[0] } else { skip }"]:
        assert oracle.check(src, block=(4, 1, 1)).status == 5
    # without the faulting operand both are plain conditions
    r = oracle.check("if (tid = 2 or tid = 3) { wr[0] } else { skip }", block=(4, 1, 1))
    assert r.status == 0 and r.witness == (0, 0, 0, 0, 2, 3, WR, WR)


def test_literal_bounds():
    # naturals are exact u64 (R3): 2^64 - 1 is a literal, 2^64 is not
    r = oracle.check("rd[18446744073709551615 - tid]", block=(2, 1, 1))
    assert r.status == 0 and r.n_accesses == 2 and r.verdict == 0
    assert oracle.check("rd[18446744073709551616]", block=(2, 1, 1)).status == 4


@pytest.mark.parametrize("name,sizes", CASES, ids=[f"{n}-{i}" for i, (n, _) in enumerate(CASES)])
def test_closed_forms(name, sizes):
    inst = config(name, **sizes)
    r = _check(inst)
    assert r.n_accesses == n_closed(name, inst)
    assert r.witness == witness_closed(name, inst)
    assert r.verdict == (r.witness is not None)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["1a", "1b", "2a", "2b", "2c", "4c", "4d"])
def test_full_size_closed_forms(name):
    inst = config(name)
    r = _check(inst, threads=os.cpu_count())
    assert r.n_accesses == n_closed(name, inst)
    assert r.witness == witness_closed(name, inst)


# ---------------------------------------------------- L0 brute force --------
BRUTE_CASES = [(n, s) for n, s in CASES if brute.config_records(config(n, **s)) is not None
               and len(brute.config_records(config(n, **s))) <= 40000]


@pytest.mark.parametrize("name,sizes", BRUTE_CASES, ids=[f"{n}-{i}" for i, (n, _) in enumerate(BRUTE_CASES)])
def test_configs_vs_hand_loops(name, sizes):
    inst = config(name, **sizes)
    recs = brute.config_records(inst)
    v, w, nseg, n = brute.races(recs)
    r = _check(inst)
    assert (r.verdict, r.witness, r.n_racy_segments, r.n_accesses) == (v, w, nseg, n)
    # and the multiset of accesses itself
    got = oracle.enumerate_accesses(inst.src, inst.grid, inst.block, inst.params)
    want = np.array(sorted(recs), dtype=np.uint64).reshape(-1, 6)
    got = got[np.lexsort(got.T[::-1])]
    np.testing.assert_array_equal(got, want)


def test_all_pairs_agrees_with_grouped_pairs():
    # the grouped naive pair test in brute.races equals the O(N^2) definition
    for name, sizes in [("1a", dict(block=3, M=4)), ("2b", dict(block=8)), ("3b", dict(ts=4, rw=2, grid=2)),
                        ("4b", dict(n=16, bs=4)), ("5b", dict(block=4, T=1, R=2, C=2))]:
        recs = brute.config_records(config(name, **sizes))
        v, w, _, _ = brute.races(recs)
        assert brute.races_all_pairs(recs) == (v, w)


N_FUZZ = int(os.environ.get("MAPCHECK_FUZZ", "1500"))


def test_fuzz_vs_brute():
    mismatches = []
    n_racy = 0
    for seed in range(N_FUZZ):
        inst, prog = fuzz.random_instance(seed)
        recs = brute.eval_ast(prog, inst.grid, inst.block, inst.params)
        v, w, nseg, n = brute.races(recs)
        r = oracle.check_instance(inst, threads=1)
        n_racy += v
        if r.status != 0 or (r.verdict, r.witness, r.n_racy_segments, r.n_accesses) != (v, w, nseg, n):
            mismatches.append((seed, inst.src, r, (v, w, nseg, n)))
    assert not mismatches, mismatches[:3]
    # the corpus must exercise both verdicts
    assert 0.1 * N_FUZZ < n_racy < 0.9 * N_FUZZ


# ------------------------------------------- race listing (NEXT-4) ---------
@pytest.mark.parametrize("name,sizes", BRUTE_CASES, ids=[f"{n}-{i}" for i, (n, _) in enumerate(BRUTE_CASES)])
def test_race_list_vs_hand_loops(name, sizes):
    # SPEC.md:434-437 races_of, one minimal pair per racy segment: the oracle's list
    # equals the naive per-cell pair test over the hand-written loops
    inst = config(name, **sizes)
    recs = brute.config_records(inst)
    assert oracle.list_races_instance(inst) == brute.race_list(recs)


def test_race_list_fuzz_vs_brute():
    bad = []
    for seed in range(0, N_FUZZ, 3):
        inst, prog = fuzz.random_instance(seed)
        recs = brute.eval_ast(prog, inst.grid, inst.block, inst.params)
        got = oracle.list_races_instance(inst, threads=1)
        if got != brute.race_list(recs):
            bad.append((seed, inst.src))
    assert not bad, bad[:3]


def test_race_list_invariants():
    for name, sizes in [("2b", dict(block=64)), ("3b", dict(ts=8, rw=2, grid=3)), ("4b", dict(n=256, bs=16)),
                        ("5b", dict(block=8, T=2, R=2, C=8)), ("2a", dict(block=64))]:
        inst = config(name, **sizes)
        r = oracle.check_instance(inst)
        lst = oracle.list_races_instance(inst)
        assert len(lst) == r.n_racy_segments
        assert lst == sorted(lst) and len(set(x[:4] for x in lst)) == len(lst)   # one entry per cell
        assert (lst[0] if lst else None) == r.witness
        for (_, _, _, _, tlo, thi, klo, khi) in lst:
            assert tlo < thi and (klo == 1 or khi == 1)


# ------------------------------------------------------------ invariants ----
def test_thread_count_independence():
    for name, sizes in [("3b", dict(ts=8, rw=2, grid=5)), ("4d", dict(n=256, bs=16)), ("5b", dict(block=16, T=2, R=2, C=4))]:
        inst = config(name, **sizes)
        a = oracle.check_instance(inst, threads=1)
        b = oracle.check_instance(inst, threads=7)
        assert (a.verdict, a.witness, a.n_racy_segments, a.n_accesses) == \
               (b.verdict, b.witness, b.n_racy_segments, b.n_accesses)


def test_single_thread_is_drf():
    for seed in range(200):
        inst, _ = fuzz.random_instance(seed)
        r = oracle.check(inst.src, (1, 1, 1), (1, 1, 1), inst.params, threads=1)
        assert r.status == 0 and r.verdict == 0


def test_adding_accesses_only_lowers_witness():
    # races are monotone under adding accesses
    base = "params M; forU x in 0..M { rd[x + 1] }; wr[tid]"
    r0 = oracle.check(base, block=(4, 1, 1), params={"M": 3})
    r1 = oracle.check(base + "; wr[0]", block=(4, 1, 1), params={"M": 3})
    assert r0.verdict == 1 and r1.verdict == 1
    assert r1.witness <= r0.witness
    assert r1.n_racy_segments >= r0.n_racy_segments


def test_sync_only_removes_races():
    racy = "wr[tid]; rd[(tid + 1) % 8]"
    assert oracle.check(racy, block=(8, 1, 1)).verdict == 1
    assert oracle.check("wr[tid]; sync; rd[(tid + 1) % 8]", block=(8, 1, 1)).verdict == 0


def test_blocks_are_independent():
    # shared arrays are per block (reading R10): no cross-block race
    assert oracle.check("wr[0]", grid=(4, 1, 1), block=(1, 1, 1)).verdict == 0
    r = oracle.check("wr[0]", grid=(3, 1, 1), block=(2, 1, 1))
    assert r.witness == (0, 0, 0, 0, 0, 1, WR, WR) and r.n_racy_segments == 3


def test_arrays_are_independent():
    r = oracle.check("shared A, B; wr A[tid]; wr B[0]", block=(2, 1, 1))
    assert r.witness == (0, 1, 0, 0, 0, 1, WR, WR)
    assert oracle.array_names("shared A, B; skip") == ["A", "B"]


def test_monus_and_operators():
    # index arithmetic on naturals: monus, floor division, shifts, min/max
    src = "rd[(tid - 3) + (7 / 2) * 10 + (5 % 3) + (1 << 4) + (64 >> 3) + min(tid, 2) + max(tid, 9)]"
    recs = oracle.enumerate_accesses(src, block=(5, 1, 1))
    for t in range(5):
        want = max(t - 3, 0) + 30 + 2 + 16 + 8 + min(t, 2) + max(t, 9)
        assert int(recs[t, 3]) == want


def test_precedence():
    recs = oracle.enumerate_accesses("rd[1 + 2 * 3 << 1]; rd[8 - 2 - 1]; rd[2 * (3 + 1)]")
    assert [int(x) for x in recs[:, 3]] == [14, 5, 8]


def test_step_loops():
    recs = oracle.enumerate_accesses("forU j in 1..10 step 3 { rd[j] }")
    assert [int(x) for x in recs[:, 3]] == [1, 4, 7]


def test_if_without_else_is_skip():
    a = oracle.enumerate_accesses("if (tid < 2) { wr[tid] }", block=(4, 1, 1))
    b = oracle.enumerate_accesses("if (tid < 2) { wr[tid] } else { skip }", block=(4, 1, 1))
    np.testing.assert_array_equal(a, b)


def test_conditions_parse():
    src = "if ((tid + 1) < 3 and (tid = 0 or tid = 1)) { wr[0] }"
    recs = oracle.enumerate_accesses(src, block=(4, 1, 1))
    assert sorted(int(t) for t in recs[:, 4]) == [0, 1]


# ---------------------------------------------------------------- errors ----
@pytest.mark.parametrize("src,status", [
    ("rd[", 1), ("forU x 0..3 { rd[x] }", 1), ("rd[x]", 2), ("rd Q[0]", 2),
    ("forU x in 0..2 { forU x in 0..2 { rd[x] } }", 2),
    ("if (tid = 0) { sync } else { skip }", 3), ("forU x in 0..2 { sync }", 3),
    ("forS x in 0..tid { sync }", 3), ("rd[1 / (tid - tid)]", 5),
    ("forU x in 0..3 step 0 { rd[x] }", 5), ("rd[18446744073709551615 + 1]", 4),
])
def test_errors(src, status):
    r = oracle.check(src, block=(2, 1, 1))
    assert r.status == status, r


def test_param_errors():
    assert oracle.check("params M; rd[M]").status == 8
    assert oracle.check("rd[0]", params={"Q": 1}).status == 8
