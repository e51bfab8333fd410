"""The cell code of the direct-address detect (include/mapcheck.h
MAP_DETECT_DIRECT), checked against the definition it replaces -- no GPU.

A cell is racy iff it holds a write and two DISTINCT tids (
same-thread pairs never race, R11).  The kernels keep per cell only
the bitwise OR of code(t, k) = t | (~t & M) << wt | k << 2wt over its
accesses.  Claim: (OR t) & (OR ~t) & M != 0  <=>  the tids are not all equal.
Brute force over every nonempty tid set for wt <= 4 (all 2^16 - 1 subsets of
16 tids), plus random multisets with kinds for larger wt, against the plain
definition (some pair of accesses with different tids, one of them a write).
"""
import itertools
import random

import pytest


def code(t, k, wt):
    m = (1 << wt) - 1
    return t | ((~t & m) << wt) | (k << (2 * wt))


def racy_from_cell(c, wt):
    m = (1 << wt) - 1
    return bool((c >> (2 * wt)) & 1) and (c & (c >> wt) & m) != 0


def racy_by_definition(accs):
    return any(t1 != t2 and (k1 or k2) for (t1, k1), (t2, k2) in itertools.combinations(accs, 2))


@pytest.mark.parametrize("wt", [0, 1, 2, 3, 4])
def test_two_distinct_tids_exhaustive(wt):
    n = 1 << wt
    m = (1 << wt) - 1
    for mask in range(1, 1 << n):
        tids = [t for t in range(n) if mask >> t & 1]
        a = b = 0
        for t in tids:
            a |= t
            b |= ~t & m
        assert ((a & b) != 0) == (len(tids) >= 2)


@pytest.mark.parametrize("wt", [1, 5, 10, 15, 16, 31])
def test_cell_code_matches_race_definition(wt):
    rng = random.Random(1000 + wt)
    for _ in range(3000):
        n = rng.randint(1, 6)
        pool = [rng.randrange(1 << wt) for _ in range(rng.randint(1, 3))]
        accs = [(rng.choice(pool), rng.random() < 0.3) for _ in range(n)]
        c = 0
        for t, k in accs:
            c |= code(t, int(k), wt)
        assert racy_from_cell(c, wt) == racy_by_definition(accs)
    # the code fits the cell: 2 wt + 1 bits (u32 cells up to wt = 15)
    assert code((1 << wt) - 1, 1, wt) < (1 << (2 * wt + 1))


# ---- the 16-bit cell code (blockDim <= 1024; devabi.h code16) ---------------
# Written from its definition, independently of the kernels: each 5-bit digit of the
# tid maps to one of the 32 smallest 7-bit words with exactly three ones.
CW7 = [x for x in range(128) if bin(x).count("1") == 3][:32]


def code16(t, k):
    return CW7[t & 31] | (CW7[(t >> 5) & 31] << 7) | (k << 14)


def racy16(c):
    return bool((c >> 14) & 1) and (bin(c & 0x7F).count("1") > 3 or bin((c >> 7) & 0x7F).count("1") > 3)


def test_code16_distinct_pairs_exhaustive():
    # any two distinct tids < 1024 -> the OR has a digit field with popcount > 3;
    # one tid alone (any number of times) -> every field has popcount exactly 3
    import numpy as np
    t = np.arange(1024)
    lo = np.array([CW7[x & 31] for x in t])
    hi = np.array([CW7[(x >> 5) & 31] for x in t])
    pc = np.vectorize(lambda v: bin(int(v)).count("1"))
    orlo = lo[:, None] | lo[None, :]
    orhi = hi[:, None] | hi[None, :]
    multi = (pc(orlo) > 3) | (pc(orhi) > 3)
    assert (multi == ~np.eye(1024, dtype=bool)).all()
    assert all(bin(code16(x, 0)).count("1") == 6 for x in range(1024))
    assert code16(1023, 1) < (1 << 16)


def test_code16_matches_race_definition():
    rng = random.Random(16)
    for _ in range(5000):
        pool = [rng.randrange(1024) for _ in range(rng.randint(1, 3))]
        accs = [(rng.choice(pool), rng.random() < 0.3) for _ in range(rng.randint(1, 6))]
        c = 0
        for t, k in accs:
            c |= code16(t, int(k))
        assert racy16(c) == racy_by_definition(accs)


def test_racy16_word_swar_exhaustive():
    # the scan's POPC-free test of two 16-bit cells per 32-bit word (direct.cu
    # racy16_word, exported for this check) against racy16 above: every value of
    # each cell with the other cell 0 or a random value, and random word pairs
    import ctypes
    import paper_2203_12878_b200 as mc
    f = mc._lib.mapc_test_racy16_word
    f.argtypes = [ctypes.c_uint32]
    f.restype = ctypes.c_uint32
    rng = random.Random(7)
    for c in range(1 << 16):
        other = rng.randrange(1 << 16)
        for w, want in ((c, racy16(c)), (c << 16, racy16(c)),
                        (c | (other << 16), racy16(c) or racy16(other)),
                        (other | (c << 16), racy16(c) or racy16(other))):
            assert (f(w) != 0) == want, hex(w)
        # lane-exact: bytes 0-1 of the result belong to the low cell, 2-3 to the high
        # one (the unit scan counts racy cells from the halves: jit.cpp racy16w)
        for w in (c | (other << 16), other | (c << 16)):
            r = f(w)
            assert ((r & 0xFFFF) != 0) == racy16(w & 0xFFFF), hex(w)
            assert ((r >> 16) != 0) == racy16(w >> 16), hex(w)


def test_jit_prelude_racy16w_is_racy16_word():
    """The NVRTC prelude's copy of the SWAR test (jit.cpp racy16w, used by the unit
    scan) is the same function as direct.cu's racy16_word checked above: same
    statements once the type names and the named kind-bit temporary are normalised."""
    import os
    import re
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    a = open(os.path.join(root, "paper_2203_12878_b200", "csrc", "capi", "jit.cpp")).read()
    b = open(os.path.join(root, "paper_2203_12878_b200", "csrc", "kernels", "direct.cu")).read()
    fa = re.search(r"u32 racy16w\(u32 w\) \{(.*?)\n\}", a, re.S).group(1)
    fb = re.search(r"uint32_t racy16_word\(uint32_t w\) \{(.*?)\n\}", b, re.S).group(1)

    def norm(t):
        t = re.sub(r"//[^\n]*", "", t).replace("uint32_t", "u32")
        t = t.replace("const u32 k = (w >> 14) & 0x00010001u;", "").replace("(k * 0x7F7Fu)",
                                                                           "(((w >> 14) & 0x00010001u) * 0x7F7Fu)")
        return re.sub(r"\s+", "", t)
    assert norm(fa) == norm(fb)
