"""CPU tests of the C-ABI library: it loads, exports every symbol the header
declares, its host compiler agrees with the oracle on static facts and error
classes, and the run entry point fails loudly without a GPU (no CPU fallback)."""
import os
import random
import re

import pytest

import oracle
import paper_2203_12878_b200 as mc
from tests.test_oracle import CASES, n_closed
from workloads import config, fuzz

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    with open(os.path.join(ROOT, "include", "mapcheck.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:map_status|size_t|void|uint64_t|int|const char \*)\s*\**\s*(map_\w+)\s*\(", text, re.M)))


def test_header_symbols_exported():
    names = declared_functions()
    assert len(names) >= 10, names
    for n in names:
        assert hasattr(mc._lib, n), f"{n} declared in include/mapcheck.h but not exported"
    assert set(mc.EXPORTS) <= set(names)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", mc.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings():
    assert mc.status_str(0) == "ok"
    assert "parse" in mc.status_str(1)


@pytest.mark.parametrize("n,d", [(0, 1), (7, 3), (2**32 - 1, 3), (2**32 - 1, 7), (123456789, 1000),
                                 (2**32 - 1, 2**31 + 1), (2**31, 3), (99, 100), (5, 5)])
def test_fastdiv_edges(n, d):
    assert mc.fastdiv_selftest(n, d) == n // d


def test_fastdiv_random():
    r = random.Random(1)
    for _ in range(20000):
        d = r.choice([r.randint(1, 100), r.randint(1, 2**16), r.randint(1, 2**32 - 1)])
        n = r.choice([r.randint(0, 2**32 - 1), r.randint(0, 1000), d * r.randint(0, 2**32 // d) - r.randint(0, 1)])
        n = max(0, min(n, 2**32 - 1))
        assert mc.fastdiv_selftest(n, d) == n // d, (n, d)


@pytest.mark.parametrize("name,sizes", CASES, ids=[f"{n}-{i}" for i, (n, _) in enumerate(CASES)])
def test_compile_bounds_cover_exact_counts(name, sizes):
    inst = config(name, **sizes)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    info = p.info
    assert info.max_accesses >= n_closed(name, inst)
    assert p.scratch_bytes() > 0
    assert p.n_chunks() >= (1 if n_closed(name, inst) else 0)


def test_full_size_plans():
    # 2^34-access stencil: one chunk per barrier phase at the default 2^30-key chunk
    inst = config("5a")
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    assert p.info.max_accesses == 2**34
    assert p.info.u32_mode
    assert p.n_chunks() == 16
    # a larger capacity does not merge phases: two phases would double the
    # direct-address table of a chunk (4 GiB) for no saving per access
    assert p.n_chunks(2**31) == 16


def test_plans_keep_direct_tables_l2_sized():
    # Hillis-Steele scan (20 phases x ~3M accesses): once a chunk holds >= 2^23 accesses
    # it is closed before its table would reach 2^24 cells (64 MiB of u32 cells)
    inst = config("4a")
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    infos = [p.chunk_info(c) for c in range(p.n_chunks())]
    assert len(infos) > 1
    assert all(i["sort_bits"] < 24 for i in infos)
    assert sum(i["phase_hi"] - i["phase_lo"] + 1 for i in infos) == p.info.n_phases - 1 or \
        sum(i["phase_hi"] - i["phase_lo"] + 1 for i in infos) == p.info.n_phases


@pytest.mark.parametrize("src,status", [
    ("rd[", 1), ("forU x 0..3 { rd[x] }", 1), ("rd[x]", 2), ("rd Q[0]", 2),
    ("forU x in 0..2 { forU x in 0..2 { rd[x] } }", 2),
    ("if (tid = 0) { sync } else { skip }", 3), ("forU x in 0..2 { sync }", 3),
    ("forS x in 0..tid { sync }", 3), ("rd[18446744073709551615 + 1]", 4), ("rd[18446744073709551616]", 4),
    ("forS x in 0..(1 / 0) { sync }", 5),
])
def test_compile_errors_match_oracle(src, status):
    o = oracle.check(src, block=(2, 1, 1))
    assert o.status == status
    with pytest.raises(mc.MapError) as e:
        mc.MapProgram(src, block=(2, 1, 1))
    assert e.value.status == status


def test_param_errors():
    with pytest.raises(mc.MapError) as e:
        mc.MapProgram("params M; rd[M]")
    assert e.value.status == 8
    with pytest.raises(mc.MapError) as e:
        mc.MapProgram("rd[0]", params={"Q": 1})
    assert e.value.status == 8


def test_fuzz_corpus_compiles():
    for seed in range(500):
        inst, _ = fuzz.random_instance(seed)
        p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
        o = oracle.check_instance(inst, threads=1)
        assert o.status == 0
        assert p.info.max_accesses >= o.n_accesses, (seed, inst.src)


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="needs a machine without a GPU")
def test_no_cpu_fallback():
    p = mc.MapProgram("wr[0]", block=(2, 1, 1))
    with pytest.raises(mc.MapError) as e:
        p.check_races()
    assert e.value.status == 6


def test_guard_refinement_tightens_layouts():
    # Inside `if (k*1024 + tid < (N >> (l+1)))` the compiler narrows k*1024 + tid, so the
    # Blelloch scan's indices (1 << l)*(2*(k*1024+tid)+1) - 1 stay below N = 2^20: the sort
    # field is phase + 20 index bits, not the bounding box's 2^30-wide hull.
    inst = config("4c")
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    info = p.chunk_info(0)
    assert info["sort_bits"] <= 6 + 20
    # the unguarded stencil keeps its exact 29-bit index field
    inst = config("5a")
    assert mc.MapProgram(inst.src, inst.grid, inst.block, inst.params).chunk_info(0)["sort_bits"] == 29


def test_guard_refinement_unreachable_branch():
    # a guard that no tuple satisfies (tid < 64 and tid >= 64) leaves no access behind it
    p = mc.MapProgram("if (tid < 64) { if (tid >= 64) { wr[tid] } else { skip } } else { skip }; rd[0]",
                      (1, 1, 1), (128, 1, 1), {})
    assert p.info.max_accesses == 128


def test_sparse_group_split_by_constant_loop():
    # Blelloch down-sweep with forU levels (4d): (N >> (l+1))*(2*(k*1024+tid)+1) - 1 couples l
    # in two factors; the group is split per value of l, so every part's hull is exact and the
    # whole MAP gets one dense chunk (sort field: 5 phase bits + 20 index bits)
    inst = config("4d")
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    assert p.n_chunks() == 1
    assert p.chunk_info(0)["sort_bits"] <= 5 + 21
    assert p.info.max_accesses >= 9 * 2**20 - 7


def _dump(p):
    import ctypes
    n = mc._lib.map_debug_dump(p._h, None, 0)
    buf = ctypes.create_string_buffer(n + 1)
    mc._lib.map_debug_dump(p._h, buf, n + 1)
    return [line for line in buf.value.decode().splitlines() if line.startswith("instance")]


def test_tuple_order_choice():
    # the compiler puts the coordinate with the unit-stride index innermost:
    # the stencil's column loop c for 5a, tid for the scans' `k*1024 + tid`
    for name, want in (("5a", False), ("4a", True)):
        inst = config(name)
        groups = _dump(mc.MapProgram(inst.src, inst.grid, inst.block, inst.params))
        assert groups and all(("tid_inner" in g) == want for g in groups), (name, groups[:2])


def _us_flags(src, params, block=(64, 1, 1)):
    p = mc.MapProgram(src, (1, 1, 1), block, params)
    m = re.search(r"constexpr bool US_\[\d+\] = \{([^}]*)\}", p.jit_source(0, mode=1))
    assert m, "direct-mode source without unit-stride flags"
    return [x.strip() == "true" for x in m.group(1).split(",")]


def test_unit_stride_sites():
    # the paired 16-bit generate skips the run-time adjacency test only for sites
    # whose index is X + c (c the innermost coordinate, X independent of c);
    # anything else keeps the test
    inst = config("5a")
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    m = re.search(r"constexpr bool US_\[\d+\] = \{([^}]*)\}", p.jit_source(0, mode=1))
    assert m and [x.strip() for x in m.group(1).split(",")] == ["true"] * 4
    # tid innermost (the scans' k * 1024 + tid): the tid advances by h instead
    inst = config("4a")
    src4 = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params).jit_source(0, mode=1)
    assert re.search(r"constexpr bool US_\[\d+\] = \{[^}]*true", src4)
    head = "params C; shared A;\nforU r in 0..4 {\n  forU c in 0..C {\n    "
    tail = "\n  }\n}"
    cases = [
        ("rd A[tid * 4 * C + r * C + c + 5]", [True]),
        ("rd A[tid * 4 * C + r * C + 2 * c]", [False]),
        ("rd A[tid * 4 * C + r * C + (c + 1) % C]", [False]),
        ("rd A[tid * 4 * C + r * C + c * 1 + c]", [False]),
        ("rd A[tid * 4 * C + r * C + c - 1]", [False]),
        ("rd A[tid * 4 * C + r]; wr A[1000000 + tid * 4 * C + r * C + c]", [False, True]),
    ]
    for body, want in cases:
        got = _us_flags(head + body + tail, {"C": 64})
        assert got[: len(want)] == want, (body, got)


def test_literal_max_accepted():
    # 2^64 - 1 is a natural literal on both sides (R3)
    assert oracle.check("rd[18446744073709551615 - tid]", block=(2, 1, 1)).status == 0
    mc.MapProgram("rd[18446744073709551615 - tid]", block=(2, 1, 1))


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="needs a machine without a GPU")
def test_scratch_alloc_without_device_fails_loudly():
    """map_scratch_alloc (include/mapcheck.h): argument errors before device errors,
    MAP_E_CUDA without a device (the library still loads: the driver API is looked
    up at run time, libcuda is not linked); freeing NULL is a no-op, a foreign
    pointer is MAP_E_ARG."""
    import ctypes
    lib = mc._lib
    p, sz, comp = ctypes.c_void_p(), ctypes.c_uint64(), ctypes.c_uint32()
    assert lib.map_scratch_alloc(0, 1 << 20, 1, None, ctypes.byref(sz), ctypes.byref(comp)) == 8
    assert lib.map_scratch_alloc(0, 0, 1, ctypes.byref(p), None, None) == 8
    assert lib.map_scratch_alloc(0, 1 << 20, 6, ctypes.byref(p), None, None) == 8
    assert lib.map_scratch_alloc(0, 1 << 20, 1, ctypes.byref(p), ctypes.byref(sz), ctypes.byref(comp)) == 6
    assert p.value is None and sz.value == 0 and comp.value == 0
    assert lib.map_scratch_free(None) == 0
    assert lib.map_scratch_free(ctypes.c_void_p(0x1000)) == 8
    with pytest.raises(mc.MapError):
        mc.alloc_scratch(1 << 20, device=0)


def test_python_flag_constants_match_header():
    """The binding's flag values are the header's #defines (marshalling only)."""
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                            "mapcheck.h")).read()
    val = lambda name: int(re.search(r"#define " + name + r" (0x[0-9A-Fa-f]+|\d+)u", hdr).group(1), 0)
    assert mc.GEN_PATHS == {"auto": val("MAP_GEN_AUTO"), "vm": val("MAP_GEN_VM"), "jit": val("MAP_GEN_JIT")}
    for k in ("sort", "table", "direct", "unit", "auto"):
        assert mc.DETECT_PATHS[k] == val("MAP_DETECT_" + k.upper())
    assert mc.EXEC_SEQUENTIAL == val("MAP_EXEC_SEQUENTIAL")
    assert mc.EXEC_PROFILE_GENERATE == val("MAP_EXEC_PROFILE_GENERATE")
    assert mc.EXEC_PROFILE_SAMPLED == val("MAP_EXEC_PROFILE_SAMPLED")
    # map_kernel_stats mirrored field by field (ms, launches, bytes, timed)
    import ctypes
    assert [f for f, _ in mc._Stats._fields_] == ["ms", "launches", "bytes", "timed"]
    assert ctypes.sizeof(mc._Stats) == 10 * (4 + 4 + 8 + 4)


def test_known_low_bits_are_sound():
    """The compiler's known low bits of every access site (map_debug_dump "knownE=kb:kv",
    the basis of the stride-compressed direct table): every index the site produces,
    evaluated independently here, is congruent to kv modulo 2^kb -- on random strided
    MAPs (workloads.fuzz.random_strided_instance) and the Blelloch configs' closed forms."""
    from workloads import fuzz
    checked = 0
    for seed in range(40):
        inst = fuzz.random_strided_instance(seed)
        p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
        known = [[tuple(int(x) for x in m.split(":")) for m in re.findall(r"known\d+=(\d+:\d+)", line)]
                 for line in p.dump().splitlines() if line.startswith("instance")]
        phases = inst.src.split("params N; shared A, B;\n", 1)[1].split(";\nsync;\n")
        assert len(known) == len(phases), (seed, len(known), len(phases))
        nt, N = inst.block[0], inst.params["N"]
        for ph, sites in zip(phases, known):
            idx = re.findall(r"(?:rd|wr) [AB]\[([^\[\]]*)\]", ph)
            assert len(idx) == len(sites), (seed, ph)
            for text, (kb, kv) in zip(idx, sites):
                expr = text.replace("/", "//")
                mod = 1 << min(kb, 64)
                for tid in range(nt):
                    for k in range(N):
                        v = eval(expr, {"tid": tid, "k": k})
                        assert v % mod == kv % mod, (seed, text, kb, kv, tid, k, v)
                        checked += 1
    assert checked > 10000
    # Blelloch up-sweep phase l (1-based): (2^(l-1)) * (2m + 1) - 1 and (2^(l-1)) * (2m + 2) - 1
    inst = config("4c", n=1 << 10, bs=64)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    lines = [l for l in p.dump().splitlines() if l.startswith("instance")]
    for l in range(1, 8):
        kb = [tuple(int(x) for x in m.split(":")) for m in re.findall(r"known\d+=(\d+:\d+)", lines[l])]
        assert kb[0] == (l, (1 << (l - 1)) - 1) and kb[1] == (l, (1 << l) - 1), (l, kb)
