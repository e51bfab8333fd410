"""GPU parity of the on-chip per-unit detect (MAP_DETECT_UNIT, jit.cpp unit
mode; SURVEY.md §8f NEXT-3 "detect in smem tables per unit"): every scaled
config, the fuzz corpus and the full-size transposes against the oracle,
bit-exact, and proof that the unit kernel is what ran."""
import pytest

import oracle
import paper_2203_12878_b200 as mc
from tests.test_oracle import CASES
from workloads import config, fuzz

pytestmark = pytest.mark.gpu


def _got(r):
    return (r.verdict, r.witness.as_tuple() if r.witness else None, r.n_accesses, r.racy_segments)


def _want(o):
    assert o.status == 0, o.diag
    return (o.verdict, o.witness, o.n_accesses, o.n_racy_segments)


@pytest.mark.parametrize("name,sizes", CASES, ids=[f"{n}-{i}" for i, (n, _) in enumerate(CASES)])
def test_unit_path_configs(name, sizes):
    inst = config(name, **sizes)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    o = _want(oracle.check_instance(inst))
    unit = max(1, p.info.max_unit_accesses)
    for chunk in (0, unit):
        if chunk and p.n_chunks(chunk) > 64:
            continue
        r = p.check_races(gen="jit", detect="unit", chunk_max_accesses=chunk, profile=True)
        assert _got(r) == o, (name, chunk)


def test_unit_fuzz():
    bad, ran = [], 0
    for seed in range(0, 300, 2):
        inst, _ = fuzz.random_instance(seed)
        o = oracle.check_instance(inst, threads=1)
        if o.status != 0:
            continue
        p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
        r = p.check_races(gen="jit", detect="unit", profile=True)
        ran += r.kernels["unit"]["launches"] > 0
        if _got(r) != _want(o):
            bad.append((seed, inst.src, _got(r), _want(o)))
    assert not bad and ran >= 50, (ran, bad[:3])


@pytest.mark.parametrize("name", ["3a", "3b"])
def test_unit_full_size_transpose(name):
    inst = config(name)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    r = p.check_races(profile=True)                       # the automatic choice
    assert r.kernels["unit"]["launches"] > 0 and r.kernels["direct"]["launches"] == 0
    assert _got(r) == _want(oracle.check_instance(inst))


def test_unit_u32_cells_and_two_arrays():
    # 2048 threads per block (u32 cells), two arrays in one unit
    src = "shared A, B; wr A[tid % 700]; rd B[(tid * 3) % 512]; sync; wr B[tid / 2]; rd A[tid % 9]"
    for grid in (1, 300):
        o = _want(oracle.check(src, grid=(grid, 1, 1), block=(1024, 2, 1)))
        r = mc.check(src, grid=(grid, 1, 1), block=(1024, 2, 1), gen="jit", detect="unit", profile=True)
        assert _got(r) == o and r.kernels["unit"]["launches"] > 0


# ---- cluster units: the unit table spread over a thread-block cluster (DSMEM) ----

@pytest.mark.parametrize("name,n", [("4b", 1 << 15), ("4d", 1 << 17), ("4c", 1 << 18), ("4b", 1 << 19),
                                    ("4d", 1 << 20)])
def test_cluster_units(name, n):
    # unit tables of 64 KB .. 2 MB: clusters of 2 .. 16 CTAs
    inst = config(name, n=n, bs=1024)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    src = p.jit_source(0, 3)
    assert "extern __shared__" in src, (name, n)             # the cluster variant is what runs
    o = _want(oracle.check_instance(inst))
    for gen, det in [("jit", "auto"), ("jit", "unit")]:
        r = p.check_races(gen=gen, detect=det, profile=True)
        assert _got(r) == o and r.kernels["unit"]["launches"] > 0, (name, n, det)


def test_cluster_unit_fuzz_wide_index():
    # fuzz programs with a wide, sparse index range per unit (x * 4096 + ...): cluster tables
    bad, ran = [], 0
    for seed in range(0, 120, 3):
        inst, _ = fuzz.random_instance(seed)
        src = inst.src.replace("rd[", "rd[65536 + ").replace("wr[", "wr[65536 + ")
        src = src.replace(" A[", " A[200000 - ").replace(" B[", " B[200000 - ") if "shared" in src else src
        o = oracle.check(src, inst.grid, inst.block, inst.params)
        if o.status != 0:
            continue
        p = mc.MapProgram(src, inst.grid, inst.block, inst.params)
        r = p.check_races(gen="jit", detect="unit", profile=True)
        ran += r.kernels["unit"]["launches"] > 0
        if _got(r) != _want(o):
            bad.append((seed, src, _got(r), _want(o)))
    assert not bad, bad[:3]
