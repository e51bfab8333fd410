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


# ---- cluster units (opt-in, MAPC_CLUSTER=1, read once per process: a subprocess) ----

_CLUSTER_SCRIPT = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import oracle, paper_2203_12878_b200 as mc
from workloads import config
out = []
# unit tables of 128 KB .. 2 MB: clusters of 2 .. 16 CTAs (4b/4c/4d, one block, a phase per unit)
for name, n in [("4b", 1 << 16), ("4d", 1 << 17), ("4c", 1 << 18), ("4b", 1 << 19), ("4d", 1 << 20), ("4c", 1 << 20)]:
    inst = config(name, n=n, bs=1024)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    clustered = "extern __shared__" in p.jit_source(0, 3)
    o = oracle.check_instance(inst)
    for det in ("auto", "unit"):
        r = p.check_races(gen="jit", detect=det, profile=True)
        got = [r.verdict, list(r.witness.as_tuple()) if r.witness else None, r.n_accesses, r.racy_segments]
        want = [o.verdict, list(o.witness) if o.witness else None, o.n_accesses, o.n_racy_segments]
        out.append([name, n, det, clustered, r.kernels["unit"]["launches"] > 0, got == want])
print(json.dumps(out))
"""


def test_cluster_units_opt_in():
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MAPC_CLUSTER="1")
    r = subprocess.run([sys.executable, "-c", _CLUSTER_SCRIPT, root], cwd=root, env=env, capture_output=True,
                       text=True, timeout=1800)
    assert r.returncode == 0, r.stderr[-3000:]
    rows = json.loads(r.stdout.strip().splitlines()[-1])
    assert all(row[3] for row in rows), rows                   # every case ran as a cluster unit
    assert all(row[4] and row[5] for row in rows), rows        # on the unit kernel, = oracle
