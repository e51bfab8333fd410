"""GPU parity of the row-jammed direct generate (jit.cpp paired_case, JU > 0): a
thread takes JU consecutive rows of one column quad and ORs a cell the next row
touches again into that row's quad before one global reduction.  Every MAP here
is shaped so that the jam applies (two nested loops, the inner range a multiple of
4 dividing or divisible by the 512-tuple tile); results are compared with the CPU
oracle, bit-exact, on the direct path, and with the jam disabled (MAPC_JAM=0, in a
subprocess: the flag is read once per process)."""
import json
import os
import subprocess
import sys

import pytest

import oracle
import paper_2203_12878_b200 as mc
from workloads import config

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, source, params, block): rows r (second-innermost) x columns c (innermost)
JAM_SRCS = [
    # stencil rows r-1, r, r+1 (periodic) read, row r written in the other half (5a-like, DRF)
    ("stencil_pingpong", """params R, C, H; shared A;
forU r in 0..R { forU c in 0..C {
  rd A[((tid * R + r + H - 1) % H) * C + c]; rd A[(tid * R + r) * C + c];
  rd A[((tid * R + r + 1) % H) * C + c]; wr A[H * C + (tid * R + r) * C + c] } }""", {}, 64),
    # in place (racy at the thread boundaries, 5b-like)
    ("stencil_inplace", """params R, C, H; shared A;
forU r in 0..R { forU c in 0..C {
  rd A[((tid * R + r + H - 1) % H) * C + c]; rd A[(tid * R + r) * C + c];
  rd A[((tid * R + r + 1) % H) * C + c]; wr A[(tid * R + r) * C + c] } }""", {}, 64),
    # rows walked backwards, the next row's cell is the previous row's neighbour
    ("reverse_rows", """params R, C, H; shared A;
forU r in 0..R { forU c in 0..C {
  rd A[(tid * R + (R - 1 - r)) * C + c]; rd A[(tid * R + (R - r)) * C + c];
  wr A[H * C + (tid * R + r) * C + c] } }""", {}, 32),
    # row stride 2: no two consecutive rows share a cell (nothing to absorb)
    ("stride2_rows", """params R, C, H; shared A;
forU r in 0..R { forU c in 0..C { rd A[(2 * (tid * R + r)) * C + c]; wr A[(2 * (tid * R + r) + 1) * C + c] } }""",
     {}, 32),
    # guarded sites: even rows read, odd rows write the same row as the next even one (racy between threads)
    ("guarded_rows", """params R, C, H; shared A;
forU r in 0..R { forU c in 0..C {
  if (r % 2 = 0) { rd A[(tid * R + r) * C + c] } else { wr A[((tid * R + r + 1) % H) * C + c] } } }""", {}, 16),
    # an unaligned column offset (quads straddle 4-cell groups) and a row shared by all threads
    ("unaligned_shared_row", """params R, C, H; shared A;
forU r in 0..R { forU c in 0..C { rd A[(tid * R + r) * C + c + 1]; rd A[r * C + c + 2] } };
sync;
forU r in 0..R { forU c in 0..C { if (tid = 3 and r = 1) { wr A[r * C + c + 2] } else { skip } } }""", {}, 8),
    # several arrays; the same row read twice per tuple and written once (same-cell merge + absorb)
    ("two_arrays", """params R, C, H; shared A, B;
forU r in 0..R { forU c in 0..C {
  rd A[(tid * R + r) * C + c]; rd A[(tid * R + r) * C + c]; rd B[(tid * R + r + 1) * C + c];
  wr B[(tid * R + r) * C + c] } }""", {}, 32),
]


def _got(r):
    return (r.verdict, r.witness.as_tuple() if r.witness else None, r.n_accesses, r.racy_segments)


def _want(o):
    assert o.status == 0, o.diag
    return (o.verdict, o.witness, o.n_accesses, o.n_racy_segments)


@pytest.mark.parametrize("C", [4, 16, 64, 512, 1024])
@pytest.mark.parametrize("R", [2, 4, 16])
@pytest.mark.parametrize("k", range(len(JAM_SRCS)))
def test_row_jam_matches_oracle(k, R, C):
    name, src, extra, nthreads = JAM_SRCS[k]
    # enough tuples per phase for whole super-tiles (jam_rows): threads * R * C >= 512 * U
    params = {"R": R, "C": C, "H": nthreads * R, **extra}
    grid, block = (2, 1, 1), (nthreads, 1, 1)
    o = _want(oracle.check(src, grid=grid, block=block, params=params))
    p = mc.MapProgram(src, grid, block, params)
    jammed = any("u_ <" in p.jit_source(c, 1) for c in range(p.n_chunks()))
    # whole super-tiles and something to merge (guarded_rows: rows r and r + 1 share a cell only from R = 3 on)
    if nthreads * R * C >= 512 * 2 and name not in ("unaligned_shared_row", "stride2_rows") and \
            not (name == "guarded_rows" and R < 4):
        assert jammed, (name, R, C)
    assert _got(p.check_races(detect="direct", gen="jit")) == o, (name, R, C, jammed)
    assert _got(p.check_races(detect="direct", gen="jit", overlap=False)) == o


def test_row_jam_full_size_5a_5b():
    """The headline configs take the jam (16 rows per thread) and keep their closed
    forms: 5a DRF, 5b 2 * blockDim * C racy cells per phase."""
    for name in ("5a", "5b"):
        inst = config(name)
        p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
        assert "u_ < 16u" in p.jit_source(0, 1)
        r = p.check_races()
        assert r.n_accesses == 1 << 34
        assert r.racy_segments == (0 if name == "5a" else 16 * 2 * 1024 * 1024)


_CHILD = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import paper_2203_12878_b200 as mc
from tests.test_gpu_jam import JAM_SRCS
out = []
for name, src, extra, nthreads in JAM_SRCS:
    for R, C in ((4, 64), (16, 1024)):
        params = {"R": R, "C": C, "H": nthreads * R, **extra}
        p = mc.MapProgram(src, (2, 1, 1), (nthreads, 1, 1), params)
        r = p.check_races(detect="direct", gen="jit")
        out.append([name, R, C, r.verdict, list(r.witness.as_tuple()) if r.witness else None, r.n_accesses,
                    r.racy_segments, "u_ <" in p.jit_source(0, 1)])
print(json.dumps(out))
"""


def test_row_jam_off_gives_same_results():
    res = {}
    for jam in ("0", "16"):
        env = dict(os.environ, MAPC_JAM=jam)
        cp = subprocess.run([sys.executable, "-c", _CHILD, ROOT], env=env, capture_output=True, text=True,
                            timeout=600, cwd=ROOT)
        assert cp.returncode == 0, cp.stderr[-2000:]
        res[jam] = json.loads(cp.stdout.strip().splitlines()[-1])
    assert not any(x[-1] for x in res["0"])
    assert any(x[-1] for x in res["16"])
    assert [x[:-1] for x in res["0"]] == [x[:-1] for x in res["16"]]


def test_row_jam_fuzz():
    """Random row x column MAPs (workloads.fuzz.random_rows_instance) on the direct
    path with the jammed JIT generate: equal to the oracle, bit-exact."""
    from workloads import fuzz
    bad, jammed = [], 0
    for seed in range(120):
        inst = fuzz.random_rows_instance(seed)
        o = oracle.check_instance(inst)
        if o.status != 0:
            continue
        p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
        jammed += any("u_ <" in p.jit_source(c, 1) for c in range(p.n_chunks()))
        if _got(p.check_races(detect="direct", gen="jit")) != _want(o):
            bad.append((seed, inst.src))
    assert not bad, bad[:3]
    assert jammed >= 40, jammed
