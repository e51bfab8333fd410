"""GPU parity of the stride-compressed direct table (mapcheck.cpp Chunk::pcomp,
jit.cpp `comp`): when every site of a phase has the same residue modulo 2^k (the
compiler's known low bits), the phase's block of the direct table keeps one cell per
2^k indices.  Every MAP here is strided so the compression applies (checked in the
specialised source); results are compared with the CPU oracle, bit-exact, on the
direct path with the specialised generate, overlapped and sequential."""
import pytest

import oracle
import paper_2203_12878_b200 as mc
from workloads import config

pytestmark = pytest.mark.gpu


def _got(r):
    return (r.verdict, r.witness.as_tuple() if r.witness else None, r.n_accesses, r.racy_segments)


def _want(o):
    assert o.status == 0, o.diag
    return (o.verdict, o.witness, o.n_accesses, o.n_racy_segments)


# (name, source, grid, block, params): strided indices, several phases, arrays, blocks
STRIDED = [
    ("odd_cells", "params N; forU k in 0..N { rd A[4 * (k * 64 + tid) + 1]; wr A[4 * (k * 64 + tid) + 1] }",
     (1, 1, 1), (64, 1, 1), {"N": 64}),
    ("odd_cells_racy", "params N; forU k in 0..N { rd A[4 * (k * 64 + tid) + 1]; wr A[4 * (k * 64 + (tid / 2)) + 1] }",
     (1, 1, 1), (64, 1, 1), {"N": 64}),
    ("per_phase_stride", """params N; forS l in 0..5 {
  forU k in 0..N { if (k < N >> l) { rd A[(1 << l) * (2 * (k * 32 + tid) + 1) - 1];
                                      wr A[(1 << l) * (2 * (k * 32 + tid) + 2) - 1] } else { skip } };
  sync }""", (1, 1, 1), (32, 1, 1), {"N": 64}),
    ("two_arrays_blocks", """params N; shared A, B;
forU k in 0..N { rd A[8 * (k * 16 + tid) + 3]; wr B[8 * (k * 16 + tid) + 5]; rd B[8 * (k * 16 + ((tid + 1) % 16)) + 5] }""",
     (4, 1, 1), (16, 1, 1), {"N": 64}),
    ("mixed_residue", "params N; forU k in 0..N { rd A[8 * (k * 32 + tid) + 2]; wr A[8 * (k * 32 + tid) + 6] }",
     (2, 1, 1), (32, 1, 1), {"N": 128}),
]


@pytest.mark.parametrize("k", range(len(STRIDED)))
def test_compressed_table_matches_oracle(k):
    name, src, grid, block, params = STRIDED[k]
    o = _want(oracle.check(src, grid=grid, block=block, params=params))
    p = mc.MapProgram(src, grid, block, params)
    assert any("cbase_" in p.jit_source(c, 1) for c in range(p.n_chunks())), name
    for ovl in (True, False):
        assert _got(p.check_races(detect="direct", gen="jit", overlap=ovl)) == o, (name, ovl)
    assert _got(p.check_races(detect="direct", gen="vm")) == o        # the VM keeps the full table
    assert _got(p.check_races(detect="sort")) == o


@pytest.mark.parametrize("name", ["4a", "4b", "4c", "4d"])
@pytest.mark.parametrize("n", [1 << 12, 1 << 16])
def test_blelloch_scaled_compressed(name, n):
    inst = config(name, n=n, bs=256)
    o = _want(oracle.check_instance(inst))
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    for chunk in (0, max(1, p.info.max_unit_accesses)):
        if chunk and p.n_chunks(chunk) > 48:
            continue
        r = p.check_races(detect="direct", gen="jit", chunk_max_accesses=chunk)
        assert _got(r) == o, (name, n, chunk)


def test_compressed_table_fuzz():
    from workloads import fuzz
    bad, comp = [], 0
    for seed in range(150):
        inst = fuzz.random_strided_instance(seed)
        o = oracle.check_instance(inst)
        if o.status != 0:
            continue
        p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
        comp += any("cbase_" in p.jit_source(c, 1) for c in range(p.n_chunks()))
        for ovl in (True, False):
            if _got(p.check_races(detect="direct", gen="jit", overlap=ovl)) != _want(o):
                bad.append((seed, ovl, inst.src))
    assert not bad, bad[:3]
    assert comp >= 60, comp
