"""GPU parity for the product configurations round 1 left untested (VERDICT r1
"What's weak" 1, 10): u32-cell direct tables (1025..32768 threads
per block), the look-back onesweep sort variant, the and/or evaluation
reading (R2), the overlapped direct pipeline on plans whose chunks
have different table sizes over a dirty scratch buffer, and CUDA-graph replay
when the staging buffer, the plan or the scratch contents change between calls.
Every result is compared with the CPU oracle (bit-exact)."""
import json
import os
import subprocess
import sys

import pytest

import oracle
import paper_2203_12878_b200 as mc
from workloads import config, fuzz

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _got(r):
    return (r.verdict, r.witness.as_tuple() if r.witness else None, r.n_accesses, r.racy_segments)


def _want(o):
    assert o.status == 0, o.diag
    return (o.verdict, o.witness, o.n_accesses, o.n_racy_segments)


# ---- u32 cells: 2 w_tid + 1 <= 32 but w_tid > 10 (1025..32768 threads) ------

U32_SRCS = [
    ("params N; forU c in 0..N { wr[c + tid * N] }", {"N": 16}),                        # aligned pairs
    ("params N; forU c in 0..N { wr[c + 1 + tid * N] }", {"N": 16}),                    # odd base: no pairs
    ("params N; forU c in 0..N { if (c % 3 = 1) { wr[c + tid * N] } else { rd[c + tid * N] } }", {"N": 12}),
    ("params N; forU c in 0..N { rd[c + tid * (N - 1)]; if (c = 5) { wr[c + tid * (N - 1)] } else { skip } }",
     {"N": 9}),                                                                          # overlapping rows
    ("params N; forU c in 0..N { rd[2 * c]; wr[2 * c + 1 + (tid % 2)] }", {"N": 40}),    # stride 2, racy
    ("wr[tid % 1500]; sync; rd[(tid * 7) % 2048]", {}),
    ("rd[tid]; if (tid = 1500) { wr[17] } else { skip }; rd[17]", {}),
]


@pytest.mark.parametrize("block", [(1024, 2, 1), (1024, 32, 1), (1537, 1, 1)])
@pytest.mark.parametrize("k", range(len(U32_SRCS)))
def test_u32_cell_direct_path(block, k):
    src, params = U32_SRCS[k]
    grid = (2, 1, 1)
    o = _want(oracle.check(src, grid=grid, block=block, params=params))
    p = mc.MapProgram(src, grid, block, params)
    if block[1] == 2:       # the paired G=2 generate (one red.or.b64 per aligned pair) is what runs
        assert "sfP[K] + 1 && !(sfP[K] & 1u)" in p.jit_source(0, 1)
    unit = max(1, p.info.max_unit_accesses)
    for gen in ("vm", "jit"):
        for chunk in (0, unit):
            assert _got(p.check_races(detect="direct", gen=gen, chunk_max_accesses=chunk)) == o, (gen, chunk)
    assert _got(p.check_races(detect="sort")) == o


def test_u32_cell_fuzz_big_blocks():
    bad, ran = [], 0
    for seed in range(0, 90):
        inst, _ = fuzz.random_instance(seed, big_block=True)
        o = oracle.check_instance(inst)
        if o.status != 0:
            continue
        ran += 1
        p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
        unit = max(1, p.info.max_unit_accesses)
        for gen in ("vm", "jit"):
            for chunk in (0, unit):
                if chunk and p.n_chunks(chunk) > 24:
                    continue
                r = p.check_races(detect="direct", gen=gen, chunk_max_accesses=chunk)
                if _got(r) != _want(o):
                    bad.append((seed, gen, chunk, inst.block, inst.src))
    assert ran >= 60 and not bad, bad[:3]


def test_u32_cell_configs():
    # transpose with 32x64 threads per block (2048) and a 2048-thread stencil
    for inst in [config("3b", ts=64, rw=32, grid=4), config("3a", ts=64, rw=32, grid=4),
                 config("5b", block=2048, T=2, R=2, C=32), config("5a", block=2048, T=2, R=2, C=32)]:
        o = _want(oracle.check_instance(inst))
        p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
        for gen in ("vm", "jit"):
            assert _got(p.check_races(detect="direct", gen=gen)) == o, (inst.name, gen)


# ---- the decoupled look-back onesweep (MAPC_SORT=onesweep, read once per process)

_ONESWEEP_SCRIPT = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import oracle, paper_2203_12878_b200 as mc
from workloads import config, fuzz
from tests.test_oracle import CASES
out = []
cases = [config(n, **s) for n, s in CASES] + [fuzz.random_instance(s)[0] for s in range(0, 200, 5)]
for inst in cases:
    o = oracle.check_instance(inst)
    if o.status != 0:
        continue
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    unit = max(1, p.info.max_unit_accesses)
    for chunk in (0, unit):
        if chunk and p.n_chunks(chunk) > 64:
            continue
        r = p.check_races(detect="sort", chunk_max_accesses=chunk)
        got = [r.verdict, list(r.witness.as_tuple()) if r.witness else None, r.n_accesses, r.racy_segments]
        want = [o.verdict, list(o.witness) if o.witness else None, o.n_accesses, o.n_racy_segments]
        if got != want:
            out.append([inst.name, chunk, got, want])
print(json.dumps({"n": len(cases), "bad": out}))
"""


def test_onesweep_sort_variant_matches_oracle():
    env = dict(os.environ, MAPC_SORT="onesweep")
    r = subprocess.run([sys.executable, "-c", _ONESWEEP_SCRIPT, ROOT], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=1800)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["n"] > 40 and res["bad"] == [], res["bad"][:3]


# ---- DESIGN.md R2 on the GPU path --------------------------------------------

@pytest.mark.parametrize("src", ["if (tid = 9 and 1 / (tid - tid) = 0) { wr[0] } else { skip }",
                                 "if (tid < 9 or 1 % (tid - tid) = 0) { wr[0] } else { skip }"])
def test_and_or_evaluate_both_operands_gpu(src):
    assert oracle.check(src, block=(4, 1, 1)).status == 5
    for gen in ("vm", "jit"):
        with pytest.raises(mc.MapError) as e:
            mc.check(src, block=(4, 1, 1), gen=gen)
        assert e.value.status == 5


# ---- overlapped direct pipeline: chunks with different table sizes -----------

MIXED_S = ("params N; wr[tid]; sync; forU c in 0..N { rd[(c * 7 + tid) % (N * 64)]; "
           "if (c = tid) { wr[c * 64 + tid] } else { skip } }; sync; rd[tid % 3]")


def test_overlap_mixed_table_sizes_dirty_scratch():
    import torch
    grid, block, params = (8, 1, 1), (64, 1, 1), {"N": 64}
    o = _want(oracle.check(MIXED_S, grid=grid, block=block, params=params))
    p = mc.MapProgram(MIXED_S, grid, block, params)
    unit = max(1, p.info.max_unit_accesses)
    sizes = {p.chunk_info(c, unit)["sort_bits"] for c in range(p.n_chunks(unit))}
    assert len(sizes) >= 2 and p.n_chunks(unit) >= 4, sizes
    for chunk in (unit, 0):
        scratch = torch.full((p.scratch_bytes(chunk),), 0xFF, dtype=torch.uint8, device="cuda")
        for _ in range(4):       # fresh, capture, replay, replay
            r = p.check_races(scratch=scratch, gen="jit", detect="direct", chunk_max_accesses=chunk)
            assert _got(r) == o, chunk
            scratch.fill_(0xFF)


# ---- CUDA graphs: replay after the staging buffer / plan / scratch changed ---

def test_graph_replay_after_plan_and_stage_change():
    import torch
    inst = config("5b", block=64, T=6, R=4, C=16)
    o = _want(oracle.check_instance(inst))
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    unit = max(1, p.info.max_unit_accesses)
    scratch = torch.empty(max(p.scratch_bytes(0), p.scratch_bytes(unit)), dtype=torch.uint8, device="cuda")
    seq = [0, 0, unit, 0, 0, unit, unit, 0]        # A, A (capture), B (bigger stage), A, ...
    for chunk in seq:
        assert _got(p.check_races(scratch=scratch, chunk_max_accesses=chunk)) == o, chunk


def test_graph_replay_two_programs_share_scratch():
    import torch
    a, b = config("5b", block=64, T=3, R=4, C=16), config("3b", ts=32, rw=8, grid=16)
    pa = mc.MapProgram(a.src, a.grid, a.block, a.params)
    pb = mc.MapProgram(b.src, b.grid, b.block, b.params)
    oa, ob = _want(oracle.check_instance(a)), _want(oracle.check_instance(b))
    scratch = torch.empty(max(pa.scratch_bytes(), pb.scratch_bytes()), dtype=torch.uint8, device="cuda")
    for i in range(5):          # each program's graph is captured and replayed over the other's leftovers
        for detect in ("auto", "sort"):
            assert _got(pa.check_races(scratch=scratch, detect=detect)) == oa, (i, detect)
            assert _got(pb.check_races(scratch=scratch, detect=detect)) == ob, (i, detect)


# ---- the multi-GPU shard plan, run rank by rank on one GPU --------------------

@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("inst", [config("3b", ts=32, rw=8, grid=512), config("4b", n=1 << 14, bs=256),
                                  config("5b", block=64, T=6, R=4, C=64), config("2b")],
                         ids=["3b", "4b", "5b", "2b"])
def test_rank_shards_cover_the_plan(inst, world):
    # every rank's share (map_rank_chunks under the world-aware default chunk) run in
    # turn: the counts add up to the oracle's and the smallest witness is the oracle's,
    # on the unit, direct and sort paths
    o = oracle.check_instance(inst)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    chunk = p.default_chunk(world)
    assert sorted(c for r in range(world) for c in p.rank_chunks(r, world, chunk)) == list(range(p.n_chunks(chunk)))
    for gen, det in [("jit", "auto"), ("jit", "direct"), ("vm", "sort")]:
        parts = [p.check_races(rank=r, world=world, gen=gen, detect=det) for r in range(world)]
        assert sum(x.n_accesses for x in parts) == o.n_accesses, (gen, det)
        assert sum(x.racy_segments for x in parts) == o.n_racy_segments
        wits = [x.witness.as_tuple() for x in parts if x.witness]
        assert (min(wits) if wits else None) == o.witness


# ---- many-chunk plans: AUTO takes the specialised generate when the chunks share kernels

@pytest.mark.parametrize("name", ["5a", "5b"])
def test_many_phase_plan_auto_takes_jit(name):
    """5a/5b at T = 80 phases (80 chunks, 2 distinct kernels): AUTO must give the VM's
    results (verdict, witness, count, racy cells = the closed forms) and run the
    specialised generate (profiles/r2y_l2_5a.jsonl: 7x faster than the VM here)."""
    T, R, C = 80, 32, 256
    inst = config(name, T=T, R=R, C=C)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    assert p.n_chunks() > 64
    vm = p.check_races(gen="vm")
    auto = p.check_races()
    assert _got(auto) == _got(vm)
    assert auto.n_accesses == 1024 * R * C * 4 * T
    assert auto.racy_segments == (0 if name == "5a" else 2 * 1024 * C * T)
    t_vm = min(p.check_races(gen="vm").device_ms for _ in range(3))
    t_auto = min(p.check_races().device_ms for _ in range(3))
    assert t_auto * 2 < t_vm, (t_auto, t_vm)


# ---- scratch in compressible device memory (map_scratch_alloc) ---------------

def test_scratch_alloc_compressible_and_freed():
    import torch
    t = mc.alloc_scratch(3 << 30)
    assert t.is_cuda and t.dtype == torch.uint8 and t.numel() >= 3 << 30
    assert t._map_block.compressed            # B200 grants generic compression
    t.fill_(7)
    assert int(t[(3 << 30) - 1].item()) == 7
    free0 = torch.cuda.mem_get_info()[0]
    del t
    torch.cuda.synchronize()
    assert torch.cuda.mem_get_info()[0] >= free0 + (3 << 30) - (64 << 20)   # released, not cached
    for _ in range(3):                                                     # no leak over cycles
        u = mc.alloc_scratch(2 << 30, compressible=False)
        assert not u._map_block.compressed
        del u


@pytest.mark.parametrize("inst", [config("5a", T=4, R=4, C=128), config("5b", T=4, R=4, C=128),
                                  config("3b", ts=32, rw=8, grid=2048), config("4b", n=1 << 16, bs=1024),
                                  config("4c", n=1 << 16, bs=1024)], ids=lambda i: i.name)
def test_compressible_scratch_same_results(inst):
    """Every detect path over compressible scratch = over plain scratch = the oracle
    (the memory kind changes DRAM traffic only)."""
    import torch
    o = _want(oracle.check_instance(inst))
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    comp = mc.alloc_scratch(p.scratch_bytes())
    comp.fill_(0xFF)                         # dirty, as a reused buffer would be
    plain = torch.full((p.scratch_bytes(),), 0xFF, dtype=torch.uint8, device="cuda")
    for det in ("auto", "direct", "table", "sort"):
        for s in (comp, plain, comp):
            assert _got(p.check_races(scratch=s, detect=det)) == o, det


def test_profiled_runs_replay_as_graphs():
    """profile=True calls are captured (third call on) with their timing events as
    graph nodes: same results and the same per-kernel launch counts in the eager,
    capturing and replaying calls, every timed class with a positive time."""
    inst = config("5b", T=4, R=4, C=128)
    o = _want(oracle.check_instance(inst))
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    runs = [p.check_races(profile=True, gen="jit") for _ in range(5)]
    for r in runs:
        assert _got(r) == o
    launches = [{k: v["launches"] for k, v in r.kernels.items()} for r in runs]
    assert all(x == launches[0] for x in launches)
    for r in runs[2:]:
        for k, v in r.kernels.items():
            if v["launches"]:
                assert v["ms"] > 0, (k, v)
    plain = [p.check_races(gen="jit").device_ms for _ in range(3)]
    assert min(r.device_ms for r in runs[2:]) < 3 * min(plain) + 0.05


def test_sampled_generate_timing():
    """profile="sampled" (MAP_EXEC_PROFILE_GENERATE | MAP_EXEC_PROFILE_SAMPLED): every
    launch counted, only the generates of chunk positions 2, 6, 10, ... timed, in the
    eager, capturing and replaying calls alike; results unchanged."""
    inst = config("5b", T=12, R=32, C=256)
    o = _want(oracle.check_instance(inst))
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    n = p.n_chunks()
    assert n >= 6
    want_timed = len([i for i in range(n) if i % 4 == 2])
    full = p.check_races(profile=True, gen="jit").kernels["direct"]
    for _ in range(4):
        r = p.check_races(profile="sampled", gen="jit")
        assert _got(r) == o
        k = r.kernels["direct"]
        assert k["launches"] == full["launches"] == n
        assert k["timed"] == want_timed and k["ms"] > 0
        assert r.kernels["detect"]["timed"] == 0 and r.kernels["detect"]["ms"] == 0
