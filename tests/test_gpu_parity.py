"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Bit-exact agreement on verdict, canonical witness, access count (multiset) and
racy-segment count -- integer work, so the bar is equality.
"""
import os

import pytest

import oracle
import paper_2203_12878_b200 as mc
from tests.test_oracle import CASES, n_closed, racy_closed, witness_closed
from workloads import config, fuzz

pytestmark = pytest.mark.gpu


def gpu(inst, chunk=0):
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    return p.check_races(chunk_max_accesses=chunk)


def same(r, o):
    assert o.status == 0, o.diag
    got = (r.verdict, r.witness.as_tuple() if r.witness else None, r.n_accesses, r.racy_segments)
    want = (o.verdict, o.witness, o.n_accesses, o.n_racy_segments)
    assert got == want


@pytest.mark.parametrize("name,sizes", CASES, ids=[f"{n}-{i}" for i, (n, _) in enumerate(CASES)])
def test_configs_scaled(name, sizes):
    inst = config(name, **sizes)
    same(gpu(inst), oracle.check_instance(inst))


@pytest.mark.parametrize("name,sizes", CASES, ids=[f"{n}-{i}" for i, (n, _) in enumerate(CASES)])
def test_configs_scaled_small_chunks(name, sizes):
    # force many chunks (phase ranges and block ranges) -> identical result
    inst = config(name, **sizes)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    unit = max(1, p.info.max_unit_accesses)
    same(p.check_races(chunk_max_accesses=unit), oracle.check_instance(inst))


@pytest.mark.parametrize("name,sizes", CASES[::2], ids=[f"{n}-{i}" for i, (n, _) in enumerate(CASES[::2])])
def test_generate_paths_agree(name, sizes):
    # the NVRTC-specialised generate and the bytecode VM give the same result
    inst = config(name, **sizes)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    o = oracle.check_instance(inst)
    for gen in ("vm", "jit"):
        same(p.check_races(gen=gen), o)


def test_fuzz_corpus_jit():
    bad = []
    for seed in range(0, 120, 3):
        inst, _ = fuzz.random_instance(seed)
        o = oracle.check_instance(inst, threads=1)
        r = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params).check_races(gen="jit")
        got = (r.verdict, r.witness.as_tuple() if r.witness else None, r.n_accesses, r.racy_segments)
        if got != (o.verdict, o.witness, o.n_accesses, o.n_racy_segments):
            bad.append((seed, inst.src))
    assert not bad, bad[:3]


def test_fuzz_corpus():
    n = int(os.environ.get("MAPCHECK_GPU_FUZZ", "400"))
    bad = []
    for seed in range(n):
        inst, _ = fuzz.random_instance(seed)
        o = oracle.check_instance(inst, threads=1)
        r = gpu(inst)
        got = (r.verdict, r.witness.as_tuple() if r.witness else None, r.n_accesses, r.racy_segments)
        want = (o.verdict, o.witness, o.n_accesses, o.n_racy_segments)
        if got != want:
            bad.append((seed, inst.src, got, want))
    assert not bad, bad[:3]


@pytest.mark.parametrize("name", ["1a", "1b", "2a", "2b", "2c", "4c", "4d"])
def test_full_size_vs_oracle(name):
    inst = config(name)
    same(gpu(inst), oracle.check_instance(inst))


@pytest.mark.parametrize("name", ["3a", "3b", "4a", "4b"])
def test_full_size_large_vs_oracle(name):
    inst = config(name)
    same(gpu(inst), oracle.check_instance(inst))


@pytest.mark.parametrize("name", ["5a", "5b"])
def test_full_size_stencil_properties(name):
    # 2^34 accesses: the oracle cannot enumerate them in test time; the access
    # count and the witness have closed forms (tests/test_oracle.py, pinned
    # there against the oracle and the brute force at smaller sizes).
    inst = config(name)
    r = gpu(inst)
    assert r.n_accesses == n_closed(name, inst) == 2**34
    w = witness_closed(name, inst)
    assert (r.witness.as_tuple() if r.witness else None) == w
    # exact racy-cell count: 0 for 5a, T*B*C*min(R, 2) = 2^25 for 5b (closed form
    # pinned against the brute force and the oracle in tests/test_oracle.py)
    assert r.racy_segments == racy_closed(name, inst) == (0 if name == "5a" else 2**25)


def test_long_segment_spans_many_tiles():
    # one (phase, index) cell read by all 1024 threads 1024 times + one write
    src = "forU x in 0..1024 { rd[0] }; wr[0]"
    for blk in (1024, 1):
        inst = config("1b", block=blk)
        inst.src = src
        same(gpu(inst), oracle.check_instance(inst))
    src2 = "forU x in 0..4096 { rd[0] }; if (tid = 1023) { wr[0] } else { skip }"
    r = mc.check(src2, block=(1024, 1, 1))
    o = oracle.check(src2, block=(1024, 1, 1))
    same(r, o)


def test_single_segment_s0():
    # S = 0 sort bits: every access in one segment (no sort at all)
    for src, blk in [("wr[0]", 8), ("rd[0]", 8), ("if (tid = 3) { wr[0] } else { rd[0] }", 8), ("wr[0]", 1)]:
        same(mc.check(src, block=(blk, 1, 1)), oracle.check(src, block=(blk, 1, 1)))


def test_empty_programs():
    for src in ["skip", "params M; forU x in 0..M { rd[x] }", "if (false) { wr[0] } else { skip }", "sync; sync"]:
        r = mc.check(src, block=(4, 1, 1), params={"M": 0} if "M" in src else None)
        assert r.verdict == 0 and r.n_accesses == 0


def test_runtime_div_by_zero():
    with pytest.raises(mc.MapError) as e:
        mc.check("rd[8 / (tid - 1)]", block=(4, 1, 1))
    assert e.value.status == 5
    assert oracle.check("rd[8 / (tid - 1)]", block=(4, 1, 1)).status == 5
    # guarded: never reached -> no error, same as the oracle
    src = "if (tid > 1) { rd[8 / (tid - 1)] } else { skip }"
    same(mc.check(src, block=(4, 1, 1)), oracle.check(src, block=(4, 1, 1)))


def test_determinism_across_runs_and_chunkings():
    inst = config("4b", n=1 << 14, bs=256)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    ref = p.check_races()
    for chunk in (0, p.info.max_unit_accesses, 3 * p.info.max_unit_accesses):
        for _ in range(3):
            r = p.check_races(chunk_max_accesses=chunk)
            assert (r.verdict, r.witness, r.n_accesses, r.racy_segments) == \
                   (ref.verdict, ref.witness, ref.n_accesses, ref.racy_segments)


def test_multi_dim_grid_and_block():
    src = "params W; wr[(tid / W) * W + (tid + 1) % W]; sync; rd[bid % 3]"
    for g, b in [((2, 3, 1), (4, 2, 1)), ((1, 1, 2), (2, 2, 2))]:
        same(mc.check(src, grid=g, block=b, params={"W": 4}), oracle.check(src, g, b, {"W": 4}))


def _fake_exchange(p, world, chunk_max=0):
    """Key-exchange mode with `world` logical ranks run one after another on
    one GPU: each rank generates + buckets its tuple slice, the buckets for
    each destination are concatenated (what all_to_all_single delivers), and
    each destination sorts + detects.  Returns (verdict, witness, n, racy)."""
    import torch
    dev = torch.device("cuda", 0)
    scratch = torch.empty(p.scratch_bytes(chunk_max), dtype=torch.uint8, device=dev)
    best, n_total, racy_total = None, 0, 0
    for c in range(p.n_chunks(chunk_max)):
        bound = max(1, p.chunk_info(c, chunk_max)["bound"])
        parts = [[] for _ in range(world)]
        for r in range(world):
            out = torch.empty(bound, dtype=torch.int64, device=dev)
            counts = p.generate_bucketed(c, r, world, out, scratch, chunk_max_accesses=chunk_max)
            assert sum(counts) <= bound
            off = 0
            for d, k in enumerate(counts):
                parts[d].append(out[off:off + k].clone())
                off += k
        for d in range(world):
            keys = torch.cat(parts[d]) if parts[d] else torch.empty(0, dtype=torch.int64, device=dev)
            n = keys.numel()
            packed, racy = p.sort_detect(c, keys if n else torch.empty(1, dtype=torch.int64, device=dev), n,
                                         scratch, chunk_max_accesses=chunk_max)
            n_total += n
            racy_total += racy
            if packed is not None:
                w = p.unpack_witness(c, packed).as_tuple()
                best = w if best is None or w < best else best
    return (1 if best else 0), best, n_total, racy_total


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("name", ["1a", "2b", "3b", "4b", "5b"])
def test_exchange_mode_matches_oracle(name, world):
    sizes = dict(CASES)[name] if name in dict(CASES) else {}
    inst = config(name, **sizes)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    o = oracle.check_instance(inst)
    assert o.status == 0
    assert _fake_exchange(p, world) == (o.verdict, o.witness, o.n_accesses, o.n_racy_segments)


def test_exchange_mode_many_chunks():
    inst = config("4b", n=1 << 14, bs=256)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    o = oracle.check_instance(inst)
    unit = max(1, p.info.max_unit_accesses)
    assert _fake_exchange(p, 3, unit) == (o.verdict, o.witness, o.n_accesses, o.n_racy_segments)


# ---- detect paths: full sort + segmented scan vs partial sort + bucket tables ----

@pytest.mark.parametrize("detect", ["sort", "table", "direct"])
@pytest.mark.parametrize("name,sizes", CASES, ids=[f"{n}-{i}" for i, (n, _) in enumerate(CASES)])
def test_detect_paths_match_oracle(name, sizes, detect):
    inst = config(name, **sizes)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    o = oracle.check_instance(inst)
    same(p.check_races(detect=detect), o)
    unit = max(1, p.info.max_unit_accesses)
    same(p.check_races(chunk_max_accesses=unit, detect=detect), o)


def test_fuzz_corpus_table_detect():
    bad = []
    for seed in range(0, 400, 2):
        inst, _ = fuzz.random_instance(seed)
        o = oracle.check_instance(inst, threads=1)
        r = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params).check_races(detect="table")
        got = (r.verdict, r.witness.as_tuple() if r.witness else None, r.n_accesses, r.racy_segments)
        if got != (o.verdict, o.witness, o.n_accesses, o.n_racy_segments):
            bad.append((seed, inst.src, got))
    assert not bad, bad[:3]


@pytest.mark.parametrize("detect", ["sort", "table", "direct"])
def test_one_bucket_across_all_ranges(detect):
    # few distinct cells, millions of keys: with the table path every range of the
    # detect kernel sees the same bucket, so the partial tables chain end to end
    for src in ["params N; forU x in 0..N { rd[x % 8] }; wr[tid % 4]",
                "params N; forU x in 0..N { rd[x % 8] }; if (tid = 5) { wr[3] } else { skip }",
                "params N; forU x in 0..N { rd[x % 8]; wr[8 + tid] }"]:
        r = mc.check(src, block=(1024, 1, 1), params={"N": 4096}, detect=detect)
        o = oracle.check(src, block=(1024, 1, 1), params={"N": 4096})
        same(r, o)


@pytest.mark.parametrize("name", ["3b", "4b", "5b"])
def test_full_size_detect_paths_agree(name):
    sizes = {"5b": {"T": 2}}.get(name, {})
    inst = config(name, **sizes)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    a = p.check_races(detect="sort")
    b = p.check_races(detect="table")
    c = p.check_races(detect="direct")
    assert (a.verdict, a.witness, a.n_accesses, a.racy_segments) == (b.verdict, b.witness, b.n_accesses, b.racy_segments)
    assert (a.verdict, a.witness, a.n_accesses, a.racy_segments) == (c.verdict, c.witness, c.n_accesses, c.racy_segments)


@pytest.mark.parametrize("detect", ["sort", "table", "direct"])
@pytest.mark.parametrize("name,sizes", [("5a", dict(T=3, R=8, C=64)), ("5b", dict(T=2, R=4, C=96)),
                                        ("5b", dict(T=1, R=3, C=40)), ("1a", dict(M=4096))])
def test_jit_single_segment_chunks(name, sizes, detect):
    # one phase per chunk, JIT generate: a single all-dense segment per chunk
    inst = config(name, **sizes)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    o = oracle.check_instance(inst)
    unit = max(1, p.info.max_unit_accesses)
    for chunk in (0, unit):
        same(p.check_races(gen="jit", chunk_max_accesses=chunk, detect=detect), o)


# ---- full race listing (NEXT-4) ----------------------------------------------

@pytest.mark.parametrize("name,sizes", CASES, ids=[f"{n}-{i}" for i, (n, _) in enumerate(CASES)])
def test_race_list_matches_oracle(name, sizes):
    inst = config(name, **sizes)
    want = oracle.list_races_instance(inst)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    total, got = p.list_races(cap=len(want) + 10)
    assert total == len(want)
    assert [w.as_tuple() for w in got] == want
    # chunks forced to one (phase, block) unit: the merged lists stay canonical
    unit = max(1, p.info.max_unit_accesses)
    total, got = p.list_races(cap=len(want) + 10, chunk_max_accesses=unit)
    assert total == len(want) and [w.as_tuple() for w in got] == want


def test_race_list_prefix_and_fuzz():
    bad = []
    for seed in range(0, 300, 3):
        inst, _ = fuzz.random_instance(seed)
        want = oracle.list_races_instance(inst, threads=1)
        p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
        for cap in (0, 1, 3, len(want) + 1):
            total, got = p.list_races(cap=cap)
            if total != len(want) or [w.as_tuple() for w in got] != want[:cap]:
                bad.append((seed, cap, inst.src))
    assert not bad, bad[:3]


def test_race_list_long_segments():
    src = "params N; forU x in 0..N { rd[x % 8] }; wr[tid % 4]"
    want = oracle.list_races(src, block=(1024, 1, 1), params={"N": 4096})
    total, got = mc.MapProgram(src, (1, 1, 1), (1024, 1, 1), {"N": 4096}).list_races(cap=100)
    assert total == len(want) and [w.as_tuple() for w in got] == want


@pytest.mark.parametrize("name", ["3b", "4b"])
def test_race_list_full_size_properties(name):
    inst = config(name)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    r = p.check_races()
    total, got = p.list_races(cap=4096)
    assert total == r.racy_segments
    assert got[0].as_tuple() == r.witness.as_tuple()
    tuples = [w.as_tuple() for w in got]
    assert tuples == sorted(tuples) and len(set(t[:4] for t in tuples)) == len(tuples)


@pytest.mark.parametrize("detect", ["table", "sort", "direct"])
def test_scattered_indices_two_bucket_passes(detect):
    # 2^21 accesses over a 2^22-cell index space, scattered by the index expression:
    # two radix passes on the bucket bits whose next-pass digits are not warp-uniform,
    # so the scatter's range-table accumulation gives up and k_range_hist recomputes it
    src = "params N, M; forU x in 0..N { rd[(x * 7919 + tid * 104729) % M] }; if (tid = 7) { wr[5] } else { skip }"
    params = {"N": 2048, "M": 1 << 22}
    r = mc.check(src, block=(1024, 1, 1), params=params, detect=detect)
    o = oracle.check(src, block=(1024, 1, 1), params=params)
    same(r, o)


# ---- sort-free direct-address detect (direct.cu) -----------------------------

def _got(r):
    return (r.verdict, r.witness.as_tuple() if r.witness else None, r.n_accesses, r.racy_segments)


def _want(o):
    return (o.verdict, o.witness, o.n_accesses, o.n_racy_segments)


@pytest.mark.parametrize("gen", ["vm", "jit"])
def test_fuzz_corpus_direct_detect(gen):
    bad = []
    seeds = range(1, 400, 2) if gen == "vm" else range(0, 120, 3)
    for seed in seeds:
        inst, _ = fuzz.random_instance(seed)
        o = oracle.check_instance(inst, threads=1)
        p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
        r = p.check_races(detect="direct", gen=gen)
        if _got(r) != _want(o):
            bad.append((seed, inst.src, _got(r), _want(o)))
        # one (phase, block) unit per chunk: the witness gate skips later racy chunks
        unit = max(1, p.info.max_unit_accesses)
        r = p.check_races(detect="direct", gen=gen, chunk_max_accesses=unit)
        if _got(r) != _want(o):
            bad.append((seed, "unit chunks", inst.src, _got(r), _want(o)))
    assert not bad, bad[:3]


@pytest.mark.parametrize("name,sizes", [("5a", dict(T=4, R=4, C=64)), ("3b", dict(ts=32, rw=8, grid=64)),
                                        ("4a", dict(n=4096)), ("2b", {})])
def test_direct_path_runs(name, sizes):
    # the automatic choice takes the direct path on dense configs: the fused
    # generate + table launches ran, and no key was generated or sorted
    inst = config(name, **sizes)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    r = p.check_races(profile=True)
    same(r, oracle.check_instance(inst))
    assert r.kernels["direct"]["launches"] > 0 and r.kernels["clear"]["launches"] > 0
    assert r.kernels["generate"]["launches"] == 0 and r.kernels["onesweep"]["launches"] == 0


def test_direct_u64_cells():
    # 65536 threads per block: w_tid = 16 > 15, so cells are u64
    for src in ["wr[tid % 7]", "rd[tid % 5]; if (tid = 40000) { wr[3] } else { skip }", "wr[tid]; rd[tid]"]:
        o = oracle.check(src, block=(1024, 64, 1))
        for detect in ("direct", "sort"):
            same(mc.check(src, block=(1024, 64, 1), detect=detect), o)


def test_direct_racy_every_chunk():
    # every phase racy, one phase per chunk: only the first racy chunk folds a
    # witness (later phases cannot hold the minimum); the racy counts still add up
    inst = config("5b", block=64, T=6, R=4, C=16)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    o = oracle.check_instance(inst)
    unit = max(1, p.info.max_unit_accesses)
    for gen in ("vm", "jit"):
        same(p.check_races(detect="direct", gen=gen, chunk_max_accesses=unit), o)


def test_direct_broadcast_witness_cell():
    # the witness cell holds 2^20 + 1024 accesses: the filter re-emits all of them
    src = "forU x in 0..1024 { rd[0] }; wr[0]"
    o = oracle.check(src, block=(1024, 1, 1))
    for gen in ("vm", "jit"):
        same(mc.check(src, block=(1024, 1, 1), detect="direct", gen=gen), o)


@pytest.mark.parametrize("src,params", [
    ("params N; forU c in 0..N { wr[c + 1 + tid * N] }", {"N": 64}),                      # odd base: no pairs
    ("params N; forU c in 0..N { if (c % 3 = 1) { wr[c + tid * N] } else { rd[c + tid * N] } }", {"N": 64}),
    ("params N; forU c in 0..N { rd[c + tid * (N - 1)]; if (c = 5) { wr[c + tid * (N - 1)] } else { skip } }",
     {"N": 33}),                                                                            # overlaps, odd rows
    ("params N; forU c in 0..N { rd[2 * c]; wr[2 * c + 1 + (tid % 2)] }", {"N": 100}),      # stride 2
])
def test_direct_paired_cells(src, params):
    # the paired direct generate (two consecutive tuples per thread, one red.or.b64
    # for adjacent aligned cells) on aligned, unaligned, guarded and strided sites
    o = oracle.check(src, block=(64, 1, 1), grid=(3, 1, 1), params=params)
    for gen in ("jit", "vm"):
        same(mc.check(src, block=(64, 1, 1), grid=(3, 1, 1), params=params, detect="direct", gen=gen), o)


@pytest.mark.parametrize("name,sizes", [("5a", dict(T=6, R=4, C=64)), ("5b", dict(T=5, R=4, C=64)),
                                        ("4b", dict(n=1 << 14, bs=256))])
def test_overlapped_and_sequential_direct_pipelines_agree(name, sizes):
    # the overlapped direct pipeline (side stream, two tables, two control blocks)
    # and MAP_EXEC_SEQUENTIAL give the oracle's result, also with every rank share
    inst = config(name, **sizes)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    o = oracle.check_instance(inst)
    unit = max(1, p.info.max_unit_accesses)
    for overlap in (True, False):
        same(p.check_races(gen="jit", detect="direct", chunk_max_accesses=unit, overlap=overlap), o)
    # a 3-way shard: the ranks' counts add up and their witnesses' minimum is the oracle's
    parts = [p.check_races(gen="jit", detect="direct", chunk_max_accesses=unit, rank=r, world=3) for r in range(3)]
    assert sum(x.n_accesses for x in parts) == o.n_accesses
    assert sum(x.racy_segments for x in parts) == o.n_racy_segments
    wits = [x.witness.as_tuple() for x in parts if x.witness]
    assert (min(wits) if wits else None) == o.witness


def test_fuzz_unit_stride_sites():
    # fuzz instances whose direct-mode JIT marks a site unit-stride (the run-time
    # adjacency test folded away at compile time), JIT generate on
    # the direct path, default and unit chunks, vs the oracle
    import re
    bad, picked = [], 0
    for seed in range(0, 1500):
        inst, _ = fuzz.random_instance(seed)
        p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
        if not any("true" in x for c in range(min(p.n_chunks(0), 4))
                   for x in re.findall(r"US_\[\d+\] = \{([^}]*)\}", p.jit_source(c, 1))):
            continue
        o = oracle.check_instance(inst, threads=1)
        if o.status != 0:
            continue
        picked += 1
        unit = max(1, p.info.max_unit_accesses)
        for chunk in (0, unit):
            if chunk and p.n_chunks(chunk) > 16:
                continue
            r = p.check_races(detect="direct", gen="jit", chunk_max_accesses=chunk)
            if _got(r) != _want(o):
                bad.append((seed, chunk, inst.src, _got(r), _want(o)))
    assert picked >= 20 and not bad, (picked, bad[:3])


# ---- the key-exchange mode through real torch.distributed (NCCL, world 1) ------

@pytest.mark.parametrize("name", ["3b", "4b", "5b", "2b"])
def test_exchange_mode_real_nccl_world1(name):
    # dist.check_races_exchange end to end on one GPU with a real NCCL process group of
    # one rank: the pipelined path (async all_to_all under the previous chunk's sort,
    # two scratch buffers and streams) gives the oracle's result, also with unit chunks
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_2203_12878_b200.dist import check_races_exchange
    sizes = dict(CASES)[name] if name in dict(CASES) else {}
    inst = config(name, **sizes)
    o = oracle.check_instance(inst)
    if not dist.is_initialized():
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(sk.getsockname()[1])
        sk.close()
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    unit = max(1, p.info.max_unit_accesses)
    for chunk in (0, unit):
        if chunk and p.n_chunks(chunk) > 64:
            continue
        scratch = torch.empty(p.scratch_bytes(chunk), dtype=torch.uint8, device="cuda")
        r = check_races_exchange(p, scratch, chunk_max_accesses=chunk)
        assert (r.verdict, r.witness.as_tuple() if r.witness else None, r.n_accesses, r.racy_segments) == \
               (o.verdict, o.witness, o.n_accesses, o.n_racy_segments), (name, chunk)


def teardown_module(module):
    import torch.distributed as dist
    if dist.is_initialized():
        dist.destroy_process_group()
