"""Multi-GPU host logic on CPU: world_size-2 gloo process group.

The GPU step is replaced by per-rank synthetic results (each rank would have
processed its share of the chunks, map_rank_chunks); what is tested is the cross-rank reduction
of paper_2203_12878_b200.dist: summed counts and the lexicographic minimum
witness, identical on every rank.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = {
    # rank -> (verdict, n, racy, witness tuple or None)
    "both_racy": {0: (1, 100, 3, (2, 0, 0, 7, 1, 4, 0, 1)), 1: (1, 50, 2, (1, 1, 0, 9, 0, 3, 1, 1))},
    "one_racy": {0: (0, 10, 0, None), 1: (1, 20, 1, (5, 0, 3, 1, 2, 9, 1, 0))},
    "none": {0: (0, 7, 0, None), 1: (0, 8, 0, None)},
    "tie_on_prefix": {0: (1, 1, 1, (0, 0, 0, 4, 2, 5, 1, 1)), 1: (1, 1, 1, (0, 0, 0, 4, 2, 5, 0, 1))},
}


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2203_12878_b200 import Result, Witness
        from paper_2203_12878_b200.dist import reduce_results
        v, n, racy, w = CASES[case][rank]
        local = Result(verdict=v, n_accesses=n, racy_segments=racy, n_chunks=1, device_ms=1.0, gpu_launches=3)
        if w:
            local.witness = Witness(*w, array_name="")
        out = reduce_results(local, ["A", "B"], device="cpu")
        q.put((rank, out.verdict, out.n_accesses, out.racy_segments,
               out.witness.as_tuple() if out.witness else None, out.witness.array_name if out.witness else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", list(CASES))
def test_reduce_results_world2(case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rows = CASES[case]
    wits = [w for (v, _, _, w) in rows.values() if v]
    want_w = min(wits) if wits else None
    want = (1 if wits else 0, sum(r[1] for r in rows.values()), sum(r[2] for r in rows.values()), want_w)
    for (_, v, n, racy, w, name) in outs:
        assert (v, n, racy, w) == want
        if w:
            assert name == ["A", "B"][w[1]]


@pytest.mark.parametrize("name", ["3a", "3b", "4a", "4b", "5a", "5b"])
def test_chunk_sharding_covers_all_chunks(name):
    # map_rank_chunks (the shard map_check_races runs): every chunk exactly once,
    # contiguous per rank, every rank busy on the large configs, balanced bounds
    import paper_2203_12878_b200 as mc
    from workloads import config
    inst = config(name)
    p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    for world in (1, 2, 4, 8):
        chunk = p.default_chunk(world)
        n = p.n_chunks(chunk)
        shares = [p.rank_chunks(r, world, chunk) for r in range(world)]
        assert sorted(c for s in shares for c in s) == list(range(n))
        for s in shares:
            assert s == list(range(s[0], s[0] + len(s))) if s else True
        if world > 1:
            assert n >= world, (name, world, n)
            assert all(len(s) >= 1 for s in shares)
            work = [sum(p.chunk_info(c, chunk)["bound"] for c in s) for s in shares]
            assert max(work) <= 2 * (sum(work) / world), (name, world, work)


# ---- key-exchange mode orchestration (dist.check_races_exchange) -------------

class FakeProg:
    """Stands in for MapProgram on CPU: chunk c of rank r generates keys
    1000*c + 10*k + r (k < 5 + r); destination = key % world.  sort_detect
    records what arrived and reports its minimum key as the 'witness'."""

    def __init__(self, world):
        self.world = world
        self.received = []

    def n_chunks(self, chunk_max_accesses=0):
        return 3

    def chunk_info(self, chunk, chunk_max_accesses=0):
        return {"bound": 64}

    def array_names(self):
        return ["A"]

    def generate_bucketed(self, chunk, rank, world, out, scratch, stream=None, chunk_max_accesses=0):
        keys = [1000 * chunk + 10 * k + rank for k in range(5 + rank)]
        by = [[x for x in keys if x % world == d] for d in range(world)]
        flat = [x for b in by for x in b]
        out[:len(flat)] = torch.tensor(flat, dtype=torch.int64)
        return [len(b) for b in by]

    def sort_detect(self, chunk, keys, n, scratch, stream=None, chunk_max_accesses=0):
        got = keys[:n].tolist()
        self.received.append((chunk, sorted(got)))
        return (min(got) if got else None), len(got)

    def unpack_witness(self, chunk, packed):
        from paper_2203_12878_b200 import Witness
        return Witness(chunk, 0, 0, packed, 0, 1, 0, 1, "A")


def _xworker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2203_12878_b200.dist import check_races_exchange
        prog = FakeProg(world)
        out = check_races_exchange(prog, torch.empty(1))
        q.put((rank, prog.received, out.verdict, out.n_accesses, out.racy_segments, out.witness.as_tuple()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_routing(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_xworker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    total = sum(5 + r for r in range(world)) * 3
    for rank, received, verdict, n, racy, w in outs:
        for chunk, keys in received:
            want = sorted(1000 * chunk + 10 * k + s for s in range(world) for k in range(5 + s)
                          if (1000 * chunk + 10 * k + s) % world == rank)
            assert keys == want                      # every key arrives once, at its hash owner
        assert (verdict, n, racy) == (1, total, total)
        assert w == (0, 0, 0, 0, 0, 1, 0, 1)         # global min over chunks and ranks


def test_collective_failure_maps_to_map_e_comm():
    # a collective that fails (here: no process group) surfaces as MAP_E_COMM (7)
    from paper_2203_12878_b200 import MapError
    from paper_2203_12878_b200.dist import _comm
    assert not dist.is_initialized()
    with pytest.raises(MapError) as e:
        _comm(dist.all_gather, [torch.empty(3)], torch.zeros(3))
    assert e.value.status == 7 and "all_gather" in str(e.value)
