"""Multi-GPU orchestration: one process per GPU, torch.distributed for plumbing.

Two modes:
  * chunk sharding (default, ``check_races_distributed``): no data-path collective;
  * key exchange (``check_races_exchange``): for (phase, block) units too large
    for one GPU -- every rank generates a slice of each chunk's tuples, keys are
    routed by hash of their sort field with one NCCL all_to_all_single, each
    rank sorts + detects what it received, and the ranks reduce the witness.


The path shards naturally: barrier phases and blocks are
independent units -- races are intra-(phase, block) -- so
the library's chunks (ranges of phases, or of blocks of one phase) are dealt
round-robin to ranks with NO data-path collective.  The only exchange is the
final reduction of the per-rank results: a 10-word all-gather from which
every rank takes the lexicographic minimum witness and the summed counts
(SURVEY.md §8e "all-reduce-min picks the global witness"; the witness tuple
does not fit one 64-bit word in general, so it is gathered, not min-reduced).
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist

from . import MapError, MapProgram, Result, Witness

_NONE = -1
MAP_E_COMM = 7          # include/mapcheck.h: a failed collective (NCCL / gloo)


def _comm(fn, *args, **kw):
    """Run a torch.distributed collective; a failure becomes MapError(MAP_E_COMM)."""
    try:
        return fn(*args, **kw)
    except (RuntimeError, ValueError) as e:          # NCCL / gloo errors surface as RuntimeError
        raise MapError(MAP_E_COMM, f"{getattr(fn, '__name__', 'collective')}: {e}") from e


def _pack(r: Result, device) -> torch.Tensor:
    w = r.witness.as_tuple() if r.witness else (_NONE,) * 8
    return torch.tensor([r.verdict, r.n_accesses, r.racy_segments, *w], dtype=torch.int64, device=device)


def reduce_results(local: Result, array_names, group=None, device="cpu") -> Result:
    """Combine per-rank results: min witness (lexicographic), summed counts."""
    world = dist.get_world_size(group)
    mine = _pack(local, device)
    bufs = [torch.empty_like(mine) for _ in range(world)]
    _comm(dist.all_gather, bufs, mine, group=group)
    rows = [b.cpu().tolist() for b in bufs]
    n = sum(r[1] for r in rows)
    racy = sum(r[2] for r in rows)
    wits = [tuple(r[3:]) for r in rows if r[0] == 1]
    out = Result(verdict=1 if wits else 0, n_accesses=n, racy_segments=racy, n_chunks=local.n_chunks,
                 device_ms=local.device_ms, gpu_launches=local.gpu_launches, h2d_bytes=local.h2d_bytes,
                 d2h_bytes=local.d2h_bytes, kernels=local.kernels)
    if wits:
        w = min(wits)
        out.witness = Witness(*w, array_name=array_names[w[1]] if array_names else "")
    return out


def check_races_distributed(prog: MapProgram, scratch=None, stream=None, chunk_max_accesses: int = 0,
                            group=None, profile: bool = False, array_names=None) -> Result:
    """Run this rank's share of the chunks, then reduce across ranks."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    local = prog.check_races(scratch=scratch, stream=stream, chunk_max_accesses=chunk_max_accesses,
                             rank=rank, world=world, profile=profile)
    dev = scratch.device if scratch is not None else (
        torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu")
    names = array_names if array_names is not None else prog.array_names()
    return reduce_results(local, names, group=group, device=dev)


def _exchange_start(prog, chunk, scratch, stream, chunk_max_accesses, group, device):
    """Generate chunk `chunk`'s slice bucketed by destination, swap the counts, and
    START the key all_to_all (async_op): returns the in-flight state."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    bound = prog.chunk_info(chunk, chunk_max_accesses)["bound"]
    out = torch.empty(max(bound, 1), dtype=torch.int64, device=device)
    counts = prog.generate_bucketed(chunk, rank, world, out, scratch, stream, chunk_max_accesses)
    send = torch.tensor(counts, dtype=torch.int64, device=device)
    recv = torch.empty_like(send)
    _comm(dist.all_to_all_single, recv, send, group=group)            # counts (small, blocking)
    rsizes = [int(x) for x in recv.tolist()]
    got = torch.empty(max(sum(rsizes), 1), dtype=torch.int64, device=device)
    work = _comm(dist.all_to_all_single, got[:sum(rsizes)], out[:sum(counts)], output_split_sizes=rsizes,
                 input_split_sizes=counts, group=group, async_op=True)   # keys, bucketed by hash
    return {"chunk": chunk, "out": out, "got": got, "n": sum(rsizes), "work": work, "scratch": scratch,
            "stream": stream}


def _exchange_finish(prog, st, chunk_max_accesses):
    """Wait for a chunk's keys and sort + detect them: (packed witness or None, racy, n)."""
    if st["stream"] is not None:                     # the sort's stream waits for the transfer
        with torch.cuda.stream(st["stream"]):
            _comm(st["work"].wait)
    else:
        _comm(st["work"].wait)
    packed, racy = prog.sort_detect(st["chunk"], st["got"], st["n"], st["scratch"], st["stream"], chunk_max_accesses)
    return packed, racy, st["n"]


def check_races_exchange(prog: MapProgram, scratch, stream=None, chunk_max_accesses: int = 0,
                         group=None, scratch2=None) -> Result:
    """Key-exchange mode over all chunks; every rank returns the global result.

    Software-pipelined two deep (the exchange "must overlap with
    K3 of the previous phase"): chunk c's keys travel (an async all_to_all)
    while chunk c-1's received keys are sorted and race-checked, each chunk on
    its own scratch buffer and CUDA stream (scratch2: a second buffer of the same
    size; allocated here when None on a GPU)."""
    device = scratch.device
    cuda = device.type == "cuda"
    if cuda and scratch2 is None:
        scratch2 = torch.empty_like(scratch)
    scratches = [scratch, scratch2 if scratch2 is not None else scratch]
    streams = [stream, torch.cuda.Stream(device=device)] if cuda else [None, None]
    best, n_total, racy_total = None, 0, 0

    def fold(c, res):
        nonlocal best, n_total, racy_total
        packed, racy, n = res
        racy_total += racy
        n_total += n
        if packed is not None:
            w = prog.unpack_witness(c, packed).as_tuple()
            best = w if best is None or w < best else best

    pending = None
    for c in range(prog.n_chunks(chunk_max_accesses)):
        slot = c % 2 if scratch2 is not None else 0
        st = _exchange_start(prog, c, scratches[slot], streams[slot], chunk_max_accesses, group, device)
        if pending is not None:                       # the previous chunk, under this chunk's transfer
            fold(pending["chunk"], _exchange_finish(prog, pending, chunk_max_accesses))
        pending = st
    if pending is not None:
        fold(pending["chunk"], _exchange_finish(prog, pending, chunk_max_accesses))
    if cuda:
        torch.cuda.current_stream(device).wait_stream(streams[1])
    local = Result(verdict=1 if best else 0, n_accesses=n_total, racy_segments=racy_total,
                   n_chunks=prog.n_chunks(chunk_max_accesses), device_ms=0.0, gpu_launches=0)
    if best:
        local.witness = Witness(*best, array_name="")
    return reduce_results(local, prog.array_names(), group=group, device=device)
