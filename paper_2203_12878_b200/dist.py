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


def _exchange_chunk(prog: MapProgram, chunk: int, scratch, stream, chunk_max_accesses: int, group, device):
    """One chunk of the key-exchange mode: (packed witness or None, racy count, n keys)."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    bound = prog.chunk_info(chunk, chunk_max_accesses)["bound"]
    out = torch.empty(max(bound, 1), dtype=torch.int64, device=device)
    counts = prog.generate_bucketed(chunk, rank, world, out, scratch, stream, chunk_max_accesses)
    send = torch.tensor(counts, dtype=torch.int64, device=device)
    recv = torch.empty_like(send)
    _comm(dist.all_to_all_single, recv, send, group=group)            # counts
    rsizes = [int(x) for x in recv.tolist()]
    got = torch.empty(max(sum(rsizes), 1), dtype=torch.int64, device=device)
    _comm(dist.all_to_all_single, got[:sum(rsizes)], out[:sum(counts)], output_split_sizes=rsizes,
          input_split_sizes=counts, group=group)                       # keys, bucketed by hash
    packed, racy = prog.sort_detect(chunk, got, sum(rsizes), scratch, stream, chunk_max_accesses)
    return packed, racy, sum(rsizes)


def check_races_exchange(prog: MapProgram, scratch, stream=None, chunk_max_accesses: int = 0,
                         group=None) -> Result:
    """Key-exchange mode over all chunks; every rank returns the global result."""
    device = scratch.device
    best, n_total, racy_total = None, 0, 0
    for c in range(prog.n_chunks(chunk_max_accesses)):
        packed, racy, n = _exchange_chunk(prog, c, scratch, stream, chunk_max_accesses, group, device)
        racy_total += racy
        n_total += n
        if packed is not None:
            w = prog.unpack_witness(c, packed).as_tuple()
            best = w if best is None or w < best else best
    local = Result(verdict=1 if best else 0, n_accesses=n_total, racy_segments=racy_total,
                   n_chunks=prog.n_chunks(chunk_max_accesses), device_ms=0.0, gpu_launches=0)
    if best:
        local.witness = Witness(*best, array_name="")
    return reduce_results(local, prog.array_names(), group=group, device=device)
