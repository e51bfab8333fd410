"""Multi-GPU orchestration: one process per GPU, torch.distributed for plumbing.

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

from . import MapProgram, Result, Witness

_NONE = -1


def _pack(r: Result, device) -> torch.Tensor:
    w = r.witness.as_tuple() if r.witness else (_NONE,) * 8
    return torch.tensor([r.verdict, r.n_accesses, r.racy_segments, *w], dtype=torch.int64, device=device)


def reduce_results(local: Result, array_names, group=None, device="cpu") -> Result:
    """Combine per-rank results: min witness (lexicographic), summed counts."""
    world = dist.get_world_size(group)
    mine = _pack(local, device)
    bufs = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(bufs, mine, group=group)
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
