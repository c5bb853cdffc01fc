"""Text-sharded HC search over several GPUs.

The window ends [m-1, n) are split into `world` contiguous ranges, one per rank.
Rank r searches only its slice of the text: y[e_lo - m + 1, e_hi), where [e_lo, e_hi)
are its window ends.  That slice has an (m-1)-byte left halo.  By reading R11
(segment exactness), HC on that slice reports exactly the occurrences
whose end lies in [e_lo, e_hi).  The ranks' lists are disjoint.  Each is sorted,
and the ranges are in rank order, so the global answer is their concatenation in
rank order; no merge is needed.

There is one exchange step, over torch.distributed (NCCL on GPUs):
  1. all_gather of the per-rank counts (one int64 each);
  2. a variable-size all-gather of the position lists, sized to the actual counts
     (all_to_all_single with output splits = the counts: rank r receives exactly
     sum(counts) positions, no padding to the largest list).
Both are negligible next to each rank reading its own n/world bytes.

The per-rank search is `hc.search` (the CUDA path) unless a `searcher` is passed;
the CPU tests pass one so that the sharding and exchange logic runs under gloo.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    """Rank `rank`'s part of a text of n bytes for a pattern of length m."""
    text_lo: int   # first text byte of the slice (the left halo starts here)
    text_hi: int   # one past the last text byte of the slice
    end_lo: int    # first window end owned
    end_hi: int    # one past the last window end owned

    @property
    def size(self) -> int:
        return self.text_hi - self.text_lo


def shard_bounds(n: int, m: int, world: int, rank: int) -> Shard:
    """Window ends [m-1, n) cut into `world` contiguous ranges; rank r owns the r-th.
    An empty range yields an empty slice (size 0)."""
    if world < 1 or not 0 <= rank < world or m < 1:
        raise ValueError("need world >= 1, 0 <= rank < world, m >= 1")
    W = max(0, n - m + 1)                      # number of windows
    e_lo = m - 1 + (W * rank) // world
    e_hi = m - 1 + (W * (rank + 1)) // world
    if e_hi <= e_lo:
        return Shard(e_lo, e_lo, e_lo, e_lo)
    return Shard(e_lo - m + 1, e_hi, e_lo, e_hi)


def gather_positions(local: torch.Tensor, offset: int = 0, group=None) -> tuple[int, torch.Tensor]:
    """All-gather of per-rank ascending int64 position lists in rank order, each shifted by
    its rank's `offset` (the slice's first text byte: positions become global).  The
    exchange moves exactly the positions that exist (no padding).  Returns (total count,
    concatenated positions) on every rank."""
    world = dist.get_world_size(group)
    dev = local.device
    local = local.to(torch.int64)
    if offset:
        local = local + offset
    cnt = torch.tensor([local.numel()], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    total = sum(counts)
    out = torch.empty(total, dtype=torch.int64, device=dev)
    if total:
        # variable all-gather: every rank sends its list to every rank
        src = local.repeat(world) if local.numel() else local
        dist.all_to_all_single(out, src, output_split_sizes=counts,
                               input_split_sizes=[local.numel()] * world, group=group)
    return total, out


def _gpu_search(h, y_slice: torch.Tensor, max_out):
    from . import hc
    return hc.search(h, y_slice, max_out=max_out)


def search_sharded(h, y_slice: torch.Tensor, shard: Shard, max_out: int | None = None,
                   group=None, searcher=None) -> tuple[int, torch.Tensor]:
    """Search this rank's slice (y_slice = y[shard.text_lo:shard.text_hi], resident on
    this rank's device), then exchange.  Returns (count, positions) on every rank.
    With max_out, each rank keeps its max_out smallest positions: the global
    max_out smallest are a prefix of the rank-ordered concatenation.  The count is
    then exact only if no rank hit max_out (the returned count is a lower bound and
    `positions` has min(count, max_out) entries)."""
    if y_slice.numel() != shard.size:
        raise ValueError("y_slice does not match the shard")
    search = searcher or _gpu_search
    if shard.size >= h.m:
        local = search(h, y_slice, max_out).to(torch.int64)
    else:
        local = torch.empty(0, dtype=torch.int64, device=y_slice.device)
    total, pos = gather_positions(local, shard.text_lo, group)
    if max_out is not None:
        pos = pos[:max_out]
    return total, pos
