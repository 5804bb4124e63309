"""Multi-GPU sharding of the match path, one process per GPU.

Every start offset is independent (reference scan.cpp:82-87), so the text is
cut into contiguous shards: rank r owns starts [lo_r, hi_r) and receives the
bytes [lo_r, min(N, hi_r + halo)), with halo = reach - 1 (hepfac_b200_halo).
Walks stop at the shard's byte end, which equals the global end for the last
shard and is never reached early by a valid walk for the others, so each
shard's list equals the whole-text list restricted to its starts.  The only
cross-GPU step is an exclusive scan of the per-shard match counts (one u64 per
rank through an all_gather), which gives each rank the offset of its slice in
the global, (start, length, id)-ordered result; concatenation in rank order is
already globally sorted.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np


# hepfac_b200_halo reports an unbounded halo (a cyclic loaded trie) as
# UINT64_MAX; Library.halo maps it to None.
UNBOUNDED = (1 << 64) - 1


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    lo: int      # first owned start (global)
    owned: int   # number of owned starts
    end: int     # one past the last byte this shard holds (global)

    @property
    def nbytes(self) -> int:
        return self.end - self.lo


def plan(n: int, world: int, rank: int, halo: Optional[int]) -> Shard:
    """Contiguous shard of an n-byte text for `rank` of `world`."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    if halo is None or halo < 0 or halo >= UNBOUNDED:
        raise ValueError("unbounded walks (cyclic trie): shards cannot be used")
    lo = rank * n // world
    hi = (rank + 1) * n // world
    return Shard(rank, world, lo, hi - lo, min(n, hi + halo))


def exclusive_offset(count: int, group=None) -> tuple:
    """K4: exclusive scan of one u64 per rank (all_gather).  Returns
    (this rank's offset, global total)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        return 0, count
    backend = dist.get_backend(group)
    device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([count], dtype=torch.int64, device=device)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    counts = [int(x.item()) for x in out]
    r = dist.get_rank(group)
    return sum(counts[:r]), sum(counts)


def scan_sharded(text: np.ndarray, shard: Shard, scanner: Callable, group=None):
    """Scan this rank's shard with `scanner(shard_bytes, lo, owned)` (the
    B200 library's scan_shard in production) and place it globally.
    `text` is either the whole text or exactly this shard's bytes.
    Returns (records, global offset, global total)."""
    if text.size == shard.nbytes:
        local_bytes = text
    else:
        local_bytes = text[shard.lo:shard.end]
    recs = scanner(local_bytes, shard.lo, shard.owned)
    off, total = exclusive_offset(int(recs.size), group)
    return recs, off, total


def gather_all(recs: np.ndarray, group=None) -> Optional[np.ndarray]:
    """Collects every rank's records on rank 0, in rank order (tests/tools)."""
    import torch.distributed as dist
    if not dist.is_initialized():
        return recs
    parts = [None] * dist.get_world_size(group)
    dist.all_gather_object(parts, recs, group=group)
    return np.concatenate(parts) if dist.get_rank(group) == 0 else None
