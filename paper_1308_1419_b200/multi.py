"""Multi-GPU lambda-range sharding, one process per GPU.

The triangular domain shards naturally: shard g of G owns the contiguous
block rows [rows[g], rows[g+1]) (tg_shard_rows: each boundary is the row start
nearest g*T(n)/G), hence a contiguous lambda-range and a contiguous slice of
the packed output in the reference layout.  Every rank writes its own slice
into its own HBM; there is no data-path collective.  The only exchange is the
optional collision hit count (one all-reduce of a u64) and the max-over-ranks
timing of the benchmark.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import trigrid as tg


@dataclass(frozen=True)
class Shard:
    index: int
    count: int
    block_rows: tuple[int, int]   # [b0, b1)
    elems: tuple[int, int]        # packed with-diagonal elements [e0, e1)
    pairs: tuple[int, int]        # packed no-diagonal pairs [p0, p1)

    @property
    def size(self) -> int:
        return self.elems[1] - self.elems[0]


def shard_plan(n: int, rho: int, world: int) -> list[Shard]:
    rows = tg.shard_rows(n, rho, world)
    out = []
    for g in range(world):
        e = tg.shard_elems(n, rho, g, world, True)
        p = tg.shard_elems(n, rho, g, world, False)
        out.append(Shard(g, world, (rows[g], rows[g + 1]), e, p))
    return out


def max_over_ranks(x: float, device=None) -> float:
    """Timing rule: a multi-GPU time is the max over ranks."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_hits(hits, device=None) -> int:
    """The single collective of the path: sum of per-shard collision counts."""
    import torch
    import torch.distributed as dist
    t = hits if isinstance(hits, torch.Tensor) else torch.tensor([int(hits)], dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())
