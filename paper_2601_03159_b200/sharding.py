"""Series-range sharding across GPUs.

Every stream depends only on (master_seed, stage, GLOBAL series index)
(reference core.py:48-82) and rows are written disjointly (core.py:146-151),
so a batch splits into contiguous row ranges with no data-path collective:
rank r runs the fused kernel on rows [lo, hi) with series_offset = lo.  After
a Repeat(r) stage the global output index is offset * r + local row
(basic.py:400-409), which the kernel derives from the same offset.
"""

from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) of n rows for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    return n * rank // world, n * (rank + 1) // world


def run_shard(pipe, values_shard, lo: int):
    """Run `pipe` on this rank's device-resident shard (rows [lo, lo + n))."""
    return pipe.run_device(values_shard, series_offset=lo)
