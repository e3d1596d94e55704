"""Multi-GPU partitioning of decode units.

A unit is one (sequence, KV head) pair: it owns its centroid segment, its selection
and its KV pages, and exchanges nothing with other units. Ranks therefore take
contiguous batch ranges (every GPU runs the identical kernel shape); when the batch
is smaller than the world (config 1: batch 1), each sequence's KV heads are split
into contiguous head ranges instead. No collective is needed on the data path.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    batch_start: int
    batch_count: int
    head_start: int
    head_count: int


def _split(n: int, parts: int, i: int) -> tuple:
    base, rem = divmod(n, parts)
    start = i * base + min(i, rem)
    return start, base + (1 if i < rem else 0)


def shard_units(batch: int, heads: int, world: int, rank: int) -> Shard:
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    if batch >= world or world % batch != 0:
        b0, bc = _split(batch, world, rank)
        return Shard(b0, bc, 0, heads if bc else 0)
    per_seq = world // batch           # ranks sharing one sequence
    b = rank // per_seq
    h0, hc = _split(heads, per_seq, rank % per_seq)
    return Shard(b, 1, h0, hc)
