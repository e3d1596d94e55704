"""Multi-GPU partitioning of decode units and the host orchestration
of one sharded decode step.

A unit is one (sequence, KV head) pair: it owns its centroid segment, its selection
and its KV pages, and exchanges nothing with other units. A BASELINE configuration
fixes the GLOBAL batch (cfg3: 16 sequences on 1/2/4/8 GPUs), so ranks take contiguous
batch ranges (every GPU runs the identical kernel shape when N divides the batch);
when the batch is smaller than the world (cfg1: batch 1), each sequence's KV heads are
split into contiguous head ranges instead. There is no collective on the data path;
the only exchange is the optional all-gather of the per-rank outputs
[b_local][Hq_local][d] into the global [b][Hq][d] (NCCL over NVLink on GPUs, gloo in
the CPU tests), reported separately from the attention throughput.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Sequence


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
    """Batch ranges when batch >= world (or world does not divide into the batch),
    otherwise KV-head ranges of one sequence per group of world // batch ranks."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    if batch >= world or world % batch != 0:
        b0, bc = _split(batch, world, rank)
        return Shard(b0, bc, 0, heads if bc else 0)
    per_seq = world // batch           # ranks sharing one sequence
    b = rank // per_seq
    h0, hc = _split(heads, per_seq, rank % per_seq)
    return Shard(b, 1, h0, hc)


@dataclass(frozen=True)
class ShardPlan:
    """The shard of rank `rank` in a world of `world` for a global batch of `batch`
    sequences with `heads` KV heads and G query heads per KV head."""
    batch: int
    heads: int
    G: int
    world: int
    rank: int

    @property
    def shard(self) -> Shard:
        return shard_units(self.batch, self.heads, self.world, self.rank)

    @property
    def head_sharded(self) -> bool:
        return self.shard.head_count != self.heads

    def shards(self) -> list:
        return [shard_units(self.batch, self.heads, self.world, r) for r in range(self.world)]

    def block_sizes(self, assignment: Sequence[int]) -> list:
        """This rank's slice of the per-KV-head block-size table."""
        s = self.shard
        return list(assignment[s.head_start:s.head_start + s.head_count])

    def local_q(self, q):
        """[b][Hq][d] global query -> this rank's [b_local][Hq_local][d] (a view)."""
        s = self.shard
        return q[s.batch_start:s.batch_start + s.batch_count,
                 s.head_start * self.G:(s.head_start + s.head_count) * self.G]

    def max_local(self) -> tuple:
        """(max b_local, max Hq_local) over ranks: the padded all-gather slot."""
        sh = self.shards()
        return max(s.batch_count for s in sh), max(s.head_count for s in sh) * self.G

    def assemble(self, slots, out):
        """slots[r]: rank r's padded [b_max][Hq_max][d] output; writes the global out."""
        for r, s in enumerate(self.shards()):
            if s.batch_count == 0 or s.head_count == 0:
                continue
            out[s.batch_start:s.batch_start + s.batch_count,
                s.head_start * self.G:(s.head_start + s.head_count) * self.G] = \
                slots[r][:s.batch_count, :s.head_count * self.G]
        return out


class ShardedDecode:
    """One sharded decode step: the rank's local step on its slice of the global query,
    then (optionally) an all-gather of every rank's output into the global layout.

    local_step(q_local, out_local) runs the rank's decode step (on a GPU:
    DecodeAttention.decode_step over the rank's own context); `group` is the
    torch.distributed process group (NCCL on GPUs, gloo in the CPU tests)."""

    def __init__(self, plan: ShardPlan, local_step: Callable, d: int, torch_mod, device=None,
                 dtype=None, group=None):
        self.plan, self.local_step, self.d = plan, local_step, d
        self.torch = torch_mod
        self.group = group
        b_max, hq_max = plan.max_local()
        dt = dtype or torch_mod.float32
        self.slot = torch_mod.zeros(b_max, hq_max, d, dtype=dt, device=device)
        self.gathered = torch_mod.zeros(plan.world, b_max, hq_max, d, dtype=dt, device=device)

    def step(self, q_global, out_global: Optional[object] = None):
        s = self.plan.shard
        local = self.slot[:s.batch_count, :s.head_count * self.plan.G]
        if s.batch_count and s.head_count:
            self.local_step(self.plan.local_q(q_global), local)
        if out_global is None:
            return local
        self.gather()
        return self.plan.assemble(list(self.gathered), out_global)

    def gather(self):
        """All-gather of the padded per-rank slots (the only exchange of the path)."""
        dist = self.torch.distributed
        if self.plan.world == 1:
            self.gathered[0].copy_(self.slot)
        else:
            dist.all_gather_into_tensor(self.gathered.view(-1), self.slot.view(-1), group=self.group)
        return self.gathered
