"""Synthetic paged layers shared by the CPU and GPU tests (numpy on the host).

A layer is a batch of sequences over per-head bf16 page pools
[H][pool_pages][P][d] with one page table per sequence; pages are handed out in
a shuffled order so that every read really goes through the page table.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from oracle.oracle import OracleSeq, f32_to_bf16, group_sum, oracle_decode


@dataclass
class Layer:
    H: int
    G: int
    d: int
    P: int
    block_sizes: list
    seq_lens: list
    k_pool: np.ndarray      # uint16 [H][pool_pages][P][d]
    v_pool: np.ndarray
    page_table: np.ndarray  # uint32 [batch][max_pages]
    q: np.ndarray           # uint16 [batch][H*G][d]

    @property
    def batch(self) -> int:
        return len(self.seq_lens)

    def qf(self, b: int) -> np.ndarray:
        return (self.q[b].astype(np.uint32) << 16).view(np.float32)

    def oracle_seq(self, b: int, method=0, bits=4, mode=1) -> OracleSeq:
        pages = (self.seq_lens[b] + self.P - 1) // self.P
        return OracleSeq(self.k_pool, self.v_pool, self.page_table[b, :pages], self.seq_lens[b], self.H,
                         self.d, self.P, self.block_sizes, method, bits, mode)


def make_layer(seed, H=8, G=4, d=128, P=16, block_sizes=(16, 32, 64), seq_lens=(1000,), extra_pages=3,
               scale=1.0, kv=None, q=None, sequential=False, swaps=0) -> Layer:
    """sequential: pages handed out in order (the reference allocator, kv_cache.cpp:53-60),
    with `swaps` random page pairs exchanged to break some contiguous runs."""
    rng = np.random.default_rng(seed)
    bs = [block_sizes[h % len(block_sizes)] for h in range(H)] if len(block_sizes) != H else list(block_sizes)
    pages_per = [(n + P - 1) // P for n in seq_lens]
    pool_pages = sum(pages_per) + extra_pages
    if kv is None:
        kf = (rng.standard_normal((H, pool_pages, P, d)) * scale).astype(np.float32)
        vf = rng.standard_normal((H, pool_pages, P, d)).astype(np.float32)
    else:
        kf, vf = kv
    perm = rng.permutation(pool_pages).astype(np.uint32)
    if sequential:
        perm = np.arange(pool_pages, dtype=np.uint32)
        for _ in range(swaps):
            a, b = rng.integers(0, pool_pages, 2)
            perm[a], perm[b] = perm[b], perm[a]
    max_pages = max(pages_per) + 1
    pt = np.zeros((len(seq_lens), max_pages), np.uint32)
    o = 0
    for b, p in enumerate(pages_per):
        pt[b, :p] = perm[o:o + p]
        o += p
    if q is None:
        qf = rng.standard_normal((len(seq_lens), H * G, d)).astype(np.float32)
    else:
        qf = q
    return Layer(H, G, d, P, bs, list(seq_lens), f32_to_bf16(kf), f32_to_bf16(vf), pt, f32_to_bf16(qf))


def oracle_step(layer: Layer, b: int, token_budget: int, method=0, bits=4, mode=1):
    """(OracleSeq, scores, selection, out[H*G][d]) for sequence b."""
    seq = layer.oracle_seq(b, method, bits, mode)
    sc, sel, out = oracle_decode(seq, layer.qf(b), layer.G, token_budget)
    return seq, sc, sel, out


__all__ = ["Layer", "make_layer", "oracle_step", "group_sum"]
