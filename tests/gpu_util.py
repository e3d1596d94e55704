"""Runs a host-side Layer (tests/layer_data.py) through the C ABI on cuda:0."""
from __future__ import annotations

import os

import numpy as np
import torch

from paper_2605_12110_b200 import (BlockAssignment, CentroidMethod, DecodeAttention, EngineConfig,
                                   QuantMode, QuantSpec)


def to_dev_u16(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda()


def to_dev_u32(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


class GpuLayer:
    def __init__(self, layer, T, method=0, bits=4, mode=1, max_seq_len=None, candidates=None, exact_select=False):
        """exact_select=True: decode steps score every centroid exactly and run the separate
        top-k (ABSP_EXACT_SELECT=1) instead of the fused filter + refine (select.cu)."""
        self.layer = layer
        cands = sorted(set(candidates or layer.block_sizes))
        self.cfg = EngineConfig(num_heads=layer.H, head_dim=layer.d, page_size=layer.P,
                                candidate_block_sizes=tuple(cands), token_budget=T,
                                centroid_method=CentroidMethod(method),
                                quant=QuantSpec(bits, QuantMode(mode)) if bits else None,
                                num_q_heads=layer.H * layer.G, max_batch=layer.batch,
                                max_seq_len=max_seq_len or max(layer.seq_lens), num_layers=1)
        old = os.environ.get("ABSP_EXACT_SELECT")
        os.environ["ABSP_EXACT_SELECT"] = "1" if exact_select else "0"
        try:
            self.da = DecodeAttention(self.cfg)
        finally:
            if old is None:
                del os.environ["ABSP_EXACT_SELECT"]
            else:
                os.environ["ABSP_EXACT_SELECT"] = old
        self.da.set_assignment(0, BlockAssignment(list(layer.block_sizes)))
        self.k = to_dev_u16(layer.k_pool)
        self.v = to_dev_u16(layer.v_pool)
        self.pt = to_dev_u32(layer.page_table)
        self.q = to_dev_u16(layer.q)
        self.da.bind(0, self.k, self.v, self.pt, layer.seq_lens)
        self.da.build_store(0)
        self.info = self.da.layer_info(0)

    def select(self):
        L = self.layer
        stride = max(self.info.max_select, 1)
        blocks = torch.zeros(L.batch, L.H, stride, dtype=torch.int32, device="cuda")
        counts = torch.zeros(L.batch, L.H, dtype=torch.int32, device="cuda")
        self.da.select(0, self.q, blocks, counts)
        torch.cuda.synchronize()
        b = blocks.cpu().numpy().view(np.uint32)
        c = counts.cpu().numpy().view(np.uint32)
        return [[b[s, h, :c[s, h]].copy() for h in range(L.H)] for s in range(L.batch)]

    def attend(self, selection):
        """selection[b][h] -> explicit-selection attention (absp_attend)."""
        L = self.layer
        stride = max(max(len(x) for s in selection for x in s), 1)
        b = np.zeros((L.batch, L.H, stride), np.uint32)
        c = np.zeros((L.batch, L.H), np.uint32)
        for s in range(L.batch):
            for h in range(L.H):
                b[s, h, :len(selection[s][h])] = selection[s][h]
                c[s, h] = len(selection[s][h])
        out = torch.empty(L.batch, L.H * L.G, L.d, dtype=torch.float32, device="cuda")
        self.da.attend(0, self.q, to_dev_u32(b), to_dev_u32(c), out)
        torch.cuda.synchronize()
        return out.cpu().numpy()

    def decode(self):
        L = self.layer
        out = torch.empty(L.batch, L.H * L.G, L.d, dtype=torch.float32, device="cuda")
        self.da.decode_step(0, self.q, out)
        torch.cuda.synchronize()
        self.step_selection = self.da.download_selection(0)
        return out.cpu().numpy()


def within_tol(got, want, atol=1e-3, rtol=1e-2):
    """The north-star tolerance: |got - want| <= 1e-3 + 1e-2 |want| elementwise."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return bool(np.all(np.abs(got - want) <= atol + rtol * np.abs(want))), float(np.abs(got - want).max())
