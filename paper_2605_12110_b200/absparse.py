"""Host-side mirror of the reference's operator API for the decode path, over the C ABI.

Reference (namespace absparse, /root/reference/proj/include/absparse):
  EngineConfig / QuantSpec / CentroidMethod      config.hpp:11-52
  BlockAssignment                                centroids.hpp:12-23
  compute_block_centroids + quantize_store       centroids.hpp:56-57, quantizer.hpp:43
      -> DecodeAttention.build_store
  estimate_scores + select_topk                  engine.hpp:47-68
      -> DecodeAttention.select
  populate_page_spans + sparse_attention         engine.hpp:71-82
      -> DecodeAttention.attend
  DecodeEngine::step (estimate->select->attend)  engine.cpp:450-461
      -> DecodeAttention.decode_step

Everything numeric runs in libabsp.so on the GPU. Device buffers are passed as
torch CUDA tensors (or raw integer pointers); PyTorch is plumbing only.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional, Sequence

import numpy as np

from . import _abi
from ._abi import (AbspError, CapacityError, CudaError, InvalidArgument, LogicError,  # noqa: F401
                   OutOfRange, check)


class CentroidMethod(IntEnum):
    MEAN = 0     # CentroidMethod::kMean
    MAXMIN = 1   # CentroidMethod::kMaxMin


class QuantMode(IntEnum):
    SYMMETRIC = 0
    ASYMMETRIC = 1


@dataclass(frozen=True)
class QuantSpec:
    """QuantSpec (config.hpp:17-26)."""
    bits: int = 4
    mode: QuantMode = QuantMode.ASYMMETRIC

    def levels(self) -> int:
        return (1 << self.bits) - 1

    def sym_mid(self) -> int:
        return (1 << (self.bits - 1)) - 1

    def validate(self) -> None:
        if self.bits not in (2, 4, 8):
            raise InvalidArgument("quant bits must be one of {2, 4, 8}")

    @property
    def name(self) -> str:  # quant_spec_name, config.cpp:14-17
        return f"int{self.bits}x{'sym' if self.mode == QuantMode.SYMMETRIC else 'asym'}"

    @staticmethod
    def parse(name: str) -> "QuantSpec":  # parse_quant_spec, config.cpp:19-28
        for bits in (2, 4, 8):
            for mode in (QuantMode.SYMMETRIC, QuantMode.ASYMMETRIC):
                s = QuantSpec(bits, mode)
                if s.name == name:
                    return s
        raise InvalidArgument(f"unknown quant spec '{name}' (expected int{{2,4,8}}x{{sym,asym}} or none)")


@dataclass
class EngineConfig:
    """EngineConfig (config.hpp:36-52) + batch/GQA/capacity extensions."""
    num_heads: int = 8                       # KV heads
    head_dim: int = 64
    page_size: int = 16
    candidate_block_sizes: Sequence[int] = (16, 32, 64)
    token_budget: int = 4096
    recall_threshold: float = 0.98           # calibration only (out of scope here)
    centroid_method: CentroidMethod = CentroidMethod.MEAN
    quant: Optional[QuantSpec] = None        # None = full-precision store
    # extensions
    num_q_heads: Optional[int] = None        # GQA: defaults to num_heads (MHA)
    max_batch: int = 1
    max_seq_len: int = 131072
    num_layers: int = 1

    def min_candidate(self) -> int:
        return min(self.candidate_block_sizes)

    def max_candidate(self) -> int:
        return max(self.candidate_block_sizes)

    @property
    def group_size(self) -> int:
        return (self.num_q_heads or self.num_heads) // self.num_heads

    def to_abi(self) -> _abi.Config:
        c = _abi.Config()
        c.num_kv_heads = self.num_heads
        c.num_q_heads = self.num_q_heads or self.num_heads
        c.head_dim = self.head_dim
        c.page_size = self.page_size
        cands = list(self.candidate_block_sizes)
        if len(cands) > _abi.ABSP_MAX_CANDIDATES:
            raise InvalidArgument("too many candidate block sizes")
        c.num_candidates = len(cands)
        for i, b in enumerate(cands):
            c.candidate_block_sizes[i] = int(b)
        c.token_budget = self.token_budget
        c.centroid_method = int(self.centroid_method)
        c.quant_bits = self.quant.bits if self.quant else 0
        c.quant_mode = int(self.quant.mode) if self.quant else int(QuantMode.ASYMMETRIC)
        c.max_batch = self.max_batch
        c.max_seq_len = self.max_seq_len
        c.num_layers = self.num_layers
        return c

    def validate(self) -> None:
        """EngineConfig::validate (config.cpp:48-78) via absp_config_validate."""
        if self.recall_threshold <= 0.0:
            raise InvalidArgument("recall_threshold must be positive")
        if self.quant is not None:
            self.quant.validate()
        check(_abi.load().absp_config_validate(C.byref(self.to_abi())))


@dataclass
class BlockAssignment:
    """Per-KV-head block sizes B_h (centroids.hpp:12-23)."""
    block_sizes: list = field(default_factory=list)

    @staticmethod
    def uniform(num_heads: int, block_size: int) -> "BlockAssignment":
        return BlockAssignment([block_size] * num_heads)

    @staticmethod
    def cycled(num_heads: int, candidates: Sequence[int]) -> "BlockAssignment":
        """Heads cycle through the candidates, as cmd_bench does (cli_commands.cpp:445-451)."""
        return BlockAssignment([candidates[h % len(candidates)] for h in range(num_heads)])

    @staticmethod
    def load(path) -> "BlockAssignment":
        """read_assignment_file (calibrator.cpp:285-311): one 'head block_size' pair per
        line, consecutive heads from 0, empty lines skipped; RuntimeError (the
        reference's std::runtime_error) on anything else."""
        try:
            lines = open(path).read().split("\n")
        except OSError:
            raise RuntimeError(f"read_assignment_file: cannot open {path}") from None
        sizes = []
        for line in lines:
            if line == "":
                continue
            parts = line.split()
            ok = len(parts) >= 2 and parts[0].isdigit() and parts[1].isdigit() and int(parts[0]) == len(sizes)
            if not ok:
                raise RuntimeError(f"read_assignment_file: malformed line '{line}' "
                                   "(expected 'head block_size' with consecutive heads)")
            if len(parts) > 2:
                raise RuntimeError(f"read_assignment_file: trailing tokens on line '{line}'")
            sizes.append(int(parts[1]))
        if not sizes:
            raise RuntimeError(f"read_assignment_file: empty file {path}")
        return BlockAssignment(sizes)

    def save(self, path) -> None:
        """write_assignment_file (calibrator.cpp:277-283)."""
        with open(path, "w") as f:
            for h, b in enumerate(self.block_sizes):
                f.write(f"{h} {b}\n")

    def num_heads(self) -> int:
        return len(self.block_sizes)

    def average_block_size(self) -> float:
        return float(np.mean(self.block_sizes)) if self.block_sizes else 0.0

    def validate(self, config: EngineConfig) -> None:
        """BlockAssignment::validate (centroids.cpp:59-76)."""
        if len(self.block_sizes) != config.num_heads:
            raise InvalidArgument(f"assignment covers {len(self.block_sizes)} heads, config has "
                                  f"{config.num_heads}")
        for h, b in enumerate(self.block_sizes):
            if b not in config.candidate_block_sizes:
                raise InvalidArgument(f"head {h}: block size {b} is not a candidate")
            if b % config.page_size:
                raise InvalidArgument(f"head {h}: block size {b} is not a multiple of page_size")


def build_offsets(seq_len: int, assignment: BlockAssignment) -> list:
    """offsets[h+1] = offsets[h] + ceil(seq_len / B_h) (centroids.cpp:78-84)."""
    out = [0]
    for b in assignment.block_sizes:
        out.append(out[-1] + (seq_len + b - 1) // b)
    return out


def _ptr(x) -> Optional[int]:
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    raise TypeError(f"cannot take a device pointer of {type(x)}")


def _stream(stream) -> Optional[int]:
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


class DecodeAttention:
    """One absp context: per-layer stores over borrowed paged KV caches on one GPU."""

    def __init__(self, config: EngineConfig, device: int = 0):
        self.config = config
        self.device = device
        self._lib = _abi.load()
        self._ctx = C.c_void_p()
        if config.quant is not None:
            config.quant.validate()
        check(self._lib.absp_ctx_create(device, C.byref(config.to_abi()), C.byref(self._ctx)))
        self._seq_lens = {}

    def close(self) -> None:
        if self._ctx:
            self._lib.absp_ctx_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- setup ---------------------------------------------------------------
    def set_assignment(self, layer: int, assignment: BlockAssignment) -> None:
        if len(assignment.block_sizes) != self.config.num_heads:
            raise InvalidArgument(f"assignment covers {len(assignment.block_sizes)} heads, config has "
                                  f"{self.config.num_heads}")
        arr = (C.c_uint32 * len(assignment.block_sizes))(*assignment.block_sizes)
        check(self._lib.absp_set_assignment(self._ctx, layer, arr))

    def bind(self, layer: int, k_pool, v_pool, page_table, seq_lens: Sequence[int]) -> None:
        """k_pool/v_pool: bf16 [H][pool_pages][P][d] device tensors; page_table: uint32/int32
        [batch][max_pages] device tensor; seq_lens: host ints."""
        pool_pages = int(k_pool.shape[1])
        max_pages = int(page_table.shape[1])
        lens = (C.c_uint32 * len(seq_lens))(*[int(s) for s in seq_lens])
        check(self._lib.absp_kv_bind(self._ctx, layer, _ptr(k_pool), _ptr(v_pool), pool_pages,
                                     _ptr(page_table), max_pages, lens, len(seq_lens)))
        self._seq_lens[layer] = list(seq_lens)

    def build_store(self, layer: int, stream=None) -> None:
        check(self._lib.absp_build_store(self._ctx, layer, _stream(stream)))

    def append(self, layer: int, k_new, v_new, stream=None) -> None:
        """One token per sequence (bf16 [batch][H][d] device tensors) + store maintenance:
        PagedKVCache::append + refresh_tail_centroids + requantize_heads (engine.cpp:443-449)."""
        check(self._lib.absp_append(self._ctx, layer, _ptr(k_new), _ptr(v_new), _stream(stream)))
        self._seq_lens[layer] = [n + 1 for n in self._seq_lens[layer]]

    # -- hot path --------------------------------------------------------------
    def select(self, layer: int, q, blocks, counts, stream=None) -> None:
        stride = int(blocks.shape[-1])
        check(self._lib.absp_select(self._ctx, layer, _ptr(q), _ptr(blocks), stride, _ptr(counts),
                                    _stream(stream)))

    def attend(self, layer: int, q, blocks, counts, out, stream=None, validate: bool = True) -> None:
        """sparse_attention over an explicit selection. validate=True (the reference's
        semantics) synchronises and raises InvalidArgument / OutOfRange for an empty
        selection, a count above the stride, a block id or a page id out of range."""
        stride = int(blocks.shape[-1])
        check(self._lib.absp_attend(self._ctx, layer, _ptr(q), _ptr(blocks), stride, _ptr(counts),
                                    _ptr(out), _stream(stream)))
        if validate:
            check(self._lib.absp_attend_validate(self._ctx, layer, _stream(stream)))

    def layout_version(self, layer: int) -> int:
        """Changes when an append alters a kernel argument of decode_step (absp_layout_version)."""
        return int(self._lib.absp_layout_version(self._ctx, layer))

    def attend_selected(self, layer: int, q, out, stream=None) -> None:
        """Attention over the layer's most recent selection (second half of decode_step)."""
        check(self._lib.absp_attend_selected(self._ctx, layer, _ptr(q), _ptr(out), _stream(stream)))

    def select_step(self, layer: int, q, stream=None) -> None:
        """The decode step's selection alone (layer-owned buffers; then attend_selected)."""
        check(self._lib.absp_select_step(self._ctx, layer, _ptr(q), _stream(stream)))

    def decode_step(self, layer: int, q, out, stream=None) -> None:
        check(self._lib.absp_decode_step(self._ctx, layer, _ptr(q), _ptr(out), _stream(stream)))

    def decode_step_host(self, layer: int, q_host, out_host, stream=None) -> None:
        check(self._lib.absp_decode_step_host(self._ctx, layer, _ptr(q_host), _ptr(out_host),
                                              _stream(stream)))

    def full_attention(self, layer: int, q, out, weights=None, stream=None) -> None:
        """full_attention_oracle (engine.cpp:357-403) over each sequence's whole context:
        out fp32 [batch][Hq][d]; weights (optional) fp64 [batch][Hq][stride], stride >= the
        longest sequence, receives the softmax weights of every cached token."""
        stride = int(weights.shape[-1]) if weights is not None else 0
        check(self._lib.absp_full_attention(self._ctx, layer, _ptr(q), _ptr(out), _ptr(weights), stride,
                                            _stream(stream)))

    def attention_recall(self, layer: int, weights, blocks, counts, recall, stream=None) -> None:
        """attention_recall (calibrator.cpp:48-71): recall fp64 [batch][Hq] = the weight mass on
        tokens inside the selected blocks (blocks / counts as select() writes them)."""
        check(self._lib.absp_attention_recall(self._ctx, layer, _ptr(weights), int(weights.shape[-1]),
                                              _ptr(blocks), int(blocks.shape[-1]), _ptr(counts), _ptr(recall),
                                              _stream(stream)))

    # -- introspection ---------------------------------------------------------
    def layer_info(self, layer: int) -> _abi.LayerInfo:
        info = _abi.LayerInfo()
        check(self._lib.absp_get_layer_info(self._ctx, layer, C.byref(info)))
        return info

    def last_selection(self, layer: int):
        """(blocks_ptr, stride, counts_ptr) of the last decode_step."""
        b, c = C.c_void_p(), C.c_void_p()
        s = C.c_uint32()
        check(self._lib.absp_last_selection(self._ctx, layer, C.byref(b), C.byref(s), C.byref(c)))
        return b.value, s.value, c.value

    def download_selection(self, layer: int) -> list:
        """The layer's last selection (decode_step or select) as [batch][kv head] arrays of
        block ids, score-descending (SelectionResult::blocks, engine.hpp:19-26)."""
        _, stride, _ = self.last_selection(layer)
        batch = len(self._seq_lens[layer])
        H = self.config.num_heads
        blocks = np.zeros((batch, H, stride), np.uint32)
        counts = np.zeros((batch, H), np.uint32)
        check(self._lib.absp_download_selection(self._ctx, layer, blocks.ctypes.data, counts.ctypes.data))
        return [[blocks[b, h, :counts[b, h]].copy() for h in range(H)] for b in range(batch)]

    def set_filter_diagnostics(self, layer: int, enable: bool = True) -> None:
        """Decode steps also store the fused selection's approximate scores and bounds."""
        check(self._lib.absp_set_filter_diagnostics(self._ctx, layer, int(enable)))

    def download_filter_scores(self, layer: int, seq: int):
        """(approximate scores [total], per-KV-head error bounds [H]) of the decode step's
        selection filter for one sequence (diagnostics)."""
        offsets = np.zeros(self.config.num_heads + 1, np.uint64)
        check(self._lib.absp_download_store(self._ctx, layer, seq, offsets.ctypes.data,
                                            None, None, None, None, None, None, None, None))
        approx = np.zeros(int(offsets[-1]), np.float32)
        err = np.zeros(self.config.num_heads, np.float32)
        check(self._lib.absp_download_filter_scores(self._ctx, layer, seq, approx.ctypes.data, err.ctypes.data))
        return approx, err

    def launch_count(self) -> int:
        return int(self._lib.absp_launch_count(self._ctx))

    def download_store(self, layer: int, seq: int) -> dict:
        """The store of one sequence in the reference layouts (CentroidStore /
        QuantizedCentroidStore): offsets, values(_min), codes(_min), scales(_min), zps(_min)."""
        cfg = self.config
        H, d = cfg.num_heads, cfg.head_dim
        offsets = np.zeros(H + 1, np.uint64)
        check(self._lib.absp_download_store(self._ctx, layer, seq, offsets.ctypes.data,
                                            None, None, None, None, None, None, None, None))
        total = int(offsets[-1])
        mm = cfg.centroid_method == CentroidMethod.MAXMIN
        out = {"offsets": offsets, "values": np.zeros((total, d), np.float32)}
        if mm:
            out["values_min"] = np.zeros((total, d), np.float32)
        if cfg.quant is not None:
            out["codes"] = np.zeros((total, d), np.uint8)
            out["scales"] = np.zeros((H, d), np.float32)
            out["zps"] = np.zeros((H, d), np.float32)
            if mm:
                out["codes_min"] = np.zeros((total, d), np.uint8)
                out["scales_min"] = np.zeros((H, d), np.float32)
                out["zps_min"] = np.zeros((H, d), np.float32)
        p = lambda k: out[k].ctypes.data if k in out else None
        check(self._lib.absp_download_store(self._ctx, layer, seq, None, p("values"), p("values_min"),
                                            p("codes"), p("codes_min"), p("scales"), p("zps"),
                                            p("scales_min"), p("zps_min")))
        return out

    def download_scores(self, layer: int, seq: int) -> np.ndarray:
        """Scores of the last select/decode_step for one sequence, flattened like
        estimate_scores' output (engine.hpp:47-49)."""
        offsets = np.zeros(self.config.num_heads + 1, np.uint64)
        check(self._lib.absp_download_store(self._ctx, layer, seq, offsets.ctypes.data,
                                            None, None, None, None, None, None, None, None))
        out = np.zeros(int(offsets[-1]), np.float32)
        check(self._lib.absp_download_scores(self._ctx, layer, seq, out.ctypes.data))
        return out


def fill_synthetic_bf16(dst, seed: int, stream_id: int, stream=None) -> None:
    """Deterministic N(0,1)-like bf16 fill on the device (same bytes as oracle/synth.py)."""
    check(_abi.load().absp_fill_synthetic_bf16(_ptr(dst), int(dst.numel()), seed, stream_id,
                                               _stream(stream)))


def _to_bf16_bits(x) -> np.ndarray:
    """fp32 -> bf16 bit patterns, round to nearest even (values already in bf16 stay exact)."""
    u = np.ascontiguousarray(np.asarray(x, np.float32)).view(np.uint32).astype(np.uint64)
    u = u + 0x7FFF + ((u >> 16) & 1)
    return (u >> 16).astype(np.uint16)


@dataclass
class StepResult:
    """StepResult (engine.hpp:84-88): output [Hq][d] fp32, selection[h] (ordered block ids)."""
    output: np.ndarray
    selection: list
    full_attention_fallback: bool


class DecodeEngine:
    """DecodeEngine (engine.hpp:90-129, engine.cpp:405-463) on the GPU for one sequence,
    over the library's engine object (absp_engine_*, no PyTorch): it owns the paged bf16
    KV cache (per-head pools, page ids handed out sequentially as kv_cache.cpp:53-60
    does), the quantized store and a stream. step = append + refresh_tail_centroids +
    requantize_heads + estimate -> select -> attend. With seq_len <= token_budget every
    block is selected, so the sparse output is the full attention the reference falls
    back to (engine.cpp:456-458). Inputs are fp32 and stored as bf16."""

    def __init__(self, config: EngineConfig, assignment: BlockAssignment, capacity_tokens: int, device: int = 0):
        assignment.validate(config)
        if config.quant is not None:
            config.quant.validate()
        cfg = EngineConfig(**{**config.__dict__, "max_batch": 1, "max_seq_len": int(capacity_tokens),
                              "num_layers": 1})
        self.config = cfg
        self.assignment = assignment
        self._lib = _abi.load()
        self._eng = C.c_void_p()
        bs = (C.c_uint32 * len(assignment.block_sizes))(*assignment.block_sizes)
        check(self._lib.absp_engine_create(device, C.byref(cfg.to_abi()), bs, int(capacity_tokens),
                                           C.byref(self._eng)))
        ctx, stride = C.c_void_p(), C.c_uint32()
        check(self._lib.absp_engine_info(self._eng, None, C.byref(stride), C.byref(ctx)))
        self._stride = stride.value
        # the engine's context, for store / selection read-back (owned by the engine)
        self.da = DecodeAttention.__new__(DecodeAttention)
        self.da.config, self.da.device, self.da._lib, self.da._ctx = cfg, device, self._lib, ctx
        self.da._seq_lens = {0: [0]}
        self.da.close = lambda: None

    def close(self) -> None:
        if self._eng:
            self._lib.absp_engine_destroy(self._eng)
            self._eng = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def seq_len(self) -> int:
        n = C.c_uint64()
        check(self._lib.absp_engine_info(self._eng, C.byref(n), None, None))
        return int(n.value)

    def prefill(self, keys, values, num_tokens: int) -> None:
        """keys / values: head-major [H][tokens][d] fp32 (engine.hpp:102-105)."""
        k = np.ascontiguousarray(keys, np.float32)
        v = np.ascontiguousarray(values, np.float32)
        check(self._lib.absp_engine_prefill(self._eng, k.ctypes.data, k.size, v.ctypes.data, v.size,
                                            int(num_tokens)))
        self.da._seq_lens[0] = [self.seq_len]

    def step(self, keys, values, query) -> StepResult:
        """keys / values: [H][d] fp32 of the new token; query: [Hq][d] fp32."""
        H, d = self.config.num_heads, self.config.head_dim
        Hq = self.config.num_q_heads or H
        k = np.ascontiguousarray(keys, np.float32)
        v = np.ascontiguousarray(values, np.float32)
        q = np.ascontiguousarray(query, np.float32)
        out = np.zeros((Hq, d), np.float32)
        blocks = np.zeros((H, self._stride), np.uint32)
        counts = np.zeros(H, np.uint32)
        fb = C.c_int()
        check(self._lib.absp_engine_step(self._eng, k.ctypes.data, k.size, v.ctypes.data, v.size, q.ctypes.data,
                                         q.size, out.ctypes.data, blocks.ctypes.data, self._stride,
                                         counts.ctypes.data, C.byref(fb)))
        self.da._seq_lens[0] = [self.seq_len]
        return StepResult(out, [blocks[h, :counts[h]].copy() for h in range(H)], bool(fb.value))

    def centroids(self) -> dict:
        """CentroidStore (+ QuantizedCentroidStore) of the sequence, reference layouts."""
        return self.da.download_store(0, 0)

    def quantized(self):
        return self.da.download_store(0, 0) if self.config.quant is not None else None
