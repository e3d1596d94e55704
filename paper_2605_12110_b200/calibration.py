"""Calibration and trace replay over the C ABI.

Reference (/root/reference/proj):
  Trace, save_trace, load_trace             workload.hpp:36-75, workload.cpp:260-309
  RecallTable, CalibrationReport,           calibrator.hpp:15-44
  TransferReport
  attention_recall                          calibrator.cpp:48-71   -> DecodeAttention.attention_recall
  profile_sensitivity                       calibrator.cpp:73-114  -> GPU per sample (absp_profile_sample)
  assign_block_sizes                        calibrator.cpp:116-140
  normalized_recall, make_report            calibrator.cpp:142-157
  transfer_check                            calibrator.cpp:159-224 -> GPU per sample
  topk_page_recall(_per_head)               calibrator.cpp:226-249
  write_recall_csv, write_min_block_csv     calibrator.cpp:253-275

The heavy work of a sample (the dense fp64 oracle with weights, a store + selection
per candidate block size, the recall sums) runs in libabsp.so on the GPU; the loops
over samples, the averaging and the Eq.-2 assignment rule are host code, as in the
reference. Traces are fp32 on disk; the GPU stores them as bf16,
so parity with the reference is checked on bf16-representable traces.
"""
from __future__ import annotations

import ctypes as C
import struct
import sys
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, List, Sequence

import numpy as np

from . import _abi
from ._abi import InvalidArgument, check
from .absparse import BlockAssignment, EngineConfig

_MAGIC = b"ABSP"
_TRACE_VERSION = 1


# ---------------------------------------------------------------------------
# Trace I/O (workload.cpp:260-309)
# ---------------------------------------------------------------------------
@dataclass
class Trace:
    """One decode sample: keys / values [num_heads][seq_len][head_dim] and one query per
    head [num_heads][head_dim], fp32 (workload.hpp:36-48)."""
    num_heads: int = 0
    head_dim: int = 0
    seq_len: int = 0
    seed: int = 0
    keys: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    queries: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    version: int = _TRACE_VERSION

    def __eq__(self, other) -> bool:
        return (isinstance(other, Trace) and self.version == other.version
                and (self.num_heads, self.head_dim, self.seq_len, self.seed)
                == (other.num_heads, other.head_dim, other.seq_len, other.seed)
                and all(np.array_equal(np.asarray(a, np.float32).view(np.uint32).ravel(),
                                       np.asarray(b, np.float32).view(np.uint32).ravel())
                        for a, b in ((self.keys, other.keys), (self.values, other.values),
                                     (self.queries, other.queries))))


def save_trace(trace: Trace, path) -> None:
    """Binary trace, little-endian: magic "ABSP" | u32 version | u32 num_heads | u32 head_dim
    | u64 seq_len | u64 seed | keys | values | queries (bit-exact round trip)."""
    try:
        f = open(path, "wb")
    except OSError:
        raise RuntimeError(f"save_trace: cannot open {path}") from None
    with f:
        f.write(_MAGIC)
        f.write(struct.pack("<IIIQQ", trace.version, trace.num_heads, trace.head_dim, trace.seq_len, trace.seed))
        for a in (trace.keys, trace.values, trace.queries):
            f.write(np.ascontiguousarray(a, dtype="<f4").tobytes())


def load_trace(path) -> Trace:
    """load_trace with the reference's checks and messages (workload.cpp:277-309); raises
    RuntimeError (std::runtime_error) on a format problem."""
    try:
        data = Path(path).read_bytes()
    except OSError:
        raise RuntimeError(f"load_trace: cannot open {path}") from None
    pos = 0

    def take(n: int, what: str) -> bytes:
        nonlocal pos
        if pos + n > len(data):
            raise RuntimeError(f"load_trace: truncated file in section '{what}'")
        b = data[pos:pos + n]
        pos += n
        return b

    if take(4, "header") != _MAGIC:
        raise RuntimeError("load_trace: format error, bad magic bytes")
    (version,) = struct.unpack("<I", take(4, "header"))
    if version != _TRACE_VERSION:
        raise RuntimeError(f"load_trace: version mismatch (file {version}, expected {_TRACE_VERSION})")
    num_heads, head_dim = struct.unpack("<II", take(8, "header"))
    seq_len, seed = struct.unpack("<QQ", take(16, "header"))
    if num_heads == 0 or head_dim == 0 or seq_len == 0:
        raise RuntimeError("load_trace: dimension inconsistency in header")
    per = num_heads * seq_len * head_dim
    keys = np.frombuffer(take(per * 4, "keys"), "<f4").astype(np.float32)
    values = np.frombuffer(take(per * 4, "values"), "<f4").astype(np.float32)
    queries = np.frombuffer(take(num_heads * head_dim * 4, "queries"), "<f4").astype(np.float32)
    if pos != len(data):
        raise RuntimeError("load_trace: trailing bytes after queries section")
    return Trace(num_heads, head_dim, seq_len, seed, keys, values, queries, version)


# ---------------------------------------------------------------------------
# Calibration (calibrator.cpp)
# ---------------------------------------------------------------------------
@dataclass
class RecallTable:
    """Mean attention recall per (head, candidate block size) (calibrator.hpp:15-28)."""
    num_heads: int = 0
    candidates: List[int] = field(default_factory=list)
    recalls: np.ndarray = field(default_factory=lambda: np.zeros((0, 0)))  # [num_heads][candidates]
    sample_count: int = 0

    def at(self, head: int, ci: int) -> float:
        return float(self.recalls[head, ci])


@dataclass
class CalibrationReport:
    assignment: BlockAssignment
    normalized_recalls: RecallTable
    min_block_sizes: List[int]
    avg_block_size: float


@dataclass
class TransferReport:
    adaptive_recall: float = 0.0
    candidates: List[int] = field(default_factory=list)
    uniform_recalls: List[float] = field(default_factory=list)
    avg_block_size: float = 0.0
    matched_candidate: int = 0
    delta: float = 0.0


TraceProvider = Callable[[int], Trace]


def _check_trace_dims(trace: Trace, config: EngineConfig, index: int) -> None:
    if trace.num_heads != config.num_heads or trace.head_dim != config.head_dim:
        raise InvalidArgument(f"calibration sample {index}: trace dimensions do not match the config")


def profile_sample(trace: Trace, config: EngineConfig, assignment: BlockAssignment | None = None,
                   device: int = 0):
    """One trace on the GPU (absp_profile_sample): recall [num_heads][candidates] of the
    uniform assignments (and, with `assignment`, its per-head recall). Queries are one per
    KV head (num_q_heads = num_heads), as the reference's traces are."""
    H, d, n = trace.num_heads, trace.head_dim, trace.seq_len
    cfg = config.to_abi()
    cfg.num_q_heads = H
    keys = np.ascontiguousarray(trace.keys, np.float32).reshape(-1)
    values = np.ascontiguousarray(trace.values, np.float32).reshape(-1)
    queries = np.ascontiguousarray(trace.queries, np.float32).reshape(-1)
    if keys.size != H * n * d or values.size != H * n * d or queries.size != H * d:
        raise InvalidArgument("profile_sample: trace tensor sizes do not match its header")
    nc = len(config.candidate_block_sizes)
    rec = np.zeros((H, nc), np.float64)
    arec = np.zeros(H, np.float64)
    asg = None
    if assignment is not None:
        asg = (C.c_uint32 * H)(*assignment.block_sizes)
    check(_abi.load().absp_profile_sample(device, C.byref(cfg), keys.ctypes.data, values.ctypes.data,
                                          queries.ctypes.data, n, asg, rec.ctypes.data,
                                          arec.ctypes.data if asg is not None else None))
    return rec, (arec if asg is not None else None)


def profile_sensitivity(provider: TraceProvider, sample_count: int, config: EngineConfig,
                        device: int = 0) -> RecallTable:
    """profile_sensitivity (calibrator.cpp:73-114): per-head recall of every candidate block
    size at the configured budget and quantization, averaged over the usable samples
    (seq_len > token_budget)."""
    config.validate()
    if sample_count == 0:
        raise InvalidArgument("profile_sensitivity: need at least one calibration sample")
    table = RecallTable(config.num_heads, list(config.candidate_block_sizes),
                        np.zeros((config.num_heads, len(config.candidate_block_sizes))), 0)
    used = 0
    for i in range(sample_count):
        trace = provider(i)
        _check_trace_dims(trace, config, i)
        if trace.seq_len <= config.token_budget:
            print(f"profile_sensitivity: skipping sample {i} (seq_len {trace.seq_len} <= budget "
                  f"{config.token_budget}, recall is trivially 1)", file=sys.stderr)
            continue
        rec, _ = profile_sample(trace, config, device=device)
        table.recalls += rec
        used += 1
    if used == 0:
        raise RuntimeError("profile_sensitivity: no usable samples (every seq_len <= token_budget)")
    table.recalls /= float(used)
    table.sample_count = used
    return table


def assign_block_sizes(table: RecallTable, tau: float) -> BlockAssignment:
    """B_h* = max{B : Recall(h, B) >= tau * Recall(h, B_min)} (calibrator.cpp:116-140)."""
    if not table.candidates or table.num_heads == 0:
        raise InvalidArgument("assign_block_sizes: empty recall table")
    if list(table.candidates) != sorted(table.candidates):
        raise InvalidArgument("assign_block_sizes: candidates must be ascending")
    sizes = []
    for h in range(table.num_heads):
        peak = table.at(h, 0)
        if peak <= 0.0:
            raise InvalidArgument(f"assign_block_sizes: head {h} has zero recall at the minimum block size")
        best = table.candidates[0]
        for ci, b in enumerate(table.candidates):
            if table.at(h, ci) >= tau * peak:
                best = max(best, b)
        sizes.append(best)
    return BlockAssignment(sizes)


def normalized_recall(table: RecallTable) -> RecallTable:
    """Each row divided by its entry at the smallest candidate (calibrator.cpp:142-155)."""
    peaks = table.recalls[:, 0]
    if np.any(peaks <= 0.0):
        raise InvalidArgument("normalized_recall: zero recall at the minimum block size")
    return RecallTable(table.num_heads, list(table.candidates), table.recalls / peaks[:, None], table.sample_count)


def make_report(table: RecallTable, tau: float) -> CalibrationReport:
    a = assign_block_sizes(table, tau)
    return CalibrationReport(a, normalized_recall(table), list(a.block_sizes), a.average_block_size())


def transfer_check(assignment: BlockAssignment, holdout: TraceProvider, sample_count: int,
                   config: EngineConfig, device: int = 0) -> TransferReport:
    """Holdout recall of an assignment against the uniform baselines, and the delta to the
    uniform candidate nearest its average block size (ties go coarser) (calibrator.cpp:159-224)."""
    config.validate()
    assignment.validate(config)
    rep = TransferReport(candidates=list(config.candidate_block_sizes),
                         uniform_recalls=[0.0] * len(config.candidate_block_sizes),
                         avg_block_size=assignment.average_block_size())
    H = config.num_heads
    used = 0
    for i in range(sample_count):
        trace = holdout(i)
        _check_trace_dims(trace, config, i)
        if trace.seq_len <= config.token_budget:
            print(f"transfer_check: skipping sample {i} (seq_len <= budget)", file=sys.stderr)
            continue
        rec, arec = profile_sample(trace, config, assignment, device)
        for r in arec:
            rep.adaptive_recall += float(r) / H
        for ci in range(len(rep.candidates)):
            for h in range(H):
                rep.uniform_recalls[ci] += float(rec[h, ci]) / H
        used += 1
    if used == 0:
        raise RuntimeError("transfer_check: no usable holdout samples")
    rep.adaptive_recall /= used
    rep.uniform_recalls = [r / used for r in rep.uniform_recalls]
    best_ci = 0
    best_gap = abs(float(rep.candidates[0]) - rep.avg_block_size)
    for ci in range(1, len(rep.candidates)):
        gap = abs(float(rep.candidates[ci]) - rep.avg_block_size)
        if gap <= best_gap:
            best_gap, best_ci = gap, ci
    rep.matched_candidate = rep.candidates[best_ci]
    rep.delta = rep.adaptive_recall - rep.uniform_recalls[best_ci]
    return rep


def topk_page_recall_per_head(selected: Sequence[Sequence[int]], reference: Sequence[Sequence[int]]) -> List[float]:
    """|selected ∩ reference| / |reference| per head (calibrator.cpp:226-243)."""
    if len(selected) != len(reference):
        raise InvalidArgument("topk_page_recall: head count mismatch")
    out = []
    for sel, ref in zip(selected, reference):
        r = set(int(x) for x in ref)
        if not r:
            raise InvalidArgument("topk_page_recall: empty reference selection")
        out.append(sum(1 for b in sel if int(b) in r) / len(r))
    return out


def topk_page_recall(selected, reference) -> float:
    per = topk_page_recall_per_head(selected, reference)
    return float(sum(per) / len(per)) if per else 0.0


def _fmt10g(v: float) -> str:
    """printf("%.10g") as the reference's format_double (calibrator.cpp:39-43)."""
    return "%.10g" % v


def write_recall_csv(path, table: RecallTable, layer_tag: str) -> None:
    """CSV head,layer,block_size,recall (calibrator.cpp:253-264)."""
    try:
        f = open(path, "w")
    except OSError:
        raise RuntimeError(f"write_recall_csv: cannot open {path}") from None
    with f:
        f.write("head,layer,block_size,recall\n")
        for h in range(table.num_heads):
            for ci, b in enumerate(table.candidates):
                f.write(f"{h},{layer_tag},{b},{_fmt10g(table.at(h, ci))}\n")


def write_min_block_csv(path, min_block_sizes: Sequence[int], layer_tag: str) -> None:
    """CSV head,layer,min_block_size (calibrator.cpp:266-275)."""
    try:
        f = open(path, "w")
    except OSError:
        raise RuntimeError(f"write_min_block_csv: cannot open {path}") from None
    with f:
        f.write("head,layer,min_block_size\n")
        for h, b in enumerate(min_block_sizes):
            f.write(f"{h},{layer_tag},{b}\n")
