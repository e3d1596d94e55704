"""Attention timeline (debug): run cfg-3 decode steps with lib/libabsp_trace.so and
summarise per-CTA globaltimer stamps: first-data latency, chunk inter-arrival,
producer lead, flush and merge durations, tail. Tooling, not product."""
import ctypes as C
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_12110_b200 import _abi  # noqa: E402

import os  # noqa: E402
_abi._lib = _abi.load(ROOT / "paper_2605_12110_b200" / "lib" / os.environ.get("ATTN_TRACE_LIB", "libabsp_trace.so"))
_abi._lib.absp_debug_attn_trace.argtypes = [C.c_void_p, C.c_size_t]
from bench import SEED, WORKLOADS  # noqa: E402
from paper_2605_12110_b200 import (BlockAssignment, DecodeAttention, EngineConfig, QuantSpec,  # noqa: E402
                                   fill_synthetic_bf16)

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
B, n, H, G, d, P, T = w["batch"], w["n"], w["H"], w["G"], w["d"], w["P"], w["T"]
pages = B * ((n + P - 1) // P)
cfg = EngineConfig(num_heads=H, head_dim=d, page_size=P, candidate_block_sizes=tuple(w["cands"]), token_budget=T,
                   quant=QuantSpec(4), num_q_heads=H * G, max_batch=B, max_seq_len=n)
da = DecodeAttention(cfg)
da.set_assignment(0, BlockAssignment.cycled(H, w["cands"]))
k = torch.empty(H, pages, P, d, dtype=torch.int16, device="cuda")
v = torch.empty_like(k)
q = torch.empty(B, H * G, d, dtype=torch.int16, device="cuda")
for t, s in ((k, 0), (v, 1), (q, 2)):
    fill_synthetic_bf16(t, SEED, s)
pt = torch.arange(pages, dtype=torch.int32, device="cuda").reshape(B, -1)
da.bind(0, k, v, pt, [n] * B)
da.build_store(0)
out = torch.empty(B, H * G, d, dtype=torch.float32, device="cuda")
for _ in range(3):
    da.decode_step(0, q, out)
torch.cuda.synchronize()
flush = torch.empty(1 << 28, dtype=torch.int8, device="cuda")
flush.fill_(1)  # evict L2
da.attend_selected(0, q, out)
torch.cuda.synchronize()
tr = np.zeros((160, 256), np.uint64)
_abi.check(_abi._lib.absp_debug_attn_trace(tr.ctypes.data, tr.nbytes))
t0 = min(int(x) for x in tr[:148, 0] if x)
rel = lambda x: (int(x) - t0) / 1000.0 if x else float("nan")
firsts, gaps, leads, flushes, tails, ends, chunks = [], [], [], [], [], [], []
fin_flush, fin_merge, npends = [], [], []
for c in range(148):
    row = tr[c]
    arr = [rel(row[64 + i]) for i in range(64) if row[64 + i]]
    iss = [rel(row[1 + i]) for i in range(63) if row[1 + i]]
    chunks.append(len(arr))
    if arr:
        firsts.append(arr[0] - rel(row[0]))
        gaps += list(np.diff(arr))
    for i in range(min(len(arr), len(iss))):
        leads.append(arr[i] - iss[i])
    for j in range(4):
        if row[192 + 2 * j] and row[193 + 2 * j]:
            flushes.append(rel(row[193 + 2 * j]) - rel(row[192 + 2 * j]))
    ends.append(max(rel(x) for x in row[242:250] if x))
    if row[240]:
        tails.append(ends[-1] - rel(row[240]))
    npends.append(int(row[250]))
    if row[240] and row[241]:
        fin_flush.append(rel(row[241]) - rel(row[240]))
        fin_merge.append(ends[-1] - rel(row[241]))
pct = lambda a: f"median {statistics.median(a):6.2f}  p90 {np.percentile(a, 90):6.2f}  max {max(a):6.2f}" if a else "-"
print(f"CTAs 148, chunks/CTA median {statistics.median(chunks)}")
print(f"kernel span (first start -> last end)  {max(ends):.2f} us")
print(f"CTA start offset                       {pct([rel(tr[c, 0]) for c in range(148)])}")
print(f"first data after CTA start (us)        {pct(firsts)}")
print(f"chunk inter-arrival at warp 0 (us)     {pct(gaps)}")
print(f"issue -> data arrival (us)             {pct(leads)}")
print(f"flush duration (us)                    {pct(flushes)}")
print(f"final flush + merges (us)              {pct(tails)}")
print(f"  final flush (us)                     {pct(fin_flush)}")
print(f"  pending merges (us)                  {pct(fin_merge)}  (units merged at the end per CTA: {pct(npends)})")
print(f"CTA end (us)                           {pct(ends)}")

# ---- in-step timeline: flush L2, then a full decode step (top-k -> attention) ----
flush.fill_(2)
torch.cuda.synchronize()
da.decode_step(0, q, out)
torch.cuda.synchronize()
_abi.check(_abi._lib.absp_debug_attn_trace(tr.ctypes.data, tr.nbytes))
t0 = min(int(x) for x in tr[:148, 0] if x)
firsts, gaps, ends, tails = [], [], [], []
for c in range(148):
    row = tr[c]
    arr = [rel(row[64 + i]) for i in range(64) if row[64 + i]]
    if arr:
        firsts.append(arr[0] - rel(row[0]))
        gaps += list(np.diff(arr))
    ends.append(max(rel(x) for x in row[242:250] if x))
    if row[240]:
        tails.append(ends[-1] - rel(row[240]))
print("--- inside decode_step (page lists hot in L2) ---")
print(f"kernel span                            {max(ends):.2f} us")
print(f"first data after CTA start (us)        {pct(firsts)}")
print(f"chunk inter-arrival at warp 0 (us)     {pct(gaps)}")
print(f"final flush + merges (us)              {pct(tails)}")
