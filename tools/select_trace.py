"""Fused-selection timeline (debug): one decode step of a layer with lib/libabsp_trace.so
after an L2 flush; per-CTA globaltimer stamps of k_select's phases (select.cu SEL_TRACE)
and the attention CTAs' first data / end (attend.cu). Tooling, not product.
usage: python tools/select_trace.py [workload] [batch]"""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_12110_b200 import _abi  # noqa: E402

_abi._lib = _abi.load(ROOT / "paper_2605_12110_b200" / "lib" / "libabsp_trace.so")
for f in ("absp_debug_select_trace", "absp_debug_attn_trace"):
    getattr(_abi._lib, f).argtypes = [C.c_void_p, C.c_size_t]
from bench import SEED, WORKLOADS  # noqa: E402
from paper_2605_12110_b200 import (BlockAssignment, DecodeAttention, EngineConfig, QuantSpec,  # noqa: E402
                                   fill_synthetic_bf16)

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
B = int(sys.argv[2]) if len(sys.argv) > 2 else w["batch"]
n, H, G, d, P, T = w["n"], w["H"], w["G"], w["d"], w["P"], w["T"]
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
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    for _ in range(3):
        da.decode_step(0, q, out, stream)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        da.decode_step(0, q, out, stream)
flush = torch.empty(1 << 28, dtype=torch.int8, device="cuda")
names = ["start", "wait done", "fin: loaded", "params", "weights", "filter done", "keys out", "arrived",
         "fin: cands", "fin: scored", "fin: ranked", "fin: hist", "published", "fin: thr"]
pct = lambda a: " ".join(f"{x:7.2f}" for x in np.percentile(a, [0, 10, 50, 90, 100]))
import os
warm = os.environ.get("SEL_TRACE_WARM") == "1"  # no L2 flush: the previous replay's code and data stay
for rep in range(2):
    if not warm:
        flush.fill_(rep)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    st = np.zeros((4096, 24), np.uint64)
    at = np.zeros((160, 256), np.uint64)
    _abi.check(_abi._lib.absp_debug_select_trace(st.ctypes.data, st.nbytes))
    _abi.check(_abi._lib.absp_debug_attn_trace(at.ctypes.data, at.nbytes))
    ncta = int((st[:, 0] > 0).sum())
    st = st[:ncta]
    t0 = st[:, 0].min()
    print(f"rep {rep}{' (warm)' if warm else ''}: {ncta} select CTAs (us from the first start; pctl 0/10/50/90/100)")
    for i in (0, 1, 3, 4, 5, 6, 7, 2, 11, 13, 8, 9, 10, 12):
        nm = names[i]
        col = st[:, i]
        col = col[col >= t0]  # stale stamps of earlier steps are older than this step's start
        if len(col):
            print(f"  {nm:14s} {pct((col.astype(np.float64) - t0) / 1e3)}  (n={len(col)})")
    fin = st[st[:, 12] >= t0]
    if len(fin):
        print("  candidates/unit", pct(fin[:, 14].astype(np.float64)))
    a0 = at[:, 0]
    live = a0 > 0
    if live.any():
        print(f"  attn CTA start {pct((at[live, 0].astype(np.float64) - t0) / 1e3)}")
        fd = at[live, 64]
        print(f"  attn 1st data  {pct((fd[fd > 0].astype(np.float64) - t0) / 1e3)}")
        ends = at[live][:, 242:250].max(1)
        print(f"  attn end       {pct((ends.astype(np.float64) - t0) / 1e3)}")
    if os.environ.get("SEL_TRACE_UNITS") == "1" and len(fin):
        # per finalizing CTA: candidates and the durations of its finalize phases (us)
        ph = [(7, "arrived"), (2, "loaded"), (11, "hist"), (13, "thr"), (8, "cands"), (9, "scored"),
              (16, "s:zeroed"), (17, "s:smem"), (18, "s:end"), (15, "sorted"), (10, "ranked"), (12, "published")]
        rows = []
        for r in fin:
            ts = [(nm, int(r[i])) for i, nm in ph if int(r[i]) >= t0]
            d = {f"{a[0]}->{b[0]}": (b[1] - a[1]) / 1e3 for a, b in zip(ts, ts[1:])}
            rows.append((int(r[14]), d))
        rows.sort(key=lambda x: x[0])
        for n_c, d in rows[:: max(1, len(rows) // 24)]:
            print(f"    n={n_c:5d} " + " ".join(f"{k}={v:.2f}" for k, v in d.items()))
