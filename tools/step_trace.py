"""Whole decode-step timeline (debug): one cfg-3 decode step with lib/libabsp_trace.so after
an L2 flush; scorer, top-k and attention per-CTA globaltimer stamps on one time base.
Tooling, not product."""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_12110_b200 import _abi  # noqa: E402

_abi._lib = _abi.load(ROOT / "paper_2605_12110_b200" / "lib" / "libabsp_trace.so")
for f in ("absp_debug_score_trace", "absp_debug_topk_trace", "absp_debug_attn_trace"):
    getattr(_abi._lib, f).argtypes = [C.c_void_p, C.c_size_t]
_abi._lib.absp_debug_refine_trace.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t]
import os  # noqa: E402
FAST = os.environ.get("ABSP_FAST_SELECT", "") == "1"
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
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    for _ in range(3):
        da.decode_step(0, q, out, stream)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        da.decode_step(0, q, out, stream)
flush = torch.empty(1 << 28, dtype=torch.int8, device="cuda")
pct = lambda a: " ".join(f"{x:7.2f}" for x in np.percentile(a, [0, 10, 50, 90, 100]))
for rep in range(2):
    flush.fill_(rep)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    sc = np.zeros((320, 16), np.uint64)
    tk = np.zeros((1024, 8), np.uint64)
    at = np.zeros((160, 256), np.uint64)
    _abi.check(_abi._lib.absp_debug_score_trace(sc.ctypes.data, sc.nbytes))
    _abi.check(_abi._lib.absp_debug_topk_trace(tk.ctypes.data, tk.nbytes))
    _abi.check(_abi._lib.absp_debug_attn_trace(at.ctypes.data, at.nbytes))
    ns = 2 * 148
    if FAST:  # tensor-core filter + refine: time base = first refine CTA start
        rf = np.zeros((1024, 8), np.uint64)
        cand = np.zeros(1024, np.uint32)
        _abi.check(_abi._lib.absp_debug_refine_trace(rf.ctypes.data, rf.nbytes, cand.ctypes.data, cand.nbytes))
        units = B * H
        t0 = int(rf[:units, 0].min())
        r = lambda a: (a.astype(np.int64) - t0) / 1e3
        print(f"rep {rep} (us from the first refine CTA start; pctl 0/10/50/90/100)")
        for j, nm in enumerate(["start", "after griddep wait", "loads", "kth bound", "candidates+table",
                                "exact scored", "ordered", "end"]):
            print(f"  refine {nm:18s} {pct(r(rf[:units, j]))}")
        sc[:] = 0
        sc[:, 0] = t0
    t0 = int(sc[:ns, 0].min())
    r = lambda a: (a.astype(np.int64) - t0) / 1e3
    units = B * H
    if not FAST:
        print(f"rep {rep} (us from the first scorer CTA start; pctl 0/10/50/90/100)")
        print(f"  scorer start      {pct(r(sc[:ns, 0]))}")
        print(f"  scorer end        {pct(r(sc[:ns, 1]))}")
    if not FAST and tk[:units, 0].max() >= sc[:ns, 0].min():
        print(f"  topk start        {pct(r(tk[:units, 0]))}")
        for j, nm in ((1, "topk keys issued"), (2, "topk threshold"), (3, "topk compacted"), (4, "topk ordered")):
            v = tk[:units, j]
            if (v > 0).any():
                print(f"  {nm:17s} {pct(r(v[v > 0]))}")
        print(f"  topk end (pages)  {pct(r(tk[:units, 5][tk[:units, 5] > 0]))}")
        te = r(tk[:units, 5])
        q4 = units // 4
        print("  topk end by unit quarter (medians):", [round(float(np.median(te[i * q4:(i + 1) * q4])), 2) for i in range(4)])
    print(f"  attn CTA start    {pct(r(at[:148, 0]))}")
    if at[:148, 250].max() > 0:
        print(f"  attn selected     {pct(r(at[:148, 250][at[:148, 250] > 0]))}")
    first = np.array([at[c, 64] for c in range(148)])
    print(f"  attn first issue  {pct(r(at[:148, 1]))}")
    print(f"  attn first data   {pct(r(first))}")
    print(f"    issue - start   {pct((at[:148, 1].astype(np.int64) - at[:148, 0].astype(np.int64)) / 1e3)}")
    print(f"    data - issue    {pct((first.astype(np.int64) - at[:148, 1].astype(np.int64)) / 1e3)}")
    print(f"    2nd - 1st data  {pct((at[:148, 65].astype(np.int64) - first.astype(np.int64)) / 1e3)}")
    last_arr = np.array([max(at[c, 64:128]) for c in range(148)])
    print(f"  attn last data    {pct(r(last_arr))}")
    ends = np.array([max(at[c, 242:250]) for c in range(148)])
    print(f"  attn end          {pct(r(ends))}")
