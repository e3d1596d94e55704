"""Scorer timeline (debug): one cfg-3 select with lib/libabsp_trace.so after an L2 flush;
per-CTA globaltimer stamps (start, per-item table ready, end). Tooling, not product."""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_12110_b200 import _abi  # noqa: E402

_abi._lib = _abi.load(ROOT / "paper_2605_12110_b200" / "lib" / "libabsp_trace.so")
_abi._lib.absp_debug_score_trace.argtypes = [C.c_void_p, C.c_size_t]
_abi._lib.absp_debug_topk_trace.argtypes = [C.c_void_p, C.c_size_t]
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
stride = da.layer_info(0).max_select
blocks = torch.empty(B, H, stride, dtype=torch.int32, device="cuda")
counts = torch.empty(B, H, dtype=torch.int32, device="cuda")
for _ in range(3):
    da.select(0, q, blocks, counts)
torch.cuda.synchronize()
flush = torch.empty(1 << 28, dtype=torch.int8, device="cuda")
for rep in range(3):
    flush.fill_(rep)  # evict L2
    torch.cuda.synchronize()
    da.select(0, q, blocks, counts)
    torch.cuda.synchronize()
    tr = np.zeros((320, 16), np.uint64)
    _abi.check(_abi._lib.absp_debug_score_trace(tr.ctypes.data, tr.nbytes))
    ctas = [c for c in range(320) if tr[c, 0] and tr[c, 1]]
    t0 = min(int(tr[c, 0]) for c in ctas)
    st = np.array([(int(tr[c, 0]) - t0) / 1e3 for c in ctas])
    en = np.array([(int(tr[c, 1]) - t0) / 1e3 for c in ctas])
    ft = np.array([(int(tr[c, 2]) - t0) / 1e3 for c in ctas])
    pct = lambda a: " ".join(f"{x:6.2f}" for x in np.percentile(a, [0, 10, 50, 90, 100]))
    print(f"rep {rep}: {len(ctas)} CTAs (pctl 0/10/50/90/100, us from first start)")
    print(f"  start       {pct(st)}")
    print(f"  first table {pct(ft)}")
    print(f"  end         {pct(en)}")
    print(f"  busy        {pct(en - st)}")
    nitems = np.array([sum(1 for i in range(14) if tr[c, 2 + i] and int(tr[c, 2 + i]) >= int(tr[c, 0])) for c in ctas])
    for k in sorted(set(nitems.tolist())):
        sel = nitems == k
        print(f"  CTAs with {k} item(s): {sel.sum():3d}, end median {np.median(en[sel]):6.2f} us, "
              f"busy median {np.median((en - st)[sel]):6.2f} us")
    print("  end by CTA index (0-147 | 148-295) medians:", np.median(en[:148]).round(2), np.median(en[148:]).round(2))
    tk = np.zeros((1024, 8), np.uint64)
    _abi.check(_abi._lib.absp_debug_topk_trace(tk.ctypes.data, tk.nbytes))
    units = [u for u in range(B * H) if tk[u, 0] and tk[u, 5]]
    if units:
        s0 = min(int(tk[u, 0]) for u in units)
        print(f"  topk: {len(units)} fast-path units; relative to first topk CTA start (kernel gap after scorer end: "
              f"{(s0 - t0) / 1e3 - en.max():.2f} us)")
        for j, name in enumerate(["start", "keys loaded", "threshold", "compacted", "sorted", "pages"]):
            print(f"    {name:12s} {pct(np.array([(int(tk[u, j]) - s0) / 1e3 for u in units]))}")
    items = [[(int(tr[c, 2 + i]) - int(tr[c, 0])) / 1e3 for i in range(14) if tr[c, 2 + i] and int(tr[c, 2 + i]) >= int(tr[c, 0])] for c in ctas[:4]]
    print("  item-ready offsets of CTAs 0-3:", [[round(x, 2) for x in it] for it in items])
