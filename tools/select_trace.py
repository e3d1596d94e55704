"""Decode-step selection timeline (debug): cfg-3 decode steps with lib/libabsp_trace.so;
per-unit phase stamps of k_select_refine and its candidate counts. Tooling, not product."""
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_12110_b200 import _abi  # noqa: E402

_abi._lib = _abi.load(ROOT / "paper_2605_12110_b200" / "lib" / "libabsp_trace.so")
_abi._lib.absp_debug_refine_trace.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t]
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
units = B * H
tr = np.zeros((1024, 8), np.uint64)
cand = np.zeros(1024, np.uint32)
_abi.check(_abi._lib.absp_debug_refine_trace(tr.ctypes.data, tr.nbytes, cand.ctypes.data, cand.nbytes))
t0 = tr[:units, 0].min()
pct = lambda a: " ".join(f"{x:7.2f}" for x in np.percentile(a, [0, 10, 50, 90, 100]))
print(f"{units} unit CTAs, candidates pctl 0/10/50/90/100: {pct(cand[:units].astype(float))}")
names = ["start", "after griddep wait", "loads", "kth bound", "candidates+table", "exact scored", "ordered", "end"]
for j, nm in enumerate(names):
    rel = (tr[:units, j].astype(np.int64) - int(t0)) / 1e3
    print(f"  {nm:20s} {pct(rel)}")
