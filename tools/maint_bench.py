"""Decode-time maintenance cost (absp_append: append + refresh_tail_centroids +
requantize_heads) on a cfg-3-shaped layer with headroom, wall-clock per call (it synchronises).
Tooling, not product."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import SEED, WORKLOADS  # noqa: E402
from paper_2605_12110_b200 import BlockAssignment, DecodeAttention, EngineConfig, QuantSpec, fill_synthetic_bf16  # noqa: E402

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
B, n, H, G, d, P, T = w["batch"], w["n"], w["H"], w["G"], w["d"], w["P"], w["T"]
extra = 64
cap = n + extra
pps = (cap + P - 1) // P
cfg = EngineConfig(num_heads=H, head_dim=d, page_size=P, candidate_block_sizes=tuple(w["cands"]), token_budget=T,
                   quant=QuantSpec(4), num_q_heads=H * G, max_batch=B, max_seq_len=cap)
da = DecodeAttention(cfg)
da.set_assignment(0, BlockAssignment.cycled(H, w["cands"]))
k = torch.empty(H, B * pps, P, d, dtype=torch.int16, device="cuda")
v = torch.empty_like(k)
for t, s in ((k, 0), (v, 1)):
    fill_synthetic_bf16(t, SEED, s)
pt = torch.arange(B * pps, dtype=torch.int32, device="cuda").reshape(B, pps)
da.bind(0, k, v, pt, [n] * B)
da.build_store(0)
q = torch.empty(B, H * G, d, dtype=torch.int16, device="cuda")
kn = torch.empty(extra, B, H, d, dtype=torch.int16, device="cuda")  # a fresh token every step
vn = torch.empty_like(kn)
for t, s in ((q, 2), (kn, 3), (vn, 4)):
    fill_synthetic_bf16(t, SEED, s)
out = torch.empty(B, H * G, d, dtype=torch.float32, device="cuda")
times, steps, enq = [], [], []
for i in range(extra - 1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    da.append(0, kn[i], vn[i])
    te = time.perf_counter()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    enq.append(te - t0)
    da.decode_step(0, q, out)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    times.append(t1 - t0)
    steps.append(t2 - t1)
times.sort()
steps.sort()
enq.sort()
print(f"append+refresh (batch {B}, {n}+ ctx): median {times[len(times) // 2] * 1e6:.1f} us, "
      f"min {times[0] * 1e6:.1f} us (host enqueue median {enq[len(enq) // 2] * 1e6:.1f} us); "
      f"eager decode_step median {steps[len(steps) // 2] * 1e6:.1f} us")
