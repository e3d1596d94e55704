"""compute-sanitizer driver (tools/gpu_sanitize.sh): a cfg1-sized layer (batch 2, 3000 and
1100 tokens, 8 KV heads, G = 4, blocks {8, 16, 32}, T = 1024) through every product entry
point that launches kernels: build_store, decode_step (fused selection + attention with
ready flags), append (incremental maintenance), decode_step_host (graph, pinned output),
select + attend (explicit selection), full_attention + attention_recall (dense fp64).
Tooling, not product; exits non-zero on any API error."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2605_12110_b200 import (BlockAssignment, DecodeAttention, EngineConfig, QuantSpec,  # noqa: E402
                                   fill_synthetic_bf16)

B, H, G, d, P, T = 2, 8, 4, 128, 8, 1024
lens = [3000, 1100]
cands = (8, 16, 32)
cap = 3200
pages_per = (cap + P - 1) // P
cfg = EngineConfig(num_heads=H, head_dim=d, page_size=P, candidate_block_sizes=cands, token_budget=T,
                   quant=QuantSpec(4), num_q_heads=H * G, max_batch=B, max_seq_len=cap)
da = DecodeAttention(cfg)
da.set_assignment(0, BlockAssignment.cycled(H, cands))
k = torch.empty(H, B * pages_per, P, d, dtype=torch.int16, device="cuda")
v = torch.empty_like(k)
q = torch.empty(B, H * G, d, dtype=torch.int16, device="cuda")
for t, s in ((k, 0), (v, 1), (q, 2)):
    fill_synthetic_bf16(t, 42, s)
pt = torch.arange(B * pages_per, dtype=torch.int32, device="cuda").reshape(B, -1)
da.bind(0, k, v, pt, lens)
da.build_store(0)
out = torch.empty(B, H * G, d, dtype=torch.float32, device="cuda")
for _ in range(2):
    da.decode_step(0, q, out)
kn = torch.empty(B, H, d, dtype=torch.int16, device="cuda")
vn = torch.empty_like(kn)
for step in range(3):
    fill_synthetic_bf16(kn, 7 + step, 10)
    fill_synthetic_bf16(vn, 7 + step, 11)
    da.append(0, kn, vn)
    da.decode_step(0, q, out)
qh = q.cpu().pin_memory()
oh = torch.empty(B, H * G, d, dtype=torch.float32).pin_memory()
for _ in range(2):
    da.decode_step_host(0, qh, oh)
stride = da.layer_info(0).max_select
blocks = torch.zeros(B, H, stride, dtype=torch.int32, device="cuda")
counts = torch.zeros(B, H, dtype=torch.int32, device="cuda")
da.select(0, q, blocks, counts)
da.attend(0, q, blocks, counts, out)
w = torch.zeros(B, H * G, cap, dtype=torch.float64, device="cuda")
da.full_attention(0, q, out, w)
rec = torch.zeros(B, H * G, dtype=torch.float64, device="cuda")
da.attention_recall(0, w, blocks, counts, rec)
torch.cuda.synchronize()
print("sanitize driver ok, launches", da.launch_count())
