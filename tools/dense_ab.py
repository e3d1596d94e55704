"""Sparse vs dense decode attention A/B: one layer of a workload's shape
on one GPU, the same synthetic KV, three paths timed with CUDA events over graph replays
(an L2-sized buffer is rewritten between replays so the KV is never L2-resident):

  sparse : absp_decode_step (fused selection + block-sparse attention, the product path)
  dense  : absp_attend over EVERY block of every head (the same flash-decode kernel, no
           selection): the bf16 / fp32-accumulate full-attention baseline
  oracle : absp_full_attention (fp64 full attention with weights, the calibration oracle)

Prints one JSON line. Tooling, not product.
usage: python tools/dense_ab.py [workload] [batch]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from bench import SEED, WORKLOADS  # noqa: E402
from paper_2605_12110_b200 import (BlockAssignment, DecodeAttention, EngineConfig, QuantSpec,  # noqa: E402
                                   fill_synthetic_bf16)

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4
n, H, G, d, P, T = w["n"], w["H"], w["G"], w["d"], w["P"], w["T"]
pages = B * ((n + P - 1) // P)
cfg = EngineConfig(num_heads=H, head_dim=d, page_size=P, candidate_block_sizes=tuple(w["cands"]), token_budget=T,
                   quant=QuantSpec(4), num_q_heads=H * G, max_batch=B, max_seq_len=n)
da = DecodeAttention(cfg)
asg = BlockAssignment.cycled(H, w["cands"])
da.set_assignment(0, asg)
k = torch.empty(H, pages, P, d, dtype=torch.int16, device="cuda")
v = torch.empty_like(k)
q = torch.empty(B, H * G, d, dtype=torch.int16, device="cuda")
for t, s in ((k, 0), (v, 1), (q, 2)):
    fill_synthetic_bf16(t, SEED, s)
pt = torch.arange(pages, dtype=torch.int32, device="cuda").reshape(B, -1)
da.bind(0, k, v, pt, [n] * B)
da.build_store(0)
out = torch.empty(B, H * G, d, dtype=torch.float32, device="cuda")
# every block of every head, in index order
nmax = max((n + b - 1) // b for b in asg.block_sizes)
blocks = torch.zeros(B, H, nmax, dtype=torch.int32, device="cuda")
counts = torch.zeros(B, H, dtype=torch.int32, device="cuda")
for h, bs in enumerate(asg.block_sizes):
    nb = (n + bs - 1) // bs
    blocks[:, h, :nb] = torch.arange(nb, dtype=torch.int32, device="cuda")
    counts[:, h] = nb
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
stream = torch.cuda.Stream()


def timed(fn, reps=10):
    with torch.cuda.stream(stream):
        for _ in range(2):
            fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            fn()
        ts = []
        for i in range(reps):
            flush.fill_(i & 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g.replay()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


kv_dense = 2 * H * B * n * d * 2
res = {"workload": sys.argv[1] if len(sys.argv) > 1 else "cfg3", "batch": B, "seq_len": n}
t_sparse = timed(lambda: da.decode_step(0, q, out, stream))
t_dense = timed(lambda: da.attend(0, q, blocks, counts, out, stream, validate=False))
t_oracle = timed(lambda: da.full_attention(0, q, out, None, stream), reps=3)
for name, t, by in (("sparse", t_sparse, None), ("dense", t_dense, kv_dense), ("oracle_fp64", t_oracle, kv_dense)):
    res[name] = {"us": round(t, 1), "tokens_per_s": round(B / (t * 1e-6)),
                 **({"kv_gbs": round(by / (t * 1e-6) / 1e9)} if by else {})}
res["dense_over_sparse"] = round(t_dense / t_sparse, 1)
print(json.dumps(res))
