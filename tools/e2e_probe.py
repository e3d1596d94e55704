"""Where the end-to-end (host buffer) step time goes: host wall time per step of
 (a) an empty graph (one tiny kernel) launched and synchronised: the launch + wake-up floor,
 (b) the decode-step graph on device buffers, launched and synchronised,
 (c) absp_decode_step_host with pinned q / out (the bench's e2e path).
Tooling, not product. usage: python tools/e2e_probe.py [workload] [batch]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

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
x = torch.zeros(1, device="cuda")


def wall(fn, reps=200):
    for _ in range(10):
        fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e6


with torch.cuda.stream(stream):
    ge = torch.cuda.CUDAGraph()
    with torch.cuda.graph(ge, stream=stream):
        x.add_(1)
    da.decode_step(0, q, out, stream)
    gs = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gs, stream=stream):
        da.decode_step(0, q, out, stream)
qh = q.cpu().pin_memory()
oh = torch.empty(out.shape, dtype=torch.float32).pin_memory()
a = wall(lambda: (ge.replay(), torch.cuda.synchronize()))
b = wall(lambda: (gs.replay(), torch.cuda.synchronize()))
c = wall(lambda: da.decode_step_host(0, qh, oh, stream))
print(f"B={B}: empty graph {a:.1f} us | decode-step graph (device buffers) {b:.1f} us | "
      f"decode_step_host (pinned) {c:.1f} us")
if "--copies" in sys.argv:  # the same with copy nodes instead of direct host access (diagnostics)
    import os
    res = {}
    for mode, name in ((1, "q copy"), (2, "out copy"), (3, "both copies"), (0, "direct")):
        os.environ["ABSP_HOST_STEP_COPY"] = str(mode)
        dx = DecodeAttention(cfg)
        dx.set_assignment(0, BlockAssignment.cycled(H, w["cands"]))
        dx.bind(0, k, v, pt, [n] * B)
        dx.build_store(0)
        res[name] = wall(lambda: dx.decode_step_host(0, qh, oh, stream))
        del dx
    print("  " + " | ".join(f"{k} {v:.1f} us" for k, v in res.items()))
