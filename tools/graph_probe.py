import sys, time
sys.path.insert(0, "/root/repo")
import torch
from bench import SEED, WORKLOADS
from paper_2605_12110_b200 import BlockAssignment, DecodeAttention, EngineConfig, QuantSpec, fill_synthetic_bf16
w = WORKLOADS["cfg3"]
B, n, H, G, d, P, T = w["batch"], w["n"], w["H"], w["G"], w["d"], w["P"], w["T"]
L = 3
pages = B * ((n + P - 1) // P)
cfg = EngineConfig(num_heads=H, head_dim=d, page_size=P, candidate_block_sizes=tuple(w["cands"]), token_budget=T,
                   quant=QuantSpec(4), num_q_heads=H * G, max_batch=B, max_seq_len=n, num_layers=L)
da = DecodeAttention(cfg)
lay = []
for l in range(L):
    da.set_assignment(l, BlockAssignment.cycled(H, w["cands"]))
    k = torch.empty(H, pages, P, d, dtype=torch.int16, device="cuda"); v = torch.empty_like(k)
    q = torch.empty(B, H * G, d, dtype=torch.int16, device="cuda")
    for t, s in ((k, 3 * l), (v, 3 * l + 1), (q, 3 * l + 2)):
        fill_synthetic_bf16(t, SEED, s)
    pt = torch.arange(pages, dtype=torch.int32, device="cuda").reshape(B, -1)
    da.bind(l, k, v, pt, [n] * B); da.build_store(l)
    lay.append(dict(k=k, v=v, q=q, pt=pt, out=torch.empty(B, H * G, d, dtype=torch.float32, device="cuda")))
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for l in range(L):
        da.decode_step(l, lay[l]["q"], lay[l]["out"], s)
    per = []
    for l in range(L):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            da.decode_step(l, lay[l]["q"], lay[l]["out"], s)
        per.append(g)
    gall = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gall, stream=s):
        for l in range(L):
            da.decode_step(l, lay[l]["q"], lay[l]["out"], s)
    att = []
    for l in range(L):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            da.attend_selected(l, lay[l]["q"], lay[l]["out"], s)
        att.append(g)
    aall = torch.cuda.CUDAGraph()
    with torch.cuda.graph(aall, stream=s):
        for l in range(L):
            da.attend_selected(l, lay[l]["q"], lay[l]["out"], s)
def tm(fn, reps):
    with torch.cuda.stream(s):
        for i in range(5): fn(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(reps): fn(i)
        e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps
K = 60
print("step per-layer graphs   %.1f us" % tm(lambda i: per[i % L].replay(), K))
print("step 3-layer graph /3   %.1f us" % (tm(lambda i: gall.replay(), K // L) / L))
print("attn per-layer graphs   %.1f us" % tm(lambda i: att[i % L].replay(), K))
print("attn 3-layer graph /3   %.1f us" % (tm(lambda i: aall.replay(), K // L) / L))
