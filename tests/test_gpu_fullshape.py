"""Parity at the benchmark's own full shapes ("the timed configurations are
not the tested ones"): the whole batch runs on the GPU exactly as bench.py builds it
(device-generated synthetic K/V/q, a shuffled page table), and sampled sequences are
read back and checked against the C restatement of the reference (oracle/):

  store (codes, scales, zero points), scores : bit-exact
  selection (absp_select and the decode step's own) : bit-exact, ordered
  attention output : |got - want| <= 1e-3 + 1e-2 |want|
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


@pytest.mark.parametrize("name,B,n,G,P,cands,T,check", [
    # cfg5 at its per-GPU shape on 8 B200s: Qwen3-32B (64q / 8kv), 128K, blocks {4..64}
    ("cfg5/8", 8, 131072, 8, 4, (4, 8, 16, 32, 64), 2048, (0, 7)),
    # cfg3 at its 1-GPU shape: Llama-3.1-8B (32q / 8kv), batch 16, 128K, blocks {16,32,64}
    ("cfg3", 16, 131072, 4, 16, (16, 32, 64), 2048, (0, 9, 15)),
])
def test_bench_shape_parity(cuda, name, B, n, G, P, cands, T, check):
    from gpu_util import within_tol
    from layer_data import Layer, oracle_step
    from paper_2605_12110_b200 import (BlockAssignment, DecodeAttention, EngineConfig, QuantSpec,
                                       fill_synthetic_bf16)
    H, d = 8, 128
    pps = (n + P - 1) // P
    pages = B * pps
    k = torch.empty(H, pages, P, d, dtype=torch.int16, device="cuda")
    v = torch.empty_like(k)
    q = torch.empty(B, H * G, d, dtype=torch.int16, device="cuda")
    fill_synthetic_bf16(k, 42, 0)
    fill_synthetic_bf16(v, 42, 1)
    fill_synthetic_bf16(q, 42, 2)
    gen = torch.Generator(device="cuda").manual_seed(7)
    pt = torch.randperm(pages, generator=gen, device="cuda", dtype=torch.int64).to(torch.int32).reshape(B, pps)
    cfg = EngineConfig(num_heads=H, head_dim=d, page_size=P, candidate_block_sizes=cands, token_budget=T,
                       quant=QuantSpec(4), num_q_heads=H * G, max_batch=B, max_seq_len=n)
    da = DecodeAttention(cfg)
    assignment = BlockAssignment.cycled(H, cands)
    da.set_assignment(0, assignment)
    da.bind(0, k, v, pt, [n] * B)
    da.build_store(0)
    info = da.layer_info(0)
    blocks = torch.zeros(B, H, info.max_select, dtype=torch.int32, device="cuda")
    counts = torch.zeros(B, H, dtype=torch.int32, device="cuda")
    da.select(0, q, blocks, counts)
    torch.cuda.synchronize()
    sel_b, sel_c = blocks.cpu().numpy().view(np.uint32), counts.cpu().numpy().view(np.uint32)
    out = torch.empty(B, H * G, d, dtype=torch.float32, device="cuda")
    da.decode_step(0, q, out)
    torch.cuda.synchronize()
    step_sel = da.download_selection(0)
    got = out.cpu().numpy()
    for b in check:
        rows = pt[b].long()
        layer = Layer(H, G, d, P, assignment.block_sizes, [n], k[:, rows].cpu().numpy().view(np.uint16),
                      v[:, rows].cpu().numpy().view(np.uint16), np.arange(pps, dtype=np.uint32).reshape(1, -1),
                      q[b:b + 1].cpu().numpy().view(np.uint16))
        seq, sc, want_sel, want = oracle_step(layer, 0, T)
        st = da.download_store(0, b)
        assert np.array_equal(st["codes"], seq.codes), (name, b)
        assert np.array_equal(_bits(st["scales"]), _bits(seq.scales)), (name, b)
        assert np.array_equal(_bits(st["zps"]), _bits(seq.zps)), (name, b)
        assert np.array_equal(_bits(da.download_scores(0, b)), _bits(sc)), (name, b)
        for h in range(H):
            assert np.array_equal(sel_b[b, h, :sel_c[b, h]], want_sel[h]), (name, b, h)
            assert np.array_equal(step_sel[b][h], want_sel[h]), (name, "decode step", b, h)
        ok, err = within_tol(got[b], want)
        assert ok, f"{name} seq {b}: max abs err {err}"
    del k, v
    torch.cuda.empty_cache()
