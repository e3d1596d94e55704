"""GPU parity of the dense fp64 path (absp_full_attention, absp_attention_recall) against the
unmodified reference (oracle/_ref): full_attention_oracle (engine.cpp:357-403) and
attention_recall (calibrator.cpp:48-71), per q head.

  weights  : |got - want| <= 1e-12 |want| + 1e-300 (logits are bit-exact; the softmax
             denominator is summed in another order)
  output   : |got - want| <= 1e-6 + 1e-6 |want|   (fp64 sums rounded once to fp32)
  recall   : |got - want| <= 1e-12
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from layer_data import make_layer  # noqa: E402
from oracle.oracle import RefSeq, ref_available  # noqa: E402


def _ref_seq(layer, b):
    seq = layer.oracle_seq(b)
    k = seq.keys_logical().astype(np.float32)
    v = seq.values_logical().astype(np.float32)
    return RefSeq(k, v, layer.P, layer.block_sizes, 0, 4, 1)


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("d,G,P,cands,seq_lens", [
    (128, 4, 16, (16, 32, 64), (5000, 777, 16)),
    (128, 8, 4, (4, 8, 16), (3001, 1)),
    (64, 1, 8, (8, 16), (2049,)),
    (128, 2, 16, (16,), (12000,)),
])
def test_full_attention_vs_reference(cuda, d, G, P, cands, seq_lens):
    from gpu_util import GpuLayer
    rng = np.random.default_rng(d + 10 * G + P)
    layer = make_layer(int(rng.integers(1 << 30)), H=4, G=G, d=d, P=P, block_sizes=cands, seq_lens=seq_lens,
                       scale=2.0)
    gl = GpuLayer(layer, 256)
    Hq = layer.H * G
    n_max = max(seq_lens)
    stride = n_max + 7
    out = torch.full((layer.batch, Hq, d), float("nan"), dtype=torch.float32, device="cuda")
    w = torch.full((layer.batch, Hq, stride), -1.0, dtype=torch.float64, device="cuda")
    gl.da.full_attention(0, gl.q, out, w)
    torch.cuda.synchronize()
    out_h = out.cpu().numpy()
    w_h = w.cpu().numpy()
    for b in range(layer.batch):
        rs = _ref_seq(layer, b)
        n = seq_lens[b]
        qg = layer.qf(b).reshape(layer.H, G, d)
        for g in range(G):
            want_o, want_w = rs.full_attention_weights(np.ascontiguousarray(qg[:, g, :]))
            for h in range(layer.H):
                hq = h * G + g
                got_w = w_h[b, hq, :n]
                assert np.all(np.abs(got_w - want_w[h]) <= 1e-12 * np.abs(want_w[h]) + 1e-300), (b, hq)
                assert np.all(w_h[b, hq, n:] == -1.0)  # nothing written past the sequence
                assert np.allclose(out_h[b, hq], want_o[h], rtol=1e-6, atol=1e-6), (b, hq)


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_attention_recall_vs_reference_selection(cuda):
    """Recall of the GPU's own (bit-exact) selection under the GPU weights equals the
    reference's attention_recall restated in numpy on the reference's weights."""
    from gpu_util import GpuLayer
    rng = np.random.default_rng(5)
    layer = make_layer(int(rng.integers(1 << 30)), H=8, G=1, d=128, P=16, block_sizes=(16, 32, 64),
                       seq_lens=(9000, 4100), scale=2.0)
    gl = GpuLayer(layer, 1024)
    sel = gl.select()
    stride = max(gl.info.max_select, 1)
    blocks = torch.zeros(layer.batch, layer.H, stride, dtype=torch.int32, device="cuda")
    counts = torch.zeros(layer.batch, layer.H, dtype=torch.int32, device="cuda")
    gl.da.select(0, gl.q, blocks, counts)
    n_max = max(layer.seq_lens)
    w = torch.zeros((layer.batch, layer.H, n_max), dtype=torch.float64, device="cuda")
    out = torch.zeros((layer.batch, layer.H, layer.d), dtype=torch.float32, device="cuda")
    gl.da.full_attention(0, gl.q, out, w)
    rec = torch.zeros((layer.batch, layer.H), dtype=torch.float64, device="cuda")
    gl.da.attention_recall(0, w, blocks, counts, rec)
    torch.cuda.synchronize()
    rec = rec.cpu().numpy()
    for b in range(layer.batch):
        rs = _ref_seq(layer, b)
        _, want_w = rs.full_attention_weights(layer.qf(b))
        n = layer.seq_lens[b]
        for h in range(layer.H):
            B = layer.block_sizes[h]
            mask = np.zeros(n, bool)
            for blk in sel[b][h]:
                mask[blk * B:(blk + 1) * B] = True
            want = float(want_w[h][mask[:n]].sum())
            assert abs(rec[b, h] - want) <= 1e-12, (b, h, rec[b, h], want)
            assert 0.0 < rec[b, h] <= 1.0 + 1e-12
