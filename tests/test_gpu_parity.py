"""GPU parity: the sm_100a path through the C ABI against the reference's committed
outputs (tests/golden) and the C restatement (oracle/), on identical bf16 inputs.

  store (centroids, codes, scales, zero points) : bit-exact
  scores                                        : bit-exact
  selected block ids (ordered)                  : bit-exact
  attention output                              : |got-want| <= 1e-3 + 1e-2|want|
"""
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from golden.make_golden import CASES, case_inputs  # noqa: E402
from layer_data import Layer, make_layer, oracle_step  # noqa: E402

GOLDEN = Path(__file__).parent / "golden" / "golden_v1.npz"


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def _golden_layer(name) -> tuple:
    c = case_inputs(name)
    pages = len(c["page_table"])
    pt = np.zeros((1, pages + 1), np.uint32)
    pt[0, :pages] = c["page_table"]
    layer = Layer(c["H"], c["G"], c["d"], c["P"], c["block_sizes"], [c["n"]], c["k_pool"], c["v_pool"], pt,
                  c["q"].reshape(1, c["H"] * c["G"], c["d"]))
    return c, layer


@pytest.mark.parametrize("name", list(CASES))
def test_golden_cases(cuda, golden, name):
    from gpu_util import GpuLayer, within_tol
    c, layer = _golden_layer(name)
    g = lambda k: golden[f"{name}/{k}"]
    gl = GpuLayer(layer, c["T"], c["method"], c["bits"], c["mode"])
    st = gl.da.download_store(0, 0)
    assert np.array_equal(st["offsets"], g("offsets"))
    assert np.array_equal(_bits(st["values"]), _bits(g("values")))
    if c["method"] == 1:
        assert np.array_equal(_bits(st["values_min"]), _bits(g("values_min")))
    if c["bits"]:
        assert np.array_equal(st["codes"], g("codes"))
        assert np.array_equal(_bits(st["scales"]), _bits(g("scales")))
        assert np.array_equal(_bits(st["zps"]), _bits(g("zps")))
        if c["method"] == 1:
            assert np.array_equal(st["codes_min"], g("codes_min"))
            assert np.array_equal(_bits(st["scales_min"]), _bits(g("scales_min")))
    sel = gl.select()[0]
    assert np.array_equal(_bits(gl.da.download_scores(0, 0)), _bits(g("scores")))
    assert np.array_equal(np.array([len(s) for s in sel], np.uint32), g("sel_counts"))
    assert np.array_equal(np.concatenate(sel), g("sel_blocks"))
    out = gl.decode()[0]
    # the decode step selects through its own path (the fused select.cu for int4 mean): same blocks
    dsel = gl.step_selection[0]
    assert np.array_equal(np.array([len(s) for s in dsel], np.uint32), g("sel_counts"))
    assert np.array_equal(np.concatenate(dsel), g("sel_blocks"))
    ok, err = within_tol(out, g("attn_out"))
    assert ok, f"max abs err {err}"
    if c["n"] <= c["T"]:  # full coverage: also within tolerance of the fp64 oracle
        ok, err = within_tol(out, g("full_out"))
        assert ok, f"vs full attention: max abs err {err}"


@pytest.mark.parametrize("G,H,P,cands,seq_lens,T", [
    (4, 8, 8, (8, 16, 32), (8192,), 1024),                  # cfg 1 shape (Llama-3.1-8B layer)
    (4, 8, 16, (16, 32, 64), (5000, 3333, 17, 12000), 2048),  # ragged batch, cfg 3 block sizes
    (8, 8, 4, (4, 8, 16, 32, 64), (9001, 6000), 2048),        # cfg 5 shape (Qwen3-32B, G=8, P=4)
    (1, 2, 16, (16,), (700, 64), 128),                        # MHA, uniform blocks
    (2, 4, 16, (16, 32, 64), (100, 2000), 4096),              # T >= n: every block selected
    (1, 2, 16, (16, 64), (3000, 700), 64),                    # K = 1 (B = 64 = T): the trailing block only
    (4, 8, 16, (16, 32, 64), (20000,) * 20, 2048),            # 160 units: one CTA per unit, slices recycled
    (4, 8, 8, (8, 24, 40), (5000, 1234), 1024),               # block sizes that do not divide the 128-row
    (4, 8, 16, (16, 48, 80, 112), (9000, 777), 2048),         #   attention chunk (any multiple of P, as the
    (8, 4, 4, (12, 20), (3000,), 512),                        #   reference allows): chunks with empty slots
    (4, 4, 2, (2, 8, 32), (3001, 515), 1024),                 # P = 2 and P = 1: 64 / 128 page slots per
    (2, 4, 1, (1, 4), (1500,), 512),                          #   chunk, 4 attention producer warps
])
def test_random_batches_vs_oracle(cuda, G, H, P, cands, seq_lens, T):
    from gpu_util import GpuLayer, within_tol
    layer = make_layer(sum(seq_lens) + G, H=H, G=G, d=128, P=P, block_sizes=cands, seq_lens=seq_lens)
    gl = GpuLayer(layer, T, 0, 4, 1, max_seq_len=max(seq_lens) + 100)
    sel = gl.select()
    out = gl.decode()
    for b in range(layer.batch):
        seq, sc, want_sel, want = oracle_step(layer, b, T)
        st = gl.da.download_store(0, b)
        assert np.array_equal(st["codes"], seq.codes)
        assert np.array_equal(_bits(st["scales"]), _bits(seq.scales))
        assert np.array_equal(_bits(gl.da.download_scores(0, b)), _bits(sc))
        for h in range(H):
            assert np.array_equal(sel[b][h], want_sel[h]), (b, h)
            assert np.array_equal(gl.step_selection[b][h], want_sel[h]), ("decode step", b, h)
        ok, err = within_tol(out[b], want)
        assert ok, f"seq {b}: max abs err {err}"


@pytest.mark.parametrize("P,cands,swaps", [
    (4, (4, 8, 16, 32, 64), 0),    # cfg 5 shape: B >= 16 chunks load as 16-row runs
    (4, (16, 32, 64), 25),          # some runs broken by swapped pages: per-page fallback
    (8, (8, 16, 32), 0),            # cfg 1 shape
    (2, (16, 32), 9),
    (1, (16, 64), 0),
])
def test_sequential_pages_run_copies(cuda, P, cands, swaps):
    """Sequentially allocated pages (the reference's allocator) with P < 16: attention chunks
    made of whole 16-row runs of consecutive pages are copied run-wise (attend.cu); the
    output must not change."""
    from gpu_util import GpuLayer, within_tol
    seq_lens, T = (7001, 4096), 1024
    layer = make_layer(P * 31 + swaps, H=8, G=8, d=128, P=P, block_sizes=cands, seq_lens=seq_lens,
                       sequential=True, swaps=swaps)
    gl = GpuLayer(layer, T, 0, 4, 1, max_seq_len=max(seq_lens) + 100)
    sel = gl.select()
    out = gl.decode()
    for b in range(layer.batch):
        seq, sc, want_sel, want = oracle_step(layer, b, T)
        for h in range(layer.H):
            assert np.array_equal(sel[b][h], want_sel[h]), (b, h)
        ok, err = within_tol(out[b], want)
        assert ok, f"seq {b}: max abs err {err}"


@pytest.mark.parametrize("method,bits,mode", [(0, 4, 0), (0, 8, 1), (0, 2, 0), (0, 0, 1), (1, 4, 1), (1, 8, 0), (1, 0, 1)])
def test_quant_grid_vs_oracle(cuda, method, bits, mode):
    from gpu_util import GpuLayer
    layer = make_layer(7 + bits + method, H=8, G=4, d=128, P=16, seq_lens=(3000, 1234), scale=3.0)
    gl = GpuLayer(layer, 512, method, bits, mode)
    sel = gl.select()
    for b in range(layer.batch):
        seq, sc, want_sel, _ = oracle_step(layer, b, 512, method, bits, mode)
        st = gl.da.download_store(0, b)
        assert np.array_equal(_bits(st["values"]), _bits(seq.values))
        if bits:
            assert np.array_equal(st["codes"], seq.codes)
        assert np.array_equal(_bits(gl.da.download_scores(0, b)), _bits(sc))
        assert all(np.array_equal(x, y) for x, y in zip(sel[b], want_sel))


def test_ties_pick_lowest_indices(cuda):
    from gpu_util import GpuLayer
    # all keys equal -> all centroids and scores equal -> lowest block ids + trailing block
    layer = make_layer(3, H=4, G=2, d=64, P=16, seq_lens=(4000,))
    layer.k_pool[:] = 0x3F80
    gl = GpuLayer(layer, 256)
    sel = gl.select()[0]
    for h, b in enumerate(layer.block_sizes):
        n_blocks = (4000 + b - 1) // b
        k = (256 + b - 1) // b
        assert sel[h].tolist() == list(range(k - 1)) + [n_blocks - 1]


@pytest.mark.parametrize("n,T", [(70000, 256), (3000, 512), (5000, 64)])
def test_fused_select_ties(cuda, n, T):
    """Constant keys: every score ties, so the fused selection's filter keeps every block
    as a candidate — past its capacity, which sends the unit through the exact fallback
    (every block scored exactly, radix select); ties go to the lowest block ids and the
    trailing block is forced in."""
    from gpu_util import GpuLayer
    layer = make_layer(5, H=2, G=2, d=128, P=16, block_sizes=(16, 32), seq_lens=(n,))
    layer.k_pool[:] = 0x3F80
    gl = GpuLayer(layer, T)
    gl.decode()
    for h, b in enumerate(layer.block_sizes):
        n_blocks = (n + b - 1) // b
        k = (T + b - 1) // b
        assert gl.step_selection[0][h].tolist() == list(range(k - 1)) + [n_blocks - 1]


@pytest.mark.parametrize("tied", [600, 1500, 2500])
def test_fused_select_large_candidate_sets(cuda, tied):
    """A group of `tied` identical blocks outscores the rest (K = 512 of 10,000 blocks,
    candidate capacity 2048): every group member is a candidate, so the finalize ranks
    600 (register bitonic sort of 1024), 1500 (of 2048) or — past the capacity — runs
    the exact fallback. The K - 1 lowest-indexed group blocks win, then the trailing block."""
    from gpu_util import GpuLayer
    n, P, b0, G = 40000, 4, 100, 2
    rng = np.random.default_rng(tied)
    pool_pages = n // P + 3
    kf = (rng.standard_normal((2, pool_pages, P, 128)) * 0.05).astype(np.float32)
    vf = rng.standard_normal((2, pool_pages, P, 128)).astype(np.float32)
    layer = make_layer(9, H=2, G=G, d=128, P=P, block_sizes=(4,), seq_lens=(n,), kv=(kf, vf),
                       q=np.ones((1, 2 * G, 128), np.float32))
    kf = layer.k_pool  # bf16 bits [H][pages][P][d]
    for t in range(4 * b0, 4 * (b0 + tied)):
        kf[:, layer.page_table[0, t // P], t % P, :] = 0x3F80  # 1.0
    gl = GpuLayer(layer, 2048)
    sel = gl.select()
    gl.decode()
    _, _, want_sel, _ = oracle_step(layer, 0, 2048)
    for h in range(2):
        assert want_sel[h].tolist() == list(range(b0, b0 + 511)) + [n // 4 - 1], h
        assert np.array_equal(sel[0][h], want_sel[h]), h
        assert np.array_equal(gl.step_selection[0][h], want_sel[h]), ("decode step", h)


def test_filter_error_bound(cuda):
    """select.cu's premise: |S_i - C_u - A_i| <= E per unit (with room to spare), so the
    candidate set provably contains the exact top-K."""
    from gpu_util import GpuLayer
    for scale in (0.05, 1.0, 20.0):
        layer = make_layer(11, H=8, G=4, d=128, P=16, seq_lens=(9000, 3000), scale=scale)
        gl = GpuLayer(layer, 1024)
        gl.select()
        exact = [gl.da.download_scores(0, b) for b in range(layer.batch)]
        gl.da.set_filter_diagnostics(0, True)
        gl.decode()
        for b in range(layer.batch):
            approx, err = gl.da.download_filter_scores(0, b)
            off = np.concatenate([[0], np.cumsum([(n + bs - 1) // bs for n, bs in
                                                  zip([layer.seq_lens[b]] * layer.H, layer.block_sizes)])])
            for h in range(layer.H):
                # the trailing block is scored exactly, never filtered: [off, off + N - 1)
                a, e = approx[off[h]:off[h + 1] - 1], exact[b][off[h]:off[h + 1] - 1]
                dev = e.astype(np.float64) - a
                spread = dev.max() - dev.min()  # = 2 max |S - C - A| for the best C
                assert spread <= 2 * err[h], (scale, b, h, spread, err[h])
                assert spread <= err[h], (scale, b, h, spread, err[h])  # room to spare
                # the bound is meaningful: well below the spread of the scores
                assert err[h] < 0.05 * (e.max() - e.min()), (scale, b, h, err[h])


def test_topk_register_classes(cuda):
    """Block sizes 4..64 on a 70K-token sequence: units of 17,500 down to 1,094 blocks run as
    separate top-k register classes (64 keys per thread down to 4); selections and outputs
    against the oracle."""
    from gpu_util import GpuLayer, within_tol
    layer = make_layer(77, H=5, G=2, d=128, P=4, block_sizes=(4, 8, 16, 32, 64), seq_lens=(70000, 30000))
    gl = GpuLayer(layer, 2048)
    sel = gl.select()
    out = gl.decode()
    for b in range(layer.batch):
        _, _, want_sel, want = oracle_step(layer, b, 2048)
        for h in range(layer.H):
            assert np.array_equal(sel[b][h], want_sel[h]), (b, h)
            assert np.array_equal(gl.step_selection[b][h], want_sel[h]), ("decode step", b, h)
        ok, err = within_tol(out[b], want)
        assert ok, f"seq {b}: max abs err {err}"


@pytest.mark.parametrize("exact_select", [False, True])
def test_decode_step_selection_many_seeds(cuda, exact_select):
    """The decode step's selection (select.cu's fused filter + exact refine, or the exact
    scorer + top-k) against the oracle's exact top-K on many units with score
    distributions of different widths (key scales 0.01 .. 10)."""
    from gpu_util import GpuLayer
    for seed, scale in enumerate((0.01, 0.3, 1.0, 10.0)):
        layer = make_layer(100 + seed, H=8, G=4, d=128, P=16, seq_lens=(20000, 7777, 513), scale=scale)
        gl = GpuLayer(layer, 2048, exact_select=exact_select)
        gl.decode()
        for b in range(layer.batch):
            _, _, want_sel, _ = oracle_step(layer, b, 2048)
            for h in range(layer.H):
                assert np.array_equal(gl.step_selection[b][h], want_sel[h]), (scale, b, h)


def test_block_to_pages_through_attend(cuda):
    """test_kv_cache.cpp:86-111 through the C ABI: zero keys (uniform weights) and value rows
    holding their physical page id; block 5 at B=32/P=16 reads pages 10,11 -> 10.5; the
    trailing block 3 of n=100 reads 4 rows of page 6 -> 6."""
    from gpu_util import GpuLayer
    from oracle.oracle import f32_to_bf16
    P, d, pages = 16, 64, 13
    vf = np.broadcast_to(np.arange(pages, dtype=np.float32)[None, :, None, None], (1, pages, P, d)).copy()
    for n, blk, want in ((192, 5, 10.5), (100, 3, 6.0)):
        layer = make_layer(1, H=1, G=1, d=d, P=P, block_sizes=(32,), seq_lens=(n,))
        layer.k_pool = np.zeros((1, pages, P, d), np.uint16)
        layer.v_pool = f32_to_bf16(vf)
        layer.page_table = np.zeros((1, pages), np.uint32)
        layer.page_table[0] = np.arange(pages)
        gl = GpuLayer(layer, 64)
        out = gl.attend([[np.array([blk], np.uint32)]])
        assert out[0, 0, 0] == pytest.approx(want, abs=1e-6)


def test_error_semantics(cuda):
    from gpu_util import GpuLayer
    from paper_2605_12110_b200 import (BlockAssignment, CapacityError, DecodeAttention, EngineConfig,
                                       InvalidArgument, LogicError, OutOfRange, QuantSpec)
    cfg = EngineConfig(num_heads=2, head_dim=64, page_size=16, candidate_block_sizes=(16, 32), token_budget=64,
                       quant=QuantSpec(), max_batch=2, max_seq_len=256)
    da = DecodeAttention(cfg)
    with pytest.raises(InvalidArgument):
        da.set_assignment(0, BlockAssignment([16, 48]))
    with pytest.raises(OutOfRange):
        da.set_assignment(1, BlockAssignment([16, 32]))
    k = torch.zeros(2, 40, 16, 64, dtype=torch.int16, device="cuda")
    pt = torch.zeros(2, 20, dtype=torch.int32, device="cuda")
    with pytest.raises(LogicError):
        da.bind(0, k, k, pt, [100, 100])
    da.set_assignment(0, BlockAssignment([16, 32]))
    with pytest.raises(CapacityError):
        da.bind(0, k, k, pt, [300, 10])
    with pytest.raises(InvalidArgument):
        da.bind(0, k, k, pt, [0, 10])
    da.bind(0, k, k, pt, [100, 10])
    q = torch.zeros(2, 2, 64, dtype=torch.int16, device="cuda")
    out = torch.zeros(2, 2, 64, dtype=torch.float32, device="cuda")
    with pytest.raises(LogicError):
        da.decode_step(0, q, out)
    da.build_store(0)
    da.decode_step(0, q, out)
    torch.cuda.synchronize()
    # zero query and zero keys: uniform weights over the selected rows of zero values
    assert torch.all(out == 0)


def test_decode_step_host_matches_device(cuda):
    from gpu_util import GpuLayer
    layer = make_layer(11, H=8, G=4, d=128, P=16, seq_lens=(6000, 7000))
    gl = GpuLayer(layer, 1024)
    dev = gl.decode()
    q_host = torch.from_numpy(layer.q.view(np.int16)).pin_memory()
    out_host = torch.empty(dev.shape, dtype=torch.float32).pin_memory()
    gl.da.decode_step_host(0, q_host, out_host)  # captured into a graph on first use
    assert np.array_equal(out_host.numpy(), dev)
    # other host buffers: the graph's copy nodes are re-pointed
    q2 = q_host.clone().pin_memory()
    out2 = torch.zeros(dev.shape, dtype=torch.float32).pin_memory()
    gl.da.decode_step_host(0, q2, out2)
    assert np.array_equal(out2.numpy(), dev)
    # pageable host memory
    out3 = torch.zeros(dev.shape, dtype=torch.float32)
    gl.da.decode_step_host(0, torch.from_numpy(layer.q.view(np.int16).copy()), out3)
    assert np.array_equal(out3.numpy(), dev)
    # back to pinned buffers (the attention writes pinned output directly)
    out_host.zero_()
    gl.da.decode_step_host(0, q_host, out_host)
    assert np.array_equal(out_host.numpy(), dev)
    # mixed: pinned q (read by the selection kernel itself) with pageable output, and
    # pageable q with pinned output; then several steps in a row on the same graph
    out4 = torch.zeros(dev.shape, dtype=torch.float32)
    gl.da.decode_step_host(0, q2, out4)
    assert np.array_equal(out4.numpy(), dev)
    out_host.zero_()
    gl.da.decode_step_host(0, torch.from_numpy(layer.q.view(np.int16).copy()), out_host)
    assert np.array_equal(out_host.numpy(), dev)
    for _ in range(3):
        out_host.zero_()
        gl.da.decode_step_host(0, q_host, out_host)
        assert np.array_equal(out_host.numpy(), dev)


def test_synthetic_generator_matches_host_twin(cuda):
    from oracle.synth import synth_bf16
    from paper_2605_12110_b200 import fill_synthetic_bf16
    t = torch.empty(1 << 20, dtype=torch.int16, device="cuda")
    fill_synthetic_bf16(t, 42, 5)
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy().view(np.uint16), synth_bf16(1 << 20, 42, 5))


def test_full_size_128k_sequence(cuda):
    """Config-3 scale for one sequence (128K tokens, 8 KV heads x G=4, d=128, B in {16,32,64},
    T=2048): store/scores/selection bit-exact and output in tolerance vs the C oracle."""
    from gpu_util import GpuLayer, within_tol
    n = 131072
    layer = make_layer(128, H=8, G=4, d=128, P=16, block_sizes=(16, 32, 64), seq_lens=(n,), extra_pages=0)
    gl = GpuLayer(layer, 2048)
    sel = gl.select()[0]
    out = gl.decode()[0]
    seq, sc, want_sel, want = oracle_step(layer, 0, 2048)
    st = gl.da.download_store(0, 0)
    assert np.array_equal(st["codes"], seq.codes)
    assert np.array_equal(_bits(gl.da.download_scores(0, 0)), _bits(sc))
    for h in range(8):
        assert np.array_equal(sel[h], want_sel[h])
    ok, err = within_tol(out, want)
    assert ok, err
