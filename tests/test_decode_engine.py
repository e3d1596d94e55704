"""DecodeEngine::step (engine.cpp:442-463) on the GPU against the reference's own DecodeEngine
(oracle/_ref, the unmodified reference core): prefill, then decode steps that append a token,
refresh the tail centroid, requantize every head, select and attend.

  store (centroids, codes, scales, zero points) after every step : bit-exact
  ordered selection                                               : bit-exact
  output                                                          : |got-want| <= 1e-3 + 1e-2|want|
     (the reference falls back to fp64 full attention while seq_len <= T; every block is
      selected then, so the sparse output is that attention up to fp32 rounding)
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _bf16_values(rng, shape, scale=1.0):
    return O.bf16_to_f32(O.f32_to_bf16((rng.standard_normal(shape) * scale).astype(np.float32)))


@pytest.mark.parametrize("H,d,P,cands,T,n0,steps", [
    (4, 64, 16, (16, 32, 64), 256, 200, 90),     # crosses T (fallback -> sparse) and block boundaries
    (8, 128, 8, (8, 16, 32), 512, 1000, 40),     # cfg-1-like heads, P = 8
    (4, 128, 8, (8, 24, 40), 256, 230, 60),      # block sizes that do not divide the attention chunk
    (4, 128, 4, (4, 8, 16), 256, 300, 50),       # P = 4: four attention producer warps
])
def test_engine_steps_match_reference(cuda, H, d, P, cands, T, n0, steps):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    from gpu_util import within_tol
    from paper_2605_12110_b200 import BlockAssignment, DecodeEngine, EngineConfig, QuantSpec
    rng = np.random.default_rng(n0 + H)
    bs = [cands[h % len(cands)] for h in range(H)]
    cap = n0 + steps + 7
    cfg = EngineConfig(num_heads=H, head_dim=d, page_size=P, candidate_block_sizes=cands, token_budget=T,
                       quant=QuantSpec(4))
    eng = DecodeEngine(cfg, BlockAssignment(bs), cap)
    ref = O.RefEngine(H, d, P, cands, T, bs, cap)
    keys = _bf16_values(rng, (H, n0, d))
    vals = _bf16_values(rng, (H, n0, d))
    eng.prefill(keys, vals, n0)
    ref.prefill(keys, vals, n0)
    for step in range(steps):
        k, v, q = (_bf16_values(rng, (H, d)) for _ in range(3))
        got = eng.step(k, v, q)
        want, want_sel, fb = ref.step(k, v, q)
        assert got.full_attention_fallback == fb
        for h in range(H):
            assert np.array_equal(got.selection[h], want_sel[h]), (step, h)
        ok, err = within_tol(got.output, want)
        assert ok, (step, err)
        if True:  # every step: maintenance is incremental, so any drift would show at once
            st = eng.da.download_store(0, 0)
            rs = ref.store()
            assert np.array_equal(st["offsets"], rs["offsets"]), step
            assert np.array_equal(st["values"].view(np.uint32), rs["values"].view(np.uint32)), step
            assert np.array_equal(st["codes"], rs["codes"]), step
            assert np.array_equal(st["scales"].view(np.uint32), rs["scales"].view(np.uint32)), step
            assert np.array_equal(st["zps"].view(np.uint32), rs["zps"].view(np.uint32)), step


def _signed_zero_keys(rng, H, n, d, n0):
    """Channel 0 >= 0 with whole blocks of -0.0 and +0.0 keys (a -0.0 / +0.0 mean centroid ties
    the channel minimum: std::min keeps the earlier one); channel 1 the other way round."""
    x = _bf16_values(rng, (H, n, d))
    x[:, :, 0] = np.abs(x[:, :, 0])
    x[:, :, 1] = np.abs(x[:, :, 1])
    x[:, 64:128, 0] = -0.0
    x[:, 192:256, 0] = 0.0
    x[:, 64:128, 1] = 0.0
    x[:, 192:256, 1] = -0.0
    x[:, n0 + 5:n0 + 40, 0] = -0.0   # decode-time blocks of zeros too
    x[:, n0 + 5:n0 + 40, 1] = 0.0
    return x


@pytest.mark.parametrize("method,bits,mode,zeros", [
    (0, 4, 1, True), (0, 4, 0, True), (1, 8, 0, False), (1, 2, 1, True), (0, 8, 1, False), (0, 0, 1, False),
])
def test_engine_maintenance_grid(cuda, method, bits, mode, zeros):
    """Incremental requantization (frozen statistics + changed-word re-encode) against the
    reference's requantize-everything step, over the QuantSpec grid, both centroid methods
    and signed-zero ties; the store is compared after every step."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    from gpu_util import within_tol
    from paper_2605_12110_b200 import BlockAssignment, CentroidMethod, DecodeEngine, EngineConfig, QuantMode, QuantSpec
    H, d, P, cands, T, n0, steps = 4, 64, 4, (4, 8, 16), 128, 300, 48
    rng = np.random.default_rng(11 + 3 * bits + method + 7 * mode)
    bs = [cands[h % len(cands)] for h in range(H)]
    cap = n0 + steps + 3
    cfg = EngineConfig(num_heads=H, head_dim=d, page_size=P, candidate_block_sizes=cands, token_budget=T,
                       centroid_method=CentroidMethod(method),
                       quant=QuantSpec(bits, QuantMode(mode)) if bits else None)
    eng = DecodeEngine(cfg, BlockAssignment(bs), cap)
    ref = O.RefEngine(H, d, P, cands, T, bs, cap, method=method, bits=bits, mode=mode)
    keys = _signed_zero_keys(rng, H, cap, d, n0) if zeros else _bf16_values(rng, (H, cap, d))
    vals = _bf16_values(rng, (H, cap, d))
    eng.prefill(keys[:, :n0], vals[:, :n0], n0)
    ref.prefill(keys[:, :n0], vals[:, :n0], n0)
    for step in range(steps):
        k, v = keys[:, n0 + step], vals[:, n0 + step]
        q = _bf16_values(rng, (H, d))
        got = eng.step(k, v, q)
        want, want_sel, fb = ref.step(k, v, q)
        for h in range(H):
            assert np.array_equal(got.selection[h], want_sel[h]), (step, h)
        ok, err = within_tol(got.output, want)
        assert ok, (step, err)
        st = eng.da.download_store(0, 0)
        rs = ref.store()
        assert np.array_equal(st["values"].view(np.uint32), rs["values"].view(np.uint32)), step
        if bits:
            assert np.array_equal(st["codes"], rs["codes"]), step
            assert np.array_equal(st["scales"].view(np.uint32), rs["scales"].view(np.uint32)), step
            assert np.array_equal(st["zps"].view(np.uint32), rs["zps"].view(np.uint32)), step


def test_engine_errors(cuda):
    from paper_2605_12110_b200 import (BlockAssignment, CapacityError, DecodeEngine, EngineConfig, InvalidArgument,
                                       LogicError, QuantSpec)
    cfg = EngineConfig(num_heads=2, head_dim=64, page_size=16, candidate_block_sizes=(16, 32), token_budget=64,
                       quant=QuantSpec(4))
    eng = DecodeEngine(cfg, BlockAssignment([16, 32]), 40)
    z = np.zeros((2, 64), np.float32)
    with pytest.raises(LogicError):
        eng.step(z, z, z)
    with pytest.raises(InvalidArgument):
        eng.prefill(np.zeros((2, 10, 64), np.float32), np.zeros((2, 10, 64), np.float32), 0)
    eng.prefill(np.ones((2, 38, 64), np.float32), np.ones((2, 38, 64), np.float32), 38)
    with pytest.raises(LogicError):
        eng.prefill(np.ones((2, 38, 64), np.float32), np.ones((2, 38, 64), np.float32), 38)
    eng.step(z, z, z)
    eng.step(z, z, z)
    with pytest.raises(CapacityError):  # kv_cache.cpp:48-50
        eng.step(z, z, z)
