"""GPU calibration (absp_profile_sample: dense fp64 oracle + per-candidate store, selection and
recall on the GPU) against the unmodified reference's profile_sensitivity / transfer_check /
assign_block_sizes (calibrator.cpp:73-224) on the same traces (the reference's own synthetic
workload generator, values rounded to bf16 so both sides see identical inputs):

  recall table, adaptive / uniform recalls : |got - want| <= 1e-9 (selections are bit-exact;
                                             the fp64 weight sums run in another order)
  assignments, matched candidate           : equal
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle.oracle import (f32_to_bf16, bf16_to_f32, ref_assign_block_sizes, ref_available,  # noqa: E402
                           ref_generate_synthetic, ref_profile_sensitivity, ref_transfer_check)

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def _bf16(x):
    return bf16_to_f32(f32_to_bf16(np.asarray(x, np.float32)))


def _samples(S, n, H, d, seed0):
    profiles = [("clustered", 2, 48), ("scattered", n // 128), ("clustered", 4, 16), ("uniform",)]
    profiles = [profiles[h % len(profiles)] for h in range(H)]
    ks, vs, qs = [], [], []
    for s in range(S):
        k, v, q = ref_generate_synthetic(n, H, d, profiles, signal=8.0, seed=seed0 + s)
        ks.append(_bf16(k))
        vs.append(_bf16(v))
        qs.append(_bf16(q))
    return np.stack(ks), np.stack(vs), np.stack(qs)


@needs_ref
@pytest.mark.parametrize("d,P,cands,T,n,bits", [
    (64, 8, (8, 16, 32), 256, 3000, 4),
    (128, 16, (16, 32, 64), 512, 4100, 4),
    (64, 4, (4, 8, 16), 128, 2500, 0),   # full-precision store (quant = nullopt)
])
def test_profile_sensitivity_and_transfer_vs_reference(cuda, d, P, cands, T, n, bits):
    from paper_2605_12110_b200 import (EngineConfig, QuantSpec, Trace, assign_block_sizes,
                                       profile_sensitivity, transfer_check)
    H, S = 4, 2
    k, v, q = _samples(S, n, H, d, seed0=d + P)
    cfg = EngineConfig(num_heads=H, head_dim=d, page_size=P, candidate_block_sizes=cands, token_budget=T,
                       quant=QuantSpec(bits) if bits else None)
    provider = lambda i: Trace(H, d, n, i, k[i], v[i], q[i])  # noqa: E731
    table = profile_sensitivity(provider, S, cfg)
    want = ref_profile_sensitivity(k, v, q, P, cands, T, bits=bits)
    assert table.sample_count == S
    assert np.all(np.abs(table.recalls - want) <= 1e-9), (table.recalls, want)
    for tau in (0.9, 0.98):
        a = assign_block_sizes(table, tau)
        assert a.block_sizes == ref_assign_block_sizes(want, cands, tau)
    a = assign_block_sizes(table, 0.9)
    rep = transfer_check(a, provider, S, cfg)
    ref = ref_transfer_check(a.block_sizes, k, v, q, P, cands, T, bits=bits)
    assert abs(rep.adaptive_recall - ref["adaptive_recall"]) <= 1e-9
    assert np.all(np.abs(np.array(rep.uniform_recalls) - np.array(ref["uniform_recalls"])) <= 1e-9)
    assert rep.matched_candidate == ref["matched_candidate"]
    assert abs(rep.delta - ref["delta"]) <= 1e-9
    assert abs(rep.avg_block_size - ref["avg_block_size"]) <= 1e-12


@needs_ref
def test_profile_sensitivity_skips_short_traces(cuda):
    from paper_2605_12110_b200 import EngineConfig, QuantSpec, Trace, profile_sensitivity
    H, d, n = 4, 64, 200
    k, v, q = _samples(1, n, H, d, seed0=3)
    cfg = EngineConfig(num_heads=H, head_dim=d, page_size=8, candidate_block_sizes=(8, 16), token_budget=256,
                       quant=QuantSpec(4))
    with pytest.raises(RuntimeError, match="no usable samples"):
        profile_sensitivity(lambda i: Trace(H, d, n, i, k[0], v[0], q[0]), 1, cfg)
