"""The reference's own known-answer tests (proj/tests/*.cpp), re-expressed against the
C restatement in oracle/ — pinning the oracle before it is trusted as the checker."""
import numpy as np
import pytest

from oracle.oracle import OracleSeq, f32_to_bf16, lib

F32 = np.float32


def _pool_from_rows(rows, P):
    """One head, rows [n][d] fp32 -> pool [1][pages][P][d] with identity page table."""
    rows = np.asarray(rows, F32)
    n, d = rows.shape
    pages = (n + P - 1) // P
    pool = np.zeros((1, pages, P, d), F32)
    pool.reshape(1, pages * P, d)[0, :n] = rows
    return f32_to_bf16(pool), np.arange(pages, dtype=np.uint32)


def _quant(values, offsets, H, d, bits, mode):
    values = np.ascontiguousarray(values, F32)
    codes = np.zeros(values.shape, np.uint8)
    sc = np.zeros((H, d), F32)
    zp = np.zeros((H, d), F32)
    assert lib().absp_oracle_quantize(values, np.asarray(offsets, np.uint64), H, d, bits, mode, codes, sc, zp) == 0
    return codes, sc, zp


def _deq(code, sc, zp, bits, mode):
    if mode == 1:
        return F32(zp + F32(code) * sc)
    mid = (1 << (bits - 1)) - 1
    return F32(F32(int(code) - mid) * sc)


def test_int4_asym_formula_kat():
    # test_quantizer.cpp:50-60: channel {-1, 0.5, 2} -> scale 0.2, zp -1, code 8, deq 0.6
    codes, sc, zp = _quant([[-1.0], [0.5], [2.0]], [0, 3], 1, 1, 4, 1)
    assert sc[0, 0] == pytest.approx(0.2, rel=1e-6)
    assert sc[0, 0] == F32(3.0) / F32(15.0)
    assert zp[0, 0] == -1.0
    assert codes[1, 0] == 8
    rec = _deq(codes[1, 0], sc[0, 0], zp[0, 0], 4, 1)
    assert rec == pytest.approx(0.6, rel=1e-6)
    assert abs(rec - 0.5) <= sc[0, 0] / 2 + 1e-6


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("mode", [0, 1])
def test_constant_channel_exact(bits, mode):
    # test_quantizer.cpp:62-72
    codes, sc, zp = _quant([[0.7]] * 4, [0, 4], 1, 1, bits, mode)
    for i in range(4):
        assert _deq(codes[i, 0], sc[0, 0], zp[0, 0], bits, mode) == F32(0.7)


@pytest.mark.parametrize("method", [0, 1])
def test_error_bound_code_range_determinism(method):
    # test_quantizer.cpp:74-124
    rng = np.random.default_rng(5)
    H, d, P, n = 3, 6, 16, 300
    pool = f32_to_bf16(rng.standard_normal((H, 19, P, d)).astype(F32))
    seq = OracleSeq(pool, pool, np.arange(19, dtype=np.uint32), n, H, d, P, [16, 32, 64], method, 0)
    for bits in (2, 4, 8):
        for mode in (0, 1):
            codes, sc, zp = _quant(seq.values, seq.offsets, H, d, bits, mode)
            codes2, sc2, zp2 = _quant(seq.values, seq.offsets, H, d, bits, mode)
            assert np.array_equal(codes, codes2) and np.array_equal(sc, sc2) and np.array_equal(zp, zp2)
            maxc = (1 << bits) - 1 if mode == 1 else 2 * ((1 << (bits - 1)) - 1)
            assert codes.max() <= maxc
            if mode == 0:
                assert np.all(zp == 0) and np.all(sc > 0)
            for h in range(H):
                for i in range(int(seq.offsets[h]), int(seq.offsets[h + 1])):
                    for c in range(d):
                        y = _deq(codes[i, c], sc[h, c], zp[h, c], bits, mode)
                        assert abs(seq.values[i, c] - y) <= sc[h, c] / 2 + 1e-6


def test_mean_and_maxmin_centroid_kats():
    # test_centroids.cpp:25-42
    pool, pt = _pool_from_rows([[1.0, 3.0], [3.0, 1.0]], 2)
    mean = OracleSeq(pool, pool, pt, 2, 1, 2, 2, [2], 0, 0)
    assert mean.values.tolist() == [[2.0, 2.0]]
    mm = OracleSeq(pool, pool, pt, 2, 1, 2, 2, [2], 1, 0)
    assert mm.values.tolist() == [[3.0, 3.0]]
    assert mm.values_min.tolist() == [[1.0, 1.0]]


def test_block_size_one_reproduces_keys():
    # test_centroids.cpp:44-56
    rng = np.random.default_rng(5)
    pool = f32_to_bf16(rng.standard_normal((2, 37, 1, 4)).astype(F32))
    seq = OracleSeq(pool, pool, np.arange(37, dtype=np.uint32), 37, 2, 4, 1, [1, 1], 0, 0)
    keys = seq.keys_logical()
    assert np.array_equal(seq.values.reshape(2, 37, 4), keys)


def test_offsets_kat():
    # test_centroids.cpp:65-82
    out = np.zeros(4, np.uint64)
    lib().absp_oracle_offsets(128, np.array([32, 64, 16], np.uint32), 3, out)
    assert out.tolist() == [0, 4, 6, 14]
    lib().absp_oracle_offsets(0, np.array([32, 64, 16], np.uint32), 3, out)
    assert out.tolist() == [0, 0, 0, 0]
    out2 = np.zeros(2, np.uint64)
    lib().absp_oracle_offsets(100, np.array([32], np.uint32), 1, out2)
    assert out2.tolist() == [0, 4]


def _select(scores, offsets, bs, n, T, max_k=64):
    blocks = np.zeros((len(bs), max_k), np.uint32)
    counts = np.zeros(len(bs), np.uint32)
    budgets = np.zeros(len(bs), np.uint32)
    rc = lib().absp_oracle_select(np.asarray(scores, F32), np.asarray(offsets, np.uint64),
                                  np.asarray(bs, np.uint32), len(bs), n, T, blocks, max_k, counts,
                                  budgets.ctypes.data)
    assert rc == 0
    return [blocks[h, :counts[h]].tolist() for h in range(len(bs))], budgets.tolist()


def test_hand_scores_and_trailing_block_kats():
    # test_engine.cpp:131-142: flattened per-head segments
    vals = np.array([[1, 0], [0, 1], [2, 0]], F32)
    sc = np.zeros(3, F32)
    lib().absp_oracle_scores_f32(np.array([1, 0, 1, 0], F32), vals, None, np.array([0, 2, 3], np.uint64), 2, 2, 0, sc)
    assert sc.tolist() == [1.0, 0.0, 2.0]
    # test_engine.cpp:203-220: K = 2, trailing block kept / displacing the weakest pick
    sel, _ = _select([1.0, 0.0, 2.0], [0, 3], [16], 48, 32)
    assert sel == [[2, 0]]
    sel, _ = _select([1.0, 2.0, -5.0], [0, 3], [16], 48, 32)
    assert sel == [[1, 2]]


def test_budget_is_ceil_T_over_B():
    # test_engine.cpp:186-201
    offs = [0, 256, 384]
    sel, budgets = _select(np.random.default_rng(1).standard_normal(384).astype(F32), offs, [32, 64], 8192, 4096,
                           max_k=256)
    assert budgets == [128, 64]
    assert [len(s) for s in sel] == [128, 64]


def _sort_oracle(scores, n_blocks, k):
    idx = sorted(range(n_blocks), key=lambda i: (-float(scores[i]), i))
    if n_blocks > k:
        idx = idx[:k]
        if n_blocks - 1 not in idx:
            idx[-1] = n_blocks - 1
    return idx


def test_selection_equals_full_sort_oracle_with_forced_ties():
    # test_engine.cpp:222-256 (25 random trials, forced ties at 0.25)
    rng = np.random.default_rng(24)
    for _ in range(25):
        H = 1 + rng.integers(4)
        bs = [int(rng.choice([16, 32, 64])) for _ in range(H)]
        n = 64 + int(rng.integers(2000))
        T = 64 + int(rng.integers(512))
        offs = [0]
        for b in bs:
            offs.append(offs[-1] + (n + b - 1) // b)
        scores = rng.standard_normal(offs[-1]).astype(F32)
        scores[rng.integers(4, size=offs[-1]) == 0] = 0.25
        sel, budgets = _select(scores, offs, bs, n, T, max_k=128)
        for h in range(H):
            seg = scores[offs[h]:offs[h + 1]]
            want = _sort_oracle(seg, len(seg), budgets[h])
            got = sel[h]
            assert set(got) == set(want)
            assert len(set(got)) == len(got)
            assert (len(seg) - 1) in got
            # ordered by (score desc, index asc); the trailing block sits at its own key
            keys = [(-float(seg[i]), i) for i in got]
            assert keys == sorted(keys)


def test_signed_zero_ties():
    # -0.0 == +0.0 under the reference's `!=` comparison: ties break to the lower index
    sel, _ = _select([0.0, -0.0, 0.0, -0.0, 1.0], [0, 5], [16], 80, 32)
    assert sel == [[4, 0]]


def test_full_coverage_matches_full_attention():
    # test_engine.cpp:282-294
    rng = np.random.default_rng(27)
    H, d, P, n = 4, 16, 16, 500
    kp = f32_to_bf16(rng.standard_normal((H, 32, P, d)).astype(F32))
    vp = f32_to_bf16(rng.standard_normal((H, 32, P, d)).astype(F32))
    seq = OracleSeq(kp, vp, np.arange(32, dtype=np.uint32), n, H, d, P, [16, 32, 64, 16], 0, 0)
    q = rng.standard_normal((H, d)).astype(F32)
    sel = seq.select(seq.scores(q), 512)
    got = seq.attend(q, sel)
    want = seq.full_attention(q)
    scale = np.maximum(np.abs(want).max(axis=1, keepdims=True), 1e-12)
    assert (np.abs(got - want) / scale).max() < 1e-5


def test_identical_value_rows_return_that_value():
    # test_engine.cpp:296-318
    rng = np.random.default_rng(29)
    d = 4
    v = np.array([0.5, -1.0, 2.0, 0.25], F32)
    kp = f32_to_bf16(rng.standard_normal((1, 4, 16, d)).astype(F32))
    vp = f32_to_bf16(np.broadcast_to(v, (1, 4, 16, d)).copy())
    seq = OracleSeq(kp, vp, np.arange(4, dtype=np.uint32), 32, 1, d, 16, [32], 0, 0)
    out = seq.attend(rng.standard_normal((1, d)).astype(F32), [np.array([0], np.uint32)])
    assert np.allclose(out[0], v, rtol=1e-6)


def test_block_to_pages_stride_kats():
    # test_kv_cache.cpp:86-111: block 5 at B=32,P=16 spans pages 10,11; trailing block 3 of n=100 -> page 6, 4 rows.
    # Keys are zero (uniform weights) and every value row holds its physical page id, so the
    # attention output over one block is the mean page id of the rows it read.
    d, P = 4, 16
    pages = 12
    kp = np.zeros((1, pages, P, d), np.uint16)
    vf = np.broadcast_to(np.arange(pages, dtype=F32)[None, :, None, None], (1, pages, P, d)).copy()
    vp = f32_to_bf16(vf)
    pt = np.arange(pages, dtype=np.uint32)
    seq = OracleSeq(kp, vp, pt, 192, 1, d, P, [32], 0, 0)
    out = seq.attend(np.zeros((1, d), F32), [np.array([5], np.uint32)])
    assert out[0, 0] == pytest.approx(10.5)
    seq = OracleSeq(kp, vp, pt, 100, 1, d, P, [32], 0, 0)
    out = seq.attend(np.zeros((1, d), F32), [np.array([3], np.uint32)])
    assert out[0, 0] == 6.0
    # B == P is the identity mapping
    seq = OracleSeq(kp, vp, pt, 192, 1, d, P, [16], 0, 0)
    out = seq.attend(np.zeros((1, d), F32), [np.array([0], np.uint32)])
    assert out[0, 0] == 0.0
