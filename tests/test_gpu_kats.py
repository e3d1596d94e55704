"""The reference unit tests' known answers re-expressed through
the GPU C ABI. The reference KATs use head_dim 1..4; this build's kernels take
head_dim 64 or 128, so each KAT's channels are embedded in channel 0..k of a 64-wide
head with the remaining channels zero (they add exact zeros to every sum and quantize
to a constant channel).

  test_quantizer.cpp:50-60   INT4-asym channel {-1, 0.5, 2} -> scale 0.2, zp -1, code 8, deq 0.6
  test_quantizer.cpp:62-72   constant channels reconstruct exactly under every spec
  test_centroids.cpp:25-42   mean [[1,3],[3,1]] -> [2,2]; maxmin -> max [3,3], min [1,1]
  test_centroids.cpp:65-82   offsets {32,64,16} @ 128 -> [0,4,6,14]; {32} @ 100 -> [0,4]
  test_engine.cpp:113-128    K_h = ceil(T / B_h): 128 / 64 at T = 4096
  test_engine.cpp:130-147    hand-sized selections keep the trailing block, ordered by score
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from layer_data import Layer  # noqa: E402
from oracle.oracle import f32_to_bf16  # noqa: E402

D = 64


def _layer(rows, H, P, block_sizes, G=1, q=None):
    """rows: fp32 [H][n][k] keys (k <= D channels); values zero; pages in order."""
    rows = np.asarray(rows, np.float32)
    n = rows.shape[1]
    pages = (n + P - 1) // P
    k = np.zeros((H, pages * P, D), np.float32)
    k[:, :n, :rows.shape[2]] = rows
    v = np.zeros_like(k)
    pt = np.zeros((1, pages + 1), np.uint32)
    pt[0, :pages] = np.arange(pages)
    qf = np.zeros((1, H * G, D), np.float32) if q is None else np.asarray(q, np.float32).reshape(1, H * G, D)
    return Layer(H, G, D, P, list(block_sizes), [n], f32_to_bf16(k.reshape(H, pages, P, D)),
                 f32_to_bf16(v.reshape(H, pages, P, D)), pt, f32_to_bf16(qf))


def _gpu(layer, T, method=0, bits=4, mode=1, cands=None):
    from gpu_util import GpuLayer
    return GpuLayer(layer, T, method, bits, mode, candidates=cands)


def test_int4_asym_formula(cuda):
    # three blocks of one row each (B = P = 1): centroids are the rows
    layer = _layer([[[-1.0], [0.5], [2.0]]], H=1, P=1, block_sizes=(1,))
    gl = _gpu(layer, 4, cands=(1,))
    st = gl.da.download_store(0, 0)
    assert st["scales"][0, 0] == np.float32(3.0) / np.float32(15.0)  # 0.2 as the fp32 division
    assert st["scales"][0, 0] == pytest.approx(0.2, rel=1e-6)
    assert st["zps"][0, 0] == -1.0
    assert st["codes"][1, 0] == 8  # round(1.5 / 0.2)
    deq = np.float32(st["zps"][0, 0]) + np.float32(8) * st["scales"][0, 0]
    assert deq == pytest.approx(0.6, rel=1e-6)
    assert abs(deq - 0.5) <= st["scales"][0, 0] / 2 + 1e-6


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("mode", [0, 1])
def test_constant_channel_exact(cuda, bits, mode):
    layer = _layer([[[0.7]] * 4], H=1, P=1, block_sizes=(1,))
    gl = _gpu(layer, 4, bits=bits, mode=mode, cands=(1,))
    st = gl.da.download_store(0, 0)
    v = (f32_to_bf16(np.float32([0.7])).astype(np.uint32) << 16).view(np.float32)[0]  # bf16(0.7)
    mid = (1 << (bits - 1)) - 1
    for i in range(4):
        c = int(st["codes"][i, 0])
        sc, zp = st["scales"][0, 0], st["zps"][0, 0]
        deq = np.float32(zp + np.float32(c) * sc) if mode == 1 else np.float32(np.float32(c - mid) * sc)
        assert deq == v, (bits, mode, i, deq, v)


@pytest.mark.parametrize("method", [0, 1])
def test_centroid_kats(cuda, method):
    layer = _layer([[[1.0, 3.0], [3.0, 1.0]]], H=1, P=2, block_sizes=(2,))
    gl = _gpu(layer, 2, method=method, bits=0, cands=(2,))
    st = gl.da.download_store(0, 0)
    assert int(st["offsets"][-1]) == 1
    if method == 0:
        assert st["values"][0, 0] == 2.0 and st["values"][0, 1] == 2.0
    else:
        assert st["values"][0, 0] == 3.0 and st["values"][0, 1] == 3.0
        assert st["values_min"][0, 0] == 1.0 and st["values_min"][0, 1] == 1.0


def test_build_offsets(cuda):
    rng = np.random.default_rng(0)
    layer = _layer(rng.standard_normal((3, 128, 4)), H=3, P=16, block_sizes=(32, 64, 16))
    gl = _gpu(layer, 64, cands=(16, 32, 64))
    assert gl.da.download_store(0, 0)["offsets"].tolist() == [0, 4, 6, 14]
    layer = _layer(rng.standard_normal((1, 100, 4)), H=1, P=16, block_sizes=(32,))
    gl = _gpu(layer, 64, cands=(32,))
    assert gl.da.download_store(0, 0)["offsets"].tolist() == [0, 4]


def test_budget_blocks_follow_ceil(cuda):
    rng = np.random.default_rng(22)
    q = np.zeros((2, D), np.float32)
    q[:, :4] = rng.standard_normal((2, 4))
    layer = _layer(rng.standard_normal((2, 8192, 4)), H=2, P=16, block_sizes=(32, 64), q=q)
    gl = _gpu(layer, 4096, bits=0, cands=(16, 32, 64))
    sel = gl.select()[0]
    assert len(sel[0]) == 128 and len(sel[1]) == 64
    assert gl.da.layer_info(0).max_select == 128


@pytest.mark.parametrize("means,want", [((1.0, 0.0, 2.0), [2, 0]), ((1.0, 2.0, -5.0), [1, 2])])
def test_hand_sized_selection(cuda, means, want):
    # one head, B = 16, n = 48: block j's rows all hold means[j] in channel 0; q = e0; T = 32 -> K = 2
    rows = np.repeat(np.asarray(means, np.float32), 16).reshape(1, 48, 1)
    q = np.zeros((1, D), np.float32)
    q[0, 0] = 1.0
    layer = _layer(rows, H=1, P=16, block_sizes=(16,), q=q)
    gl = _gpu(layer, 32, bits=0, cands=(16,))
    assert gl.select()[0][0].tolist() == want
    gl.decode()
    assert gl.step_selection[0][0].tolist() == want
