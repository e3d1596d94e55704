"""Oracle pinning: the C restatement reproduces the reference's committed outputs
(tests/golden/golden_v1.npz, written by tests/golden/make_golden.py from the
unmodified reference) bit for bit, and — when the reference core is built here —
agrees with it live on fresh random inputs."""
from pathlib import Path

import numpy as np
import pytest

from golden.make_golden import CASES, case_inputs
from oracle import oracle as O

GOLDEN = Path(__file__).parent / "golden" / "golden_v1.npz"


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_matches_golden(golden, name):
    c = case_inputs(name)
    seq = O.OracleSeq(c["k_pool"], c["v_pool"], c["page_table"], c["n"], c["H"], c["d"], c["P"],
                      c["block_sizes"], c["method"], c["bits"], c["mode"])
    g = lambda k: golden[f"{name}/{k}"]
    assert np.array_equal(seq.offsets, g("offsets"))
    assert np.array_equal(_bits(seq.values), _bits(g("values")))
    if c["method"] == 1:
        assert np.array_equal(_bits(seq.values_min), _bits(g("values_min")))
    if c["bits"]:
        assert np.array_equal(seq.codes, g("codes"))
        assert np.array_equal(_bits(seq.scales), _bits(g("scales")))
        assert np.array_equal(_bits(seq.zps), _bits(g("zps")))
        if c["method"] == 1:
            assert np.array_equal(seq.codes_min, g("codes_min"))
    qf = O.bf16_to_f32(c["q"])
    sc, sel, out = O.oracle_decode(seq, qf, c["G"], c["T"])
    assert np.array_equal(_bits(sc), _bits(g("scores")))
    assert np.array_equal(np.array([len(s) for s in sel], np.uint32), g("sel_counts"))
    assert np.array_equal(np.concatenate(sel), g("sel_blocks"))
    assert np.array_equal(_bits(out), _bits(g("attn_out")))
    H, G, d = c["H"], c["G"], c["d"]
    full = np.zeros_like(qf)
    for gg in range(G):
        full.reshape(H, G, d)[:, gg] = seq.full_attention(np.ascontiguousarray(qf.reshape(H, G, d)[:, gg]))
    assert np.array_equal(_bits(full), _bits(g("full_out")))


@pytest.mark.skipif(not O.ref_available(), reason="reference core not built here (make -C oracle ref)")
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_matches_live_reference(seed):
    from layer_data import make_layer
    rng = np.random.default_rng(seed)
    H = int(rng.integers(1, 6))
    P = int(rng.choice([1, 2, 4, 8, 16]))
    cands = sorted({P * int(m) for m in rng.choice([1, 2, 4, 8], size=3)})
    n = int(rng.integers(1, 3000))
    T = int(max(cands) * rng.integers(1, 8))
    method, bits, mode = int(rng.integers(2)), int(rng.choice([0, 2, 4, 8])), int(rng.integers(2))
    layer = make_layer(seed, H=H, G=1, d=32, P=P, block_sizes=cands, seq_lens=(n,), scale=float(rng.choice([0.01, 1, 100])))
    seq = layer.oracle_seq(0, method, bits, mode)
    ref = O.RefSeq(seq.keys_logical(), seq.values_logical(), P, layer.block_sizes, method, bits, mode)
    st = ref.store()
    assert np.array_equal(_bits(st["values"]), _bits(seq.values))
    if bits:
        assert np.array_equal(st["codes"], seq.codes)
        assert np.array_equal(_bits(st["scales"]), _bits(seq.scales))
    q = layer.qf(0)
    a, b = seq.scores(q), ref.scores(q)
    assert np.array_equal(_bits(a), _bits(b))
    sa, sb = seq.select(a, T), ref.select(b, T)
    assert all(np.array_equal(x, y) for x, y in zip(sa, sb))
    assert np.array_equal(_bits(seq.attend(q, sa)), _bits(ref.attend(q)))
