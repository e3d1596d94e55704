"""GPU parity of the explicit-selection attention entry points (absp_attend,
absp_attend_selected) — the path the benchmark's roofline figure times — against the
C restatement of sparse_attention (engine.cpp:285-327, oracle/absp_oracle.c), plus the
selection validation of check_selection / block_to_pages (engine.cpp:212-232,
kv_cache.cpp:118-138) and regressions for the step's cross-launch protocols.

  attention output : |got - want| <= 1e-3 + 1e-2 |want|  (north-star tolerance)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from layer_data import make_layer, oracle_step  # noqa: E402


def _random_selection(rng, layer, stride_extra, shuffle=True, short=True):
    """Per (b, h): a random subset of distinct valid block ids, random order, random length
    in [1, min(N, K_cap)], the stride larger than any count by `stride_extra`."""
    sel = []
    for b in range(layer.batch):
        row = []
        for h in range(layer.H):
            B = layer.block_sizes[h]
            N = (layer.seq_lens[b] + B - 1) // B
            cap = max(1, min(N, 2048 // B))
            k = int(rng.integers(1, cap + 1)) if short else cap
            ids = rng.choice(N, size=k, replace=False).astype(np.uint32)
            if not shuffle:
                ids.sort()
            row.append(ids)
        sel.append(row)
    stride = max(len(x) for r in sel for x in r) + stride_extra
    return sel, stride


def _oracle_attend(layer, b, sel_b):
    seq = layer.oracle_seq(b)
    qg = layer.qf(b).reshape(layer.H, layer.G, layer.d)
    out = np.zeros((layer.H, layer.G, layer.d), np.float32)
    for g in range(layer.G):
        out[:, g, :] = seq.attend(np.ascontiguousarray(qg[:, g, :]), sel_b)
    return out.reshape(layer.H * layer.G, layer.d)


def _attend(gl, selection, stride):
    from gpu_util import to_dev_u32
    L = gl.layer
    blocks = np.zeros((L.batch, L.H, stride), np.uint32)
    counts = np.zeros((L.batch, L.H), np.uint32)
    for s in range(L.batch):
        for h in range(L.H):
            blocks[s, h, :len(selection[s][h])] = selection[s][h]
            counts[s, h] = len(selection[s][h])
    out = torch.full((L.batch, L.H * L.G, L.d), float("nan"), dtype=torch.float32, device="cuda")
    gl.da.attend(0, gl.q, to_dev_u32(blocks), to_dev_u32(counts), out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("d,G,P,cands,seq_lens,extra", [
    (128, 4, 16, (16, 32, 64), (131072 // 8, 5000, 777), 0),   # cfg 3 block sizes, ragged
    (128, 8, 4, (4, 8, 16, 32, 64), (9001, 3000), 9),         # cfg 5 shape (G=8, P=4)
    (128, 4, 8, (8, 16, 32), (8192,), 33),                    # cfg 1 shape
    (128, 8, 16, (16, 64), (6000, 100, 4097), 1),
    (64, 2, 16, (16, 32), (3000, 20), 5),                     # d = 64
    (128, 1, 4, (4, 16), (2500,), 200),                       # MHA, stride far above counts
    (128, 4, 16, (16, 48, 112), (5000, 700), 3),              # blocks that do not divide the 128-row chunk
    (128, 4, 2, (2, 8, 32), (3001, 515), 7),                  # P = 2: 64 slots, 4 producer warps
    (128, 2, 1, (1, 4, 16), (1500,), 2),                      # P = 1: 128 slots per chunk
    (64, 4, 4, (4, 12, 32), (4099, 64), 11),                  # d = 64 with 4 producer warps
])
def test_attend_random_selections_vs_oracle(cuda, d, G, P, cands, seq_lens, extra):
    from gpu_util import GpuLayer, within_tol
    rng = np.random.default_rng(d * 1000 + G * 100 + P)
    layer = make_layer(int(rng.integers(1 << 30)), H=8, G=G, d=d, P=P, block_sizes=cands, seq_lens=seq_lens)
    gl = GpuLayer(layer, 2048, max_seq_len=max(seq_lens) + 64)
    for trial, (shuffle, short) in enumerate(((True, True), (False, False), (True, False))):
        sel, stride = _random_selection(rng, layer, extra + trial, shuffle, short)
        got = _attend(gl, sel, stride)
        for b in range(layer.batch):
            want = _oracle_attend(layer, b, sel[b])
            ok, err = within_tol(got[b], want)
            assert ok, f"trial {trial} seq {b}: max abs err {err}"


def test_attend_selected_after_select_vs_oracle(cuda):
    """absp_attend_selected (the benchmark's attention-only graph) over absp_select's
    selection, and over the decode step's own selection, against the oracle."""
    from gpu_util import GpuLayer, within_tol
    layer = make_layer(31, H=8, G=4, d=128, P=16, block_sizes=(16, 32, 64), seq_lens=(20000, 9000, 131))
    gl = GpuLayer(layer, 2048)
    for step in ("select", "decode"):
        if step == "select":
            gl.select()
        else:
            gl.decode()
        out = torch.full((layer.batch, layer.H * layer.G, layer.d), float("nan"), dtype=torch.float32,
                         device="cuda")
        gl.da.attend_selected(0, gl.q, out)
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        for b in range(layer.batch):
            _, _, want_sel, want = oracle_step(layer, b, 2048)
            ok, err = within_tol(got[b], want)
            assert ok, f"{step} seq {b}: max abs err {err}"


def test_attend_validation_matches_reference_errors(cuda):
    from gpu_util import GpuLayer, to_dev_u32
    from paper_2605_12110_b200 import InvalidArgument, OutOfRange
    layer = make_layer(5, H=2, G=2, d=64, P=16, block_sizes=(16, 32), seq_lens=(500, 300))
    gl = GpuLayer(layer, 256)
    good = [[np.array([0, 3], np.uint32), np.array([1], np.uint32)] for _ in range(2)]
    _attend(gl, good, 4)  # no error

    def run(blocks, counts, stride):
        out = torch.empty(layer.batch, layer.H * layer.G, layer.d, dtype=torch.float32, device="cuda")
        b = np.zeros((layer.batch, layer.H, stride), np.uint32)
        for s in range(layer.batch):
            for h in range(layer.H):
                b[s, h, :len(blocks[s][h])] = blocks[s][h]
        gl.da.attend(0, gl.q, to_dev_u32(b), to_dev_u32(np.array(counts, np.uint32)), out)
        torch.cuda.synchronize()
        return out.cpu().numpy()

    with pytest.raises(InvalidArgument):  # empty selection (engine.cpp:224-226)
        run(good, [[2, 0], [2, 1]], 4)
    with pytest.raises(OutOfRange):       # block id past N (kv_cache.cpp:125-127)
        run([[np.array([0, 40], np.uint32), np.array([1], np.uint32)]] * 2, [[2, 1], [2, 1]], 4)
    with pytest.raises(InvalidArgument):  # count above the stride
        run(good, [[5, 1], [2, 1]], 4)
    # the flags are cleared by the check: a good call afterwards passes
    _attend(gl, good, 4)
    # an empty unit never reads out of bounds and writes zeros, not NaN
    gl.da.attend(0, gl.q, to_dev_u32(np.zeros((2, 2, 4), np.uint32)),
                 to_dev_u32(np.zeros((2, 2), np.uint32)),
                 out := torch.full((2, 4, 64), 7.0, device="cuda"), validate=False)
    torch.cuda.synchronize()
    assert torch.all(out == 0)
    with pytest.raises(InvalidArgument):
        from paper_2605_12110_b200._abi import check
        check(gl.da._lib.absp_attend_validate(gl.da._ctx, 0, None))


def test_attend_between_host_steps_keeps_graph_valid(cuda):
    """an explicit attention with a new, larger stride between two
    decode_step_host calls must not free buffers the captured host-step graph uses."""
    from gpu_util import GpuLayer
    layer = make_layer(21, H=8, G=4, d=128, P=16, block_sizes=(16, 32, 64), seq_lens=(9000, 12000))
    gl = GpuLayer(layer, 1024)
    dev = gl.decode()
    q_host = torch.from_numpy(layer.q.view(np.int16)).pin_memory()
    out_host = torch.empty(dev.shape, dtype=torch.float32).pin_memory()
    gl.da.decode_step_host(0, q_host, out_host)
    assert np.array_equal(out_host.numpy(), dev)
    rng = np.random.default_rng(3)
    for stride_extra in (0, 300, 700):
        sel, stride = _random_selection(rng, layer, stride_extra, short=False)
        _attend(gl, sel, stride)
        out_host.zero_()
        gl.da.decode_step_host(0, q_host, out_host)
        assert np.array_equal(out_host.numpy(), dev), stride_extra


def test_back_to_back_decode_steps_small_layer(cuda):
    """many decode steps on one small layer (attention grid far below
    the SM count) with no synchronisation in between; every step's output must be that
    of its own query (no step may consume the previous step's ready flags)."""
    from gpu_util import GpuLayer, to_dev_u16, within_tol
    from oracle.oracle import f32_to_bf16
    layer = make_layer(8, H=2, G=2, d=128, P=16, block_sizes=(16, 32), seq_lens=(3000,))
    gl = GpuLayer(layer, 512)
    rng = np.random.default_rng(9)
    qs = [f32_to_bf16(rng.standard_normal(layer.q.shape).astype(np.float32)) for _ in range(24)]
    qd = [to_dev_u16(q) for q in qs]
    outs = [torch.empty(1, 4, 128, dtype=torch.float32, device="cuda") for _ in qs]
    for q, o in zip(qd, outs):
        gl.da.decode_step(0, q, o)
    torch.cuda.synchronize()
    for q, o in zip(qs, outs):
        layer.q = q
        _, _, _, want = oracle_step(layer, 0, 512)
        ok, err = within_tol(o.cpu().numpy()[0], want)
        assert ok, err


def test_layout_version_and_append_graph_reuse(cuda):
    """Long sequences (N >= K for every unit): appends do not change any kernel argument
    of the step, so the layout version stays put and a captured graph of decode_step
    keeps producing the reference result after appends."""
    from gpu_util import GpuLayer, to_dev_u16, within_tol
    from oracle.oracle import f32_to_bf16
    n0, steps = 4000, 40
    # pages (and page-table entries) for the final lengths; the cache starts shorter
    layer = make_layer(12, H=4, G=2, d=128, P=16, block_sizes=(16, 32), seq_lens=(n0 + steps, n0 + 7 + steps))
    layer.seq_lens = [n0, n0 + 7]
    gl = GpuLayer(layer, 512, max_seq_len=n0 + 600)
    v0 = gl.da.layout_version(0)
    stream = torch.cuda.Stream()
    out = torch.empty(2, 8, 128, dtype=torch.float32, device="cuda")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        gl.da.decode_step(0, gl.q, out, stream)
    stream.synchronize()
    with torch.cuda.graph(g, stream=stream):
        gl.da.decode_step(0, gl.q, out, stream)
    rng = np.random.default_rng(4)
    pt = layer.page_table.copy()
    for step in range(steps):
        kn = f32_to_bf16(rng.standard_normal((2, 4, 128)).astype(np.float32))
        vn = f32_to_bf16(rng.standard_normal((2, 4, 128)).astype(np.float32))
        # host copy of the pools: write the new rows where the append will put them
        for b in range(2):
            n = layer.seq_lens[b]
            page, row = pt[b, n // 16], n % 16
            layer.k_pool[:, page, row, :] = kn[b]
            layer.v_pool[:, page, row, :] = vn[b]
            layer.seq_lens[b] = n + 1
        with torch.cuda.stream(stream):
            gl.da.append(0, to_dev_u16(kn), to_dev_u16(vn), stream)
            g.replay()
        stream.synchronize()
        assert gl.da.layout_version(0) == v0
        got = out.cpu().numpy()
        for b in range(2):
            _, _, _, want = oracle_step(layer, b, 512)
            ok, err = within_tol(got[b], want)
            assert ok, (step, b, err)
