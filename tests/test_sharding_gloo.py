"""World-size-2 gloo runs of the sharded host orchestration (paper_2605_12110_b200.sharding):
each rank builds its shard of a BASELINE-style global batch (batch ranges, or KV-head
ranges when the batch is smaller than the world), runs its local decode step on its
slice of the global query, and the outputs are all-gathered into the global layout.
On CPU the local step is the oracle (the GPU runs DecodeAttention.decode_step in the
same slot, tests/test_gpu_sharding.py); the assembled output must equal the
single-process result exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def sub_layer(layer, shard):
    """The rank's shard of a host Layer: its sequences and KV heads (tests/layer_data.py)."""
    from layer_data import Layer
    b0, bc, h0, hc = shard.batch_start, shard.batch_count, shard.head_start, shard.head_count
    G = layer.G
    return Layer(hc, G, layer.d, layer.P, layer.block_sizes[h0:h0 + hc], layer.seq_lens[b0:b0 + bc],
                 np.ascontiguousarray(layer.k_pool[h0:h0 + hc]), np.ascontiguousarray(layer.v_pool[h0:h0 + hc]),
                 layer.page_table[b0:b0 + bc], np.ascontiguousarray(layer.q[b0:b0 + bc, h0 * G:(h0 + hc) * G]))


LAYERS = {
    "batch": dict(seed=5, H=4, G=2, d=64, P=16, seq_lens=(900, 1500, 700, 2000, 333)),
    "heads": dict(seed=6, H=4, G=2, d=64, P=16, seq_lens=(2100,)),
}


def _layer(kind):
    from layer_data import make_layer
    kw = dict(LAYERS[kind])
    return make_layer(kw.pop("seed"), **kw)


def _worker(rank, world, port, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path
        sys.path.insert(0, str(Path(__file__).parent))
        from layer_data import oracle_step
        from paper_2605_12110_b200.sharding import ShardedDecode, ShardPlan
        layer = _layer(kind)
        plan = ShardPlan(layer.batch, layer.H, layer.G, world, rank)
        local = sub_layer(layer, plan.shard)
        q_global = torch.from_numpy((layer.q.astype(np.uint32) << 16).view(np.float32))

        def local_step(q_local, out_local):
            # the rank's slice of the global query is exactly its shard's query
            assert np.array_equal(q_local.numpy(), (local.q.astype(np.uint32) << 16).view(np.float32))
            for b in range(local.batch):
                out_local[b] = torch.from_numpy(oracle_step(local, b, 256)[3])

        sd = ShardedDecode(plan, local_step, layer.d, torch)
        out = torch.full((layer.batch, layer.H * layer.G, layer.d), float("nan"))
        sd.step(q_global, out)
        if rank == 0:
            q.put((plan.shard, out.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["batch", "heads"])
def test_gloo_world2_sharded_step(kind):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).parent))
    from layer_data import oracle_step
    from paper_2605_12110_b200.sharding import ShardPlan
    layer = _layer(kind)
    plans = [ShardPlan(layer.batch, layer.H, layer.G, 2, r) for r in range(2)]
    if kind == "heads":
        assert all(p.head_sharded for p in plans)
    else:
        assert not any(p.head_sharded for p in plans)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    shard0, got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert shard0 == plans[0].shard
    want = np.stack([oracle_step(layer, b, 256)[3] for b in range(layer.batch)])
    assert np.array_equal(got, want)


def test_shard_plans_cover_baseline_configs():
    from paper_2605_12110_b200.sharding import ShardPlan
    for batch, world in [(16, 1), (16, 2), (16, 4), (16, 8), (32, 8), (64, 8), (1, 2), (1, 4), (1, 8), (8, 8), (5, 2)]:
        plans = [ShardPlan(batch, 8, 4, world, r) for r in range(world)]
        units = set()
        for p in plans:
            s = p.shard
            for b in range(s.batch_start, s.batch_start + s.batch_count):
                for h in range(s.head_start, s.head_start + s.head_count):
                    assert (b, h) not in units
                    units.add((b, h))
        assert len(units) == batch * 8, (batch, world)
        if batch % world == 0:  # identical per-rank shapes
            assert len({(p.shard.batch_count, p.shard.head_count) for p in plans}) == 1
