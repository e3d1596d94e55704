"""World-size-2 gloo run of the multi-GPU partitioning on CPU: each rank evaluates its
shard of a small layer with the oracle, the outputs are all-gathered, and the union
equals the single-process result (units exchange nothing but the optional gather)."""
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


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from layer_data import make_layer, oracle_step
        from paper_2605_12110_b200.sharding import shard_units
        layer = make_layer(5, H=4, G=2, d=64, P=16, seq_lens=(900, 1500, 700, 2000))
        s = shard_units(layer.batch, layer.H, world, rank)
        out = torch.zeros(layer.batch, layer.H * layer.G, layer.d)
        for b in range(s.batch_start, s.batch_start + s.batch_count):
            _, _, _, o = oracle_step(layer, b, 256)
            out[b] = torch.from_numpy(o)
        gathered = [torch.zeros_like(out) for _ in range(world)]
        dist.all_gather(gathered, out)
        if rank == 0:
            q.put(torch.stack(gathered).sum(0).numpy())
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shards_cover_batch():
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).parent))
    from layer_data import make_layer, oracle_step
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    layer = make_layer(5, H=4, G=2, d=64, P=16, seq_lens=(900, 1500, 700, 2000))
    want = np.stack([oracle_step(layer, b, 256)[3] for b in range(layer.batch)])
    assert np.array_equal(got, want)
