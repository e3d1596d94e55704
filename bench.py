#!/usr/bin/env python
"""Decode-attention benchmark (BASELINE.json metric: decode-attn tokens/s @128K ctx on
1/2/4/8 B200; % of the HBM roofline on the bytes loaded).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl absp|reference]
                    [--workload cfg3] [--shard-of M [--shard-rank r]] [--no-verify]

A step is one decode step of the sparse attention path over one layer (cfg2: all 32
layers) for the workload's GLOBAL batch — BASELINE's configs fix it (cfg3: 16
sequences on 1/2/4/8 GPUs): quantized centroid scoring -> per-head Top-K -> sparse
paged flash-decode + LSE merge over a prefill-built store. Under
torchrun each rank builds and runs only its shard (paper_2605_12110_b200.sharding:
batch ranges, KV-head ranges when the batch is smaller than the world); there is no
collective on the data path. Inputs are resident in HBM; consecutive steps rotate
over independent layers (own KV cache, store and query) whose bytes exceed the L2.

value = global_batch / max-over-ranks(step time)            [tokens/s, strong scaling]
e2e   = the same through absp_decode_step_host: pinned host q -> H2D -> step -> the fp32
        output in pinned host memory -> stream sync, every step, max over ranks.
--shard-of M (1 GPU): time rank r's shard of the M-GPU run here (the per-GPU shape of
        that configuration); the line reports that shard's time and the projected
        M-GPU aggregate global_batch / shard time.

After timing, --verify (default) reads back one sequence per rotated layer and checks
store, scores, selection (bit-exact) and output (1e-3 + 1e-2|x|) against the unmodified
reference core (oracle/_ref); the line carries "verified".

--impl reference times the reference's own CPU implementation (oracle/_ref, the
unmodified reference core) on this host's cores for the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: GLOBAL batch (BASELINE.json), seq len, kv heads, G, head dim, page, candidates, budget
    "cfg1": dict(batch=1, n=8192, H=8, G=4, d=128, P=8, cands=(8, 16, 32), T=1024,
                 desc="Llama-3.1-8B single attention layer, batch 1, 8K ctx, blocks {8,16,32}, T=1024"),
    # a step is the decode attention of all 32 layers (one graph, layer after layer)
    "cfg2": dict(batch=8, n=32768, H=8, G=4, d=128, P=16, cands=(16, 32, 64), T=2048, layers_per_step=32,
                 desc="Llama-3.1-8B all 32 layers, batch 8, 32K ctx, blocks {16,32,64}, T=2048 (assumed), int4 mean"),
    "cfg3": dict(batch=16, n=131072, H=8, G=4, d=128, P=16, cands=(16, 32, 64), T=2048,
                 desc="Llama-3.1-8B decode attention, batch 16, 128K ctx, blocks {16,32,64}, T=2048"),
    "cfg4u": dict(batch=32, n=131072, H=8, G=4, d=128, P=16, cands=(16,), T=2048,
                  desc="Quest-style uniform block 16, batch 32, 128K ctx, T=2048"),
    "cfg4a": dict(batch=32, n=131072, H=8, G=4, d=128, P=16, cands=(16, 32, 64), T=2048,
                  desc="adaptive blocks {16,32,64}, batch 32, 128K ctx, T=2048"),
    "cfg5": dict(batch=64, n=131072, H=8, G=8, d=128, P=4, cands=(4, 8, 16, 32, 64), T=2048,
                 desc="Qwen3-32B shape (64q/8kv), batch 64, 128K ctx, blocks {4..64}, T=2048 (assumed)"),
}
METRIC = "decode-attn tokens/sec @128K ctx (1/2/4/8 B200); % HBM roofline on bytes loaded"
SEED = 42
L2_BYTES = 126 * 2**20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["absp", "reference"], default="absp")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg3")
    ap.add_argument("--shard-of", type=int, default=1, help="1 GPU: time rank r's shard of an M-GPU run")
    ap.add_argument("--shard-rank", type=int, default=0)
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-reps", type=int, default=5)
    ap.add_argument("--layers", type=int, default=0, help="rotated layers (0: enough to defeat the L2)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def stream_id(layer, b, h, kind):
    """Synthetic-data stream of (layer, global sequence, global KV head, K/V/q): every
    sharding of a workload sees the same bytes per unit."""
    return ((layer * 128 + b) * 16 + h) * 4 + kind


def make_config(args, w, plan):
    """The config dict both arms print (same keys, same values)."""
    s = plan.shard
    return {
        "workload": args.workload, "desc": w["desc"], "global_batch": w["batch"], "seq_len": w["n"],
        "kv_heads": w["H"], "q_heads": w["H"] * w["G"], "head_dim": w["d"], "page_size": w["P"],
        "block_sizes": [w["cands"][h % len(w["cands"])] for h in range(w["H"])], "token_budget": w["T"],
        "quant": "int4xasym", "centroids": "mean", "layers_per_step": w.get("layers_per_step", 1),
        "parallelism": (f"{plan.world}-way {'kv-head' if plan.head_sharded else 'batch'} shards of the global "
                        f"batch, no data-path collective"),
        "shard": {"of": plan.world, "rank": plan.rank, "batch": [s.batch_start, s.batch_count],
                  "kv_heads": [s.head_start, s.head_count]},
    }


def algorithmic_bytes(w, Hl, kv_bytes, total_centroids, batch):
    """packed codes + per-(h,c) scale/zp + selected K/V rows + q + out."""
    d = w["d"]
    codes = total_centroids * d * 4 // 8
    params = batch * Hl * 2 * d * 4
    q = batch * Hl * w["G"] * d * 2
    out = batch * Hl * w["G"] * d * 4
    return codes + params + kv_bytes + q + out, codes + params, kv_bytes


class ClockSampler:
    """Samples the SM clock and throttle reasons through NVML while work runs (polling
    without sleeping: the timed region can be ~1 ms)."""

    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
             0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
             0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int, period_s: float = 0.0):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self.period = period_s
        self._stop = threading.Event()
        self._t = None
        self.t0 = self.t1 = 0.0
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - NVML missing
            self.nv = None
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.NAMES.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            if self.period:
                time.sleep(self.period)

    def __enter__(self):
        self.t0 = time.perf_counter()
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()
        self.t1 = time.perf_counter()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples), "reasons": sorted(self.reasons),
                "window_ms": round((self.t1 - self.t0) * 1e3, 2)}


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref = the unmodified reference core), host cores
# ---------------------------------------------------------------------------
def _host_sequence(w, b=0, layer=0):
    """Sequence b of layer `layer` as the GPU arm generates it (same bytes, oracle/synth.py)."""
    import numpy as np
    from oracle import oracle as O
    from oracle.synth import synth_bf16
    H, n, d, G = w["H"], w["n"], w["d"], w["G"]
    keys = np.empty((H, n, d), np.float32)
    vals = np.empty((H, n, d), np.float32)
    q = np.empty((H * G, d), np.float32)
    for h in range(H):
        keys[h] = O.bf16_to_f32(synth_bf16(n * d, SEED, stream_id(layer, b, h, 0))).reshape(n, d)
        vals[h] = O.bf16_to_f32(synth_bf16(n * d, SEED, stream_id(layer, b, h, 1))).reshape(n, d)
        q[h * G:(h + 1) * G] = O.bf16_to_f32(synth_bf16(G * d, SEED, stream_id(layer, b, h, 2))).reshape(G, d)
    return keys, vals, q


def cpu_reference(w, reps: int, warmup: int, seq=None):
    """Times the reference's own decode path for one sequence of the workload (the bounded
    sample): estimate_scores(group-summed q, int4 store) -> select_topk -> populate_page_spans
    -> G x sparse_attention, on the same bf16 bytes the GPU sees."""
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    os.environ.setdefault("OMP_PROC_BIND", "true")
    from oracle import oracle as O
    if not O.ref_available():
        return None, "oracle/_ref not built"
    keys, vals, q = seq if seq is not None else _host_sequence(w)
    H = keys.shape[0]
    bs = [w["cands"][h % len(w["cands"])] for h in range(H)]
    t0 = time.perf_counter()
    ref = O.RefSeq(keys, vals, w["P"], bs, 0, 4, 1)
    build_s = time.perf_counter() - t0
    del keys, vals
    for _ in range(warmup):
        ref.decode_gqa(q, w["G"], w["T"])
    times = []
    for _ in range(reps):
        t = time.perf_counter()
        ref.decode_gqa(q, w["G"], w["T"])
        times.append(time.perf_counter() - t)
    return {"seconds_per_sequence": statistics.median(times), "all": times, "cores": cores,
            "prefill_build_s": build_s}, None


def run_reference(args, w, rank, world):
    from paper_2605_12110_b200.sharding import ShardPlan
    if rank != 0:
        return
    plan = ShardPlan(w["batch"], w["H"], w["G"], max(world, args.shard_of), 0 if world > 1 else args.shard_rank)
    res, err = cpu_reference(w, max(args.steps, 1), max(args.warmup, 0))
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": err}))
        return
    lps = w.get("layers_per_step", 1)
    t = res["seconds_per_sequence"] * lps  # a token passes every layer of a step
    value = 1.0 / t  # a batch of b sequences takes b*t on the host, producing b tokens
    sample = (f"1 sequence of the {w['batch']}-sequence global batch per step ({w['n']} ctx, layer 0, "
              f"all {w['H']} kv heads); tokens/s = batch / (batch x per-sequence time x {lps} layers)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3 * w["batch"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": make_config(args, w, plan),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": res["cores"], "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ---------------------------------------------------------------------------
# B200 path
# ---------------------------------------------------------------------------
def source_sha() -> str:
    """Hash of the kernel sources: ties a committed ncu capture to the build it measured."""
    h = hashlib.sha256()
    csrc = ROOT / "paper_2605_12110_b200" / "csrc"
    for f in sorted(csrc.glob("*")):
        h.update(f.name.encode())
        h.update(f.read_bytes())
    return h.hexdigest()[:16]


def measured_traffic(workload, shard_of):
    """DRAM read+write bytes of one k_attn launch from the committed ncu capture
    (profiles/attn_traffic.json), used only when it was taken on this workload and shard
    AND on the current kernel sources (source_sha), else None."""
    f = ROOT / "profiles" / "attn_traffic.json"
    try:
        recs = json.loads(f.read_text())
    except (OSError, ValueError):
        return None, "no capture"
    sha = source_sha()
    for t in recs if isinstance(recs, list) else [recs]:
        if t.get("workload") == workload and t.get("shard_of", 1) == shard_of:
            if t.get("source_sha") != sha:
                return None, f"capture {t.get('source_sha')} is stale (sources {sha})"
            return t["dram_bytes_read"] + t["dram_bytes_write"], f"ncu --set full, sources {sha}"
    return None, "no capture of this workload"


def trace(msg):
    if os.environ.get("ABSP_BENCH_TRACE"):
        print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def verify_layer(da, l, lay, b, w, Hl, bs_local):
    """One sequence of one layer against the unmodified reference core (oracle/_ref):
    store, scores and the decode step's selection bit-exact, output in tolerance."""
    import numpy as np
    from oracle import oracle as O
    d, P, n, G, T = w["d"], w["P"], w["n"], w["G"], w["T"]
    rows = lay["pt"][b].long()
    kb = lay["k"][:, rows].cpu().numpy().view(np.uint16).reshape(Hl, -1, d)[:, :n]
    vb = lay["v"][:, rows].cpu().numpy().view(np.uint16).reshape(Hl, -1, d)[:, :n]
    ref = O.RefSeq(O.bf16_to_f32(kb), O.bf16_to_f32(vb), P, bs_local, 0, 4, 1)
    del kb, vb
    want = ref.store()
    got = da.download_store(l, b)
    bits = lambda a: np.ascontiguousarray(a).view(np.uint8)
    fails = []
    for key in ("codes", "scales", "zps", "values"):
        if not np.array_equal(bits(got[key]), bits(want[key])):
            fails.append(f"store.{key}")
    qb = O.bf16_to_f32(lay["q"][b].cpu().numpy().view(np.uint16)).reshape(Hl * G, d)
    qsum = O.group_sum(qb, Hl, G)
    sc = ref.scores(qsum)
    import torch
    info = da.layer_info(l)
    Bl = lay["q"].shape[0]
    sb = torch.empty(Bl, Hl, max(info.max_select, 1), dtype=torch.int32, device=lay["q"].device)
    scnt = torch.empty(Bl, Hl, dtype=torch.int32, device=lay["q"].device)
    da.select(l, lay["q"], sb, scnt)  # absp_select materialises every exact score (estimate_scores)
    torch.cuda.synchronize()
    if not np.array_equal(bits(da.download_scores(l, b)), bits(sc)):
        fails.append("scores")
    sel_sel = sb[b].cpu().numpy().view(np.uint32)
    sel_cnt = scnt[b].cpu().numpy().view(np.uint32)
    want_sel = ref.select(sc, T)
    if not all(np.array_equal(sel_sel[h, :sel_cnt[h]], want_sel[h]) for h in range(Hl)):
        fails.append("selection (absp_select)")
    got_sel = lay["step_sel"][b]  # the decode step's own selection (fused path), read before
    if not all(np.array_equal(x, y) for x, y in zip(got_sel, want_sel)):
        fails.append("selection (decode step)")
    want_out = ref.decode_gqa(qb, G, T)
    got_out = lay["out"][b].cpu().numpy()
    err = np.abs(got_out.astype(np.float64) - want_out)
    if not np.all(err <= 1e-3 + 1e-2 * np.abs(want_out)):
        fails.append(f"output (max abs err {err.max():.3g})")
    return fails, float(err.max())


def run_absp(args, w, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2605_12110_b200 import (BlockAssignment, DecodeAttention, EngineConfig, QuantSpec,
                                       fill_synthetic_bf16)
    from paper_2605_12110_b200.sharding import ShardedDecode, ShardPlan

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    M = world if world > 1 else max(1, args.shard_of)
    plan = ShardPlan(w["batch"], w["H"], w["G"], M, rank if world > 1 else args.shard_rank)
    sh = plan.shard
    B, Hl = sh.batch_count, sh.head_count
    n, H, G, d, P, T = w["n"], w["H"], w["G"], w["d"], w["P"], w["T"]
    lps = w.get("layers_per_step", 1)
    cands_all = [w["cands"][h % len(w["cands"])] for h in range(H)]
    bs_local = plan.block_sizes(cands_all)
    pps = (n + P - 1) // P
    pages_total = B * pps
    # rotated layers: enough that a step never finds the previous steps' bytes in the L2
    per_layer_kv = Hl * pages_total * P * d * 2 * 2
    est_step = B * sum((-(-n // bsz)) * d // 2 + min(n, T + bsz) * d * 4 for bsz in bs_local)
    L = args.layers or max(lps, 2, math.ceil(3 * L2_BYTES / max(est_step, 1)))
    L = -(-L // lps) * lps
    L = min(L, max(lps, int(110e9 // per_layer_kv) // lps * lps))
    cfg = EngineConfig(num_heads=Hl, head_dim=d, page_size=P, candidate_block_sizes=tuple(w["cands"]),
                       token_budget=T, quant=QuantSpec(4), num_q_heads=Hl * G, max_batch=B, max_seq_len=n,
                       num_layers=L)
    da = DecodeAttention(cfg, device=local)
    assignment = BlockAssignment(bs_local)
    stream = torch.cuda.Stream(device=dev)
    pt = torch.arange(pages_total, dtype=torch.int32, device=dev).reshape(B, pps)  # the reference allocator's order
    layers = []
    with torch.cuda.stream(stream):
        for l in range(L):
            k = torch.empty(Hl, pages_total, P, d, dtype=torch.int16, device=dev)
            v = torch.empty_like(k)
            q = torch.empty(B, Hl * G, d, dtype=torch.int16, device=dev)
            for bl in range(B):
                gb = sh.batch_start + bl
                for hl in range(Hl):
                    gh = sh.head_start + hl
                    fill_synthetic_bf16(k[hl, bl * pps:(bl + 1) * pps], SEED, stream_id(l, gb, gh, 0), stream)
                    fill_synthetic_bf16(v[hl, bl * pps:(bl + 1) * pps], SEED, stream_id(l, gb, gh, 1), stream)
                    fill_synthetic_bf16(q[bl, hl * G:(hl + 1) * G], SEED, stream_id(l, gb, gh, 2), stream)
            out = torch.empty(B, Hl * G, d, dtype=torch.float32, device=dev)
            da.set_assignment(l, assignment)
            da.bind(l, k, v, pt, [n] * B)
            da.build_store(l, stream)
            layers.append(dict(k=k, v=v, q=q, out=out, pt=pt))
    stream.synchronize()
    trace(f"{L} layers built (shard {sh})")
    info = da.layer_info(0)
    step_bytes, select_bytes, attn_kv_bytes = algorithmic_bytes(w, Hl, info.kv_bytes_selected,
                                                                info.total_centroids, B)
    step_bytes *= lps  # every layer of a step reads its own store and KV
    attn_bytes = attn_kv_bytes + B * Hl * G * d * (2 + 4)

    # The timed loops replay CUDA graphs that run the L rotating layers back to back, as a
    # model's decode step runs its layers: one graph per chain of all L layers (plus the
    # partial chains a step count that is not a multiple of L needs), so no per-layer graph
    # launch gap is timed. A "step" stays one layer's decode (cfg2: lps = 32 layers).
    launches_before = da.launch_count()
    with torch.cuda.stream(stream):
        for l in range(L):  # eager warm-up (also initialises the selection buffers)
            da.decode_step(l, layers[l]["q"], layers[l]["out"], stream)
    stream.synchronize()
    per_step_launches = (da.launch_count() - launches_before) // L * lps
    S = L // lps  # steps per chain

    def chains(layer_fn):
        """graphs[r] runs steps 0..r-1 of the chain (r = 1..S)."""
        out = {}
        for r in range(1, S + 1):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for l in range(r * lps):
                    layer_fn(l)
            out[r] = g
        return out

    step_chain = chains(lambda l: da.decode_step(l, layers[l]["q"], layers[l]["out"], stream))
    att_chain = chains(lambda l: da.attend_selected(l, layers[l]["q"], layers[l]["out"], stream))
    sel_chain = chains(lambda l: da.select_step(l, layers[l]["q"], stream))

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def run_steps(chain, steps):
        """`steps` layer-steps as full chains plus one partial chain."""
        for _ in range(steps // S):
            chain[S].replay()
        if steps % S:
            chain[steps % S].replay()

    def timed(fn, steps, warm, sampler=None):
        """fn(n): enqueue n steps on the stream; CUDA events around `steps` of them."""
        with torch.cuda.stream(stream):
            fn(warm)
        stream.synchronize()
        sync_all()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if sampler:
            sampler.__enter__()
        with torch.cuda.stream(stream):
            e0.record(stream)
            fn(steps)
            e1.record(stream)
        e1.synchronize()
        if sampler:
            sampler.__exit__()
        sync_all()
        return max_over_ranks(e0.elapsed_time(e1) / steps)

    K, W = args.steps, max(args.warmup, 3)
    step_fn = lambda n: run_steps(step_chain, n)
    # clocks: a >= 100 ms window of the same step back to back just before the timed
    # region (the timed region itself can be ~1 ms), plus samples during the timed region
    window = ClockSampler(local, 0.002)
    reps = 0
    with window:
        t_end = time.perf_counter() + 0.12
        while time.perf_counter() < t_end:
            with torch.cuda.stream(stream):
                step_fn(64)
            reps += 64
            stream.synchronize()
    sampler = ClockSampler(local, 0.0)
    ms_step = timed(step_fn, K, W, sampler)
    trace(f"step timed: {ms_step * 1e3:.1f} us")
    # per-kernel breakdown: the attention alone and the selection alone, per layer
    ms_attn = timed(lambda n: run_steps(att_chain, n), K, W) / lps
    ms_sel = timed(lambda n: run_steps(sel_chain, n), K, W) / lps

    # optional all-gather of the per-rank outputs into the global [b][Hq][d] (reported
    # separately: the path itself exchanges nothing)
    gather_us = None
    if world > 1:
        sd = ShardedDecode(plan, lambda ql, ol: None, d, torch, device=dev, group=None)
        ms_gather = timed(lambda n: [sd.gather() for _ in range(n)], K, W)
        gather_us = ms_gather * 1e3

    # end to end through the public C ABI with host buffers
    q_host = [torch.empty(B, Hl * G, d, dtype=torch.int16).pin_memory() for _ in range(L)]
    for l in range(L):
        q_host[l].copy_(layers[l]["q"].cpu())
    out_host = torch.empty(B, Hl * G, d, dtype=torch.float32).pin_memory()

    def host_step(i):
        first = (i * lps) % L
        for l in range(first, first + lps):
            da.decode_step_host(l, q_host[l], out_host, stream)

    for i in range(max(W, L // lps)):  # every layer's host graph is captured before timing
        host_step(i)
    sync_all()
    t0 = time.perf_counter()
    for i in range(K):
        host_step(i)
    e2e_s = max_over_ranks((time.perf_counter() - t0) / K)
    trace(f"e2e timed: {e2e_s * 1e6:.1f} us")

    # parity of what was just timed, outside the timed region
    verified, vinfo = None, None
    if not args.no_verify:
        from oracle import oracle as O
        if O.ref_available():
            with torch.cuda.stream(stream):
                for l in range(L):
                    da.decode_step(l, layers[l]["q"], layers[l]["out"], stream)
            stream.synchronize()
            for l in range(L):
                layers[l]["step_sel"] = da.download_selection(l)
            fails, errs, checked = [], [], []
            # one sequence per rotated layer, up to ~1M verified tokens (cfg2: all 32 layers)
            for l in range(min(L, max(1, (1 << 20) // n))):
                b = l % B
                f, e = verify_layer(da, l, layers[l], b, w, Hl, bs_local)
                fails += [f"layer {l} seq {b}: {x}" for x in f]
                errs.append(e)
                checked.append([l, sh.batch_start + b])
            ok = torch.tensor([0 if fails else 1], device=dev)
            if world > 1:
                dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            verified = bool(ok.item())
            vinfo = {"against": "oracle/_ref (unmodified reference core)", "checked_layer_seq": checked,
                     "store_scores_selection": "bit-exact" if not fails else "MISMATCH",
                     "max_abs_err_output": max(errs), "tolerance": "1e-3 + 1e-2|x|", "failures": fails[:8]}
            if fails:
                print("VERIFY FAILED: " + "; ".join(fails[:8]), file=sys.stderr)
        else:
            vinfo = {"skipped": "oracle/_ref not built"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if plan.head_sharded:
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": "skipped: head-sharded shard (run --shard-of 1 for the full-sequence baseline)"}
        else:
            import numpy as np  # noqa: F811
            from oracle import oracle as O
            lay = layers[0]
            rows = lay["pt"][0].long()
            kf = O.bf16_to_f32(lay["k"][:, rows].cpu().numpy().view(np.uint16).reshape(Hl, -1, d)[:, :n])
            vf = O.bf16_to_f32(lay["v"][:, rows].cpu().numpy().view(np.uint16).reshape(Hl, -1, d)[:, :n])
            qf = O.bf16_to_f32(lay["q"][0].cpu().numpy().view(np.uint16)).reshape(Hl * G, d)
            res, err = cpu_reference(w, args.cpu_reps, 1, (kf, vf, qf))
            if res:
                cpu = {"value": 1.0 / (res["seconds_per_sequence"] * lps), "unit": "tokens/s",
                       "cores": res["cores"], "kind": "reference",
                       "sample": f"1 sequence ({n} ctx, layer 0, the bytes the GPU timed), median of "
                                 f"{args.cpu_reps} after 1 warm-up; OMP over all host cores; tokens/s = "
                                 f"1 / (per-sequence per-layer time x {lps} layers)"}
            else:
                cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "reference", "sample": err}

    if rank == 0:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
        peak = float(peaks.get("hbm_gbs", 6650.0))
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"
        shard_tokens = B if not plan.head_sharded else B * Hl / H
        if world > 1:
            value = w["batch"] / (ms_step / 1e3)
        else:
            value = shard_tokens / (ms_step / 1e3)  # this GPU's tokens/s (the whole job when M = 1)
        attn_gbs = attn_bytes / (ms_attn / 1e3) / 1e9
        traffic, traffic_src = measured_traffic(args.workload, M)
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (device-generated counter-based N(0,1) bf16 K/V/q)",
            "config": make_config(args, w, plan),
            "notes": {"l2": f"{L} rotating layers x {step_bytes / lps / 1e6:.1f} MB algorithmic bytes per "
                            f"layer-step (> 126 MB L2 between reuses)", "layers_rotated": L,
                      "compute": "int4 codes -> exact fp32 scores; bf16 MMA (mma.sync) fp32 accumulate"},
            "roofline": {"bound": "hbm", "kernel": "k_attn (absp_attend_selected: paged flash-decode + fused LSE merge)",
                         "achieved": attn_gbs, "peak": peak, "unit": "GB/s", "frac": attn_gbs / peak,
                         "traffic": traffic, "traffic_source": traffic_src, "bytes_per_launch": attn_bytes,
                         "peak_source": peak_src, "timing": "CUDA events over K attention-only launches, the "
                                                           "rotating layers back to back in one graph / K"},
            "step_roofline": {"bytes_per_step": step_bytes, "achieved_gbs": step_bytes / (ms_step / 1e3) / 1e9,
                              "frac": step_bytes / (ms_step / 1e3) / 1e9 / peak},
            "kernels_us": {"step": ms_step * 1e3, "select": ms_sel * 1e3, "attend": ms_attn * 1e3,
                           "select_bytes": select_bytes},
            "cpu_baseline": cpu,
            "e2e": {"value": (w["batch"] if world > 1 else shard_tokens) / e2e_s, "unit": "tokens/s",
                    "h2d_bytes_per_step": B * Hl * G * d * 2 * lps, "d2h_bytes_per_step": B * Hl * G * d * 4 * lps,
                    "ms_per_step": e2e_s * 1e3},
            "gpu_launches": per_step_launches * K,
            "clocks": dict(window.summary(), timed_region=sampler.summary(), window_steps=reps),
            "verified": verified, "verify": vinfo,
        }
        if M > 1 and world == 1:
            line["projected"] = {
                "gpus": M, "aggregate_tokens_per_s": w["batch"] / (ms_step / 1e3),
                "note": f"rank {plan.rank}'s shard of the {M}-GPU run timed on this GPU; every rank's shard "
                        f"has this shape when {M} divides the batch (no data-path collective)"}
        if gather_us is not None:
            line["allgather_us"] = {"value": gather_us, "bytes_per_rank": int(sd.slot.numel() * 4),
                                    "op": "ncclAllGather of fp32 [b_local][Hq_local][d] outputs (not in value)"}
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, w, rank, world)
        return
    run_absp(args, w, rank, world, local)


if __name__ == "__main__":
    main()
