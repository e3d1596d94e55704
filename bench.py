#!/usr/bin/env python
"""Decode-attention benchmark (BASELINE.json metric: decode-attn tokens/s @128K ctx).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl absp|reference] [--workload cfg3]

A step is one decode step of the sparse attention path over one layer for the whole
per-GPU batch: quantized centroid scoring -> per-head Top-K -> sparse paged
flash-decode + LSE merge, over a prefill-built store. Inputs are
resident in HBM; consecutive steps rotate over `layers` independent layers (each with
its own KV cache, store and query) so no step finds the previous steps' bytes in L2.

value = (batch_per_gpu * N) / max-over-ranks(step time)   [tokens/s, weak scaling]
e2e   = the same through absp_decode_step_host: pinned host q -> H2D -> step -> D2H
        of the fp32 output -> stream sync, every step.

--impl reference times the reference's own CPU implementation (oracle/_ref, the
unmodified reference core) on this host's cores for the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: batch per GPU, seq len, kv heads, G, head dim, page, candidates, budget, layers rotated
    "cfg1": dict(batch=1, n=8192, H=8, G=4, d=128, P=8, cands=(8, 16, 32), T=1024, layers=64,
                 desc="Llama-3.1-8B single layer, batch 1, 8K ctx, blocks {8,16,32}, T=1024"),
    # a step is the decode attention of all 32 layers (one graph, layer after layer)
    "cfg2": dict(batch=8, n=32768, H=8, G=4, d=128, P=16, cands=(16, 32, 64), T=2048, layers=32,
                 layers_per_step=32,
                 desc="Llama-3.1-8B all 32 layers, batch 8, 32K ctx, blocks {16,32,64}, T=2048 (assumed), int4 mean"),
    "cfg3": dict(batch=16, n=131072, H=8, G=4, d=128, P=16, cands=(16, 32, 64), T=2048, layers=4,
                 desc="Llama-3.1-8B decode attention, batch 16/GPU, 128K ctx, blocks {16,32,64}, T=2048"),
    "cfg4u": dict(batch=32, n=131072, H=8, G=4, d=128, P=16, cands=(16,), T=2048, layers=2,
                  desc="Quest-style uniform block 16, batch 32/GPU, 128K ctx, T=2048"),
    "cfg4a": dict(batch=32, n=131072, H=8, G=4, d=128, P=16, cands=(16, 32, 64), T=2048, layers=2,
                  desc="adaptive blocks {16,32,64}, batch 32/GPU, 128K ctx, T=2048"),
    "cfg5": dict(batch=64, n=131072, H=8, G=8, d=128, P=4, cands=(4, 8, 16, 32, 64), T=2048, layers=2,
                 desc="Qwen3-32B shape (64q/8kv), batch 64/GPU, 128K ctx, blocks {4..64}, T=2048 (assumed)"),
}
METRIC = "decode-attn tokens/sec @128K ctx (1/2/4/8 B200); % HBM roofline on bytes loaded"
SEED = 42


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["absp", "reference"], default="absp")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-reps", type=int, default=5)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def algorithmic_bytes(w, info_kv_bytes, total_centroids, batch):
    """packed codes + per-(h,c) scale/zp + selected K/V rows + q + out."""
    d = w["d"]
    codes = total_centroids * d * 4 // 8
    params = batch * w["H"] * 2 * d * 4
    q = batch * w["H"] * w["G"] * d * 2
    out = batch * w["H"] * w["G"] * d * 4
    return codes + params + info_kv_bytes + q + out, codes + params, info_kv_bytes


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML while the timed region runs."""

    def __init__(self, device_index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - NVML missing
            self.nv = None
            self.err = str(e)

    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
             0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
             0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

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
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples), "reasons": sorted(self.reasons)}


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref = the unmodified reference core), host cores
# ---------------------------------------------------------------------------
def cpu_reference(w, reps: int, warmup: int):
    """Times the reference's own decode path for one sequence of the workload (the bounded
    sample): estimate_scores(group-summed q, int4 store) -> select_topk -> populate_page_spans
    -> G x sparse_attention, on the same bf16 bytes the GPU sees."""
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    os.environ.setdefault("OMP_PROC_BIND", "true")
    import numpy as np
    from oracle import oracle as O
    from oracle.synth import synth_bf16
    if not O.ref_available():
        return None, "oracle/_ref not built"
    H, n, d, P, G = w["H"], w["n"], w["d"], w["P"], w["G"]
    pages_total = w["batch"] * ((n + P - 1) // P)
    keys = np.empty((H, n, d), np.float32)
    vals = np.empty((H, n, d), np.float32)
    for h in range(H):  # sequence 0 of layer 0 occupies the first n rows of each head's pool
        start = h * pages_total * P * d
        keys[h] = O.bf16_to_f32(synth_bf16(n * d, SEED, 0, start)).reshape(n, d)
        vals[h] = O.bf16_to_f32(synth_bf16(n * d, SEED, 1, start)).reshape(n, d)
    q = O.bf16_to_f32(synth_bf16(w["batch"] * H * G * d, SEED, 2))[: H * G * d].reshape(H * G, d)
    bs = [w["cands"][h % len(w["cands"])] for h in range(H)]
    t0 = time.perf_counter()
    seq = O.RefSeq(keys, vals, P, bs, 0, 4, 1)
    build_s = time.perf_counter() - t0
    del keys, vals
    for _ in range(warmup):
        seq.decode_gqa(q, G, w["T"])
    times = []
    for _ in range(reps):
        t = time.perf_counter()
        seq.decode_gqa(q, G, w["T"])
        times.append(time.perf_counter() - t)
    return {"seconds_per_sequence": statistics.median(times), "all": times, "cores": cores,
            "prefill_build_s": build_s}, None


def run_reference(args, w, rank, world):
    if rank != 0:
        return
    res, err = cpu_reference(w, max(args.steps, 1), max(args.warmup, 0))
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": err}))
        return
    t = res["seconds_per_sequence"] * w.get("layers_per_step", 1)  # a token passes every layer of a step
    value = 1.0 / t  # a batch of b sequences takes b*t, producing b tokens
    sample = (f"1 sequence of the {w['batch']}-sequence batch per step ({w['n']} ctx, layer 0); "
              f"tokens/s = batch / (batch x per-sequence time x {w.get('layers_per_step', 1)} layers)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3 * w["batch"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": args.workload, "desc": w["desc"]},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": res["cores"], "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ---------------------------------------------------------------------------
# B200 path
# ---------------------------------------------------------------------------
def measured_traffic(workload):
    """DRAM read+write bytes of one k_attn launch from the committed ncu capture
    (profiles/r1/attn_traffic.json) when it is of this workload, else None."""
    f = ROOT / "profiles" / "r1" / "attn_traffic.json"
    try:
        t = json.loads(f.read_text())
    except (OSError, ValueError):
        return None
    return t["dram_bytes_read"] + t["dram_bytes_write"] if t.get("workload") == workload else None


def trace(msg):
    if os.environ.get("ABSP_BENCH_TRACE"):
        print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def run_absp(args, w, rank, world, local):
    import torch
    import torch.distributed as dist
    from paper_2605_12110_b200 import (BlockAssignment, DecodeAttention, EngineConfig, QuantSpec,
                                       fill_synthetic_bf16)

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    B, n, H, G, d, P, T, L = w["batch"], w["n"], w["H"], w["G"], w["d"], w["P"], w["T"], w["layers"]
    pages_per_seq = (n + P - 1) // P
    pages_total = B * pages_per_seq
    cfg = EngineConfig(num_heads=H, head_dim=d, page_size=P, candidate_block_sizes=tuple(w["cands"]),
                       token_budget=T, quant=QuantSpec(4), num_q_heads=H * G, max_batch=B, max_seq_len=n,
                       num_layers=L)
    da = DecodeAttention(cfg, device=local)
    assignment = BlockAssignment.cycled(H, w["cands"])
    stream = torch.cuda.Stream(device=dev)
    pt = torch.arange(pages_total, dtype=torch.int32, device=dev).reshape(B, pages_per_seq)
    layers = []
    with torch.cuda.stream(stream):
        for l in range(L):
            k = torch.empty(H, pages_total, P, d, dtype=torch.int16, device=dev)
            v = torch.empty_like(k)
            q = torch.empty(B, H * G, d, dtype=torch.int16, device=dev)
            sid = (rank * L + l) * 3
            fill_synthetic_bf16(k, SEED, sid, stream)
            fill_synthetic_bf16(v, SEED, sid + 1, stream)
            fill_synthetic_bf16(q, SEED, sid + 2, stream)
            out = torch.empty(B, H * G, d, dtype=torch.float32, device=dev)
            da.set_assignment(l, assignment)
            da.bind(l, k, v, pt, [n] * B)
            da.build_store(l, stream)
            layers.append(dict(k=k, v=v, q=q, out=out))
    stream.synchronize()
    trace("layers built")
    info = da.layer_info(0)
    step_bytes, select_bytes, attn_kv_bytes = algorithmic_bytes(w, info.kv_bytes_selected, info.total_centroids, B)
    step_bytes *= w.get("layers_per_step", 1)  # every layer of a step reads its own store and KV
    attn_bytes = attn_kv_bytes + B * H * G * d * (2 + 4)

    # one CUDA graph per step (select + attend of layers_per_step layers) and, per
    # layer, attention-only and selection-only graphs for the kernel breakdown
    lps = w.get("layers_per_step", 1)
    graphs, sel_graphs, att_graphs = [], [], []
    launches_before = da.launch_count()
    with torch.cuda.stream(stream):
        for l in range(L):  # eager warm-up (also initialises the selection buffers)
            da.decode_step(l, layers[l]["q"], layers[l]["out"], stream)
    stream.synchronize()
    per_step_launches = (da.launch_count() - launches_before) // L * lps
    trace("eager warm-up done")
    for first in range(0, L, lps):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for l in range(first, first + lps):
                da.decode_step(l, layers[l]["q"], layers[l]["out"], stream)
        graphs.append(g)
    for l in range(L):
        _, stride, _ = da.last_selection(l)
        ga = torch.cuda.CUDAGraph()
        with torch.cuda.graph(ga, stream=stream):
            da.attend_selected(l, layers[l]["q"], layers[l]["out"], stream)
        att_graphs.append(ga)
        sel_blocks = torch.empty(B, H, stride, dtype=torch.int32, device=dev)
        sel_counts = torch.empty(B, H, dtype=torch.int32, device=dev)
        gs = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gs, stream=stream):
            da.select(l, layers[l]["q"], sel_blocks, sel_counts, stream)
        sel_graphs.append((gs, sel_blocks, sel_counts))

    def timed(fn, steps, warm):
        with torch.cuda.stream(stream):
            for i in range(warm):
                fn(i)
        stream.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for i in range(steps):
                fn(i)
            e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    K, W = args.steps, max(args.warmup, 3)
    trace("graphs captured")
    sampler = ClockSampler(local)
    with sampler:
        ms_step = timed(lambda i: graphs[i % len(graphs)].replay(), K, W)
    trace(f"step timed: {ms_step * 1e3:.1f} us")
    ms_attn = timed(lambda i: att_graphs[i % L].replay(), K, W)
    trace(f"attend timed: {ms_attn * 1e3:.1f} us")
    ms_sel = timed(lambda i: sel_graphs[i % L][0].replay(), K, W)
    trace(f"select timed: {ms_sel * 1e3:.1f} us")

    # end to end through the public C ABI with host buffers
    q_host = [torch.empty(B, H * G, d, dtype=torch.int16).pin_memory() for _ in range(L)]
    for l in range(L):
        q_host[l].copy_(layers[l]["q"].cpu())
    out_host = torch.empty(B, H * G, d, dtype=torch.float32).pin_memory()
    def host_step(i):
        first = (i * lps) % L
        for l in range(first, first + lps):
            da.decode_step_host(l, q_host[l], out_host, stream)

    for i in range(max(W, L // lps)):  # every layer's host graph is captured before timing
        host_step(i)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(K):
        host_step(i)
    e2e_s = (time.perf_counter() - t0) / K
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    trace(f"e2e timed: {e2e_s * 1e6:.1f} us")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res, err = cpu_reference(w, args.cpu_reps, 1)
        if res:
            cpu = {"value": 1.0 / (res["seconds_per_sequence"] * lps), "unit": "tokens/s", "cores": res["cores"],
                   "kind": "reference",
                   "sample": f"1 of {B} sequences ({n} ctx, layer 0), median of {args.cpu_reps} after 1 warm-up; "
                             f"OMP over all host cores; tokens/s = 1 / (per-sequence per-layer time x {lps} layers)"}
        else:
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "reference", "sample": err}

    if rank == 0:
        import json as _json
        peaks = _json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
        peak = float(peaks.get("hbm_gbs", 6650.0))
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"
        tokens = B * world
        value = tokens / (ms_step / 1e3)
        attn_gbs = attn_bytes / (ms_attn / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": args.workload, "desc": w["desc"], "batch_per_gpu": B, "global_batch": tokens,
                       "seq_len": n, "kv_heads": H, "q_heads": H * G, "head_dim": d, "page_size": P,
                       "block_sizes": assignment.block_sizes, "token_budget": T, "quant": "int4xasym",
                       "centroids": "mean", "layers_rotated": L, "layers_per_step": lps,
                       "l2": f"{L} rotating layers x {step_bytes / 1e6:.0f} MB algorithmic bytes per step (> 126 MB L2)",
                       "parallelism": f"batch-sharded x{world}, no collective",
                       "compute": "int4 codes -> exact fp32 scores; bf16 MMA (mma.sync) fp32 accumulate"},
            "roofline": {"bound": "hbm", "kernel": "k_attn (absp_attend_selected: paged flash-decode + fused LSE merge)",
                         "achieved": attn_gbs, "peak": peak, "unit": "GB/s", "frac": attn_gbs / peak,
                         "traffic": measured_traffic(args.workload), "bytes_per_launch": attn_bytes,
                         "peak_source": peak_src},
            "step_roofline": {"bytes_per_step": step_bytes, "achieved_gbs": step_bytes / (ms_step / 1e3) / 1e9,
                              "frac": step_bytes / (ms_step / 1e3) / 1e9 / peak},
            "kernels_us": {"step": ms_step * 1e3, "select": ms_sel * 1e3, "attend": ms_attn * 1e3,
                           "select_bytes": select_bytes},
            "cpu_baseline": cpu,
            "e2e": {"value": tokens / e2e_s, "unit": "tokens/s",
                    "h2d_bytes_per_step": B * H * G * d * 2 * lps, "d2h_bytes_per_step": B * H * G * d * 4 * lps,
                    "ms_per_step": e2e_s * 1e3},
            "gpu_launches": per_step_launches * K,
            "clocks": sampler.summary(),
        }
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
