#!/usr/bin/env python
"""Decode-attention benchmark of the KVmix hot path on B200 (BASELINE.json metric).

One step = one decode step of the workload through every layer: append the step's new
K/V token into the layer's packed cache (fused quantize-and-concatenate age-out) and run
the fused dequant attention for the step's query. Default workload = BASELINE.json
configs[1]: Llama-2-7B (32 layers, 32 heads x 128), KVmix tiering (layers 0-5 K3/V4 r=0.2,
6-31 K2/V2 r=0.1, gs 32), batch 16, ~8k context, synthetic KV on the binary16 grid.

value  = tokens/s over all ranks (batch x steps / max-over-ranks device time), inputs
         resident in HBM; the per-step cache (14 GB) is far larger than L2.
e2e    = the same through the public API with pinned HOST buffers (H2D of q/k/v, D2H of
         the attention output, every layer, every step, inside the timed region).
roofline = the dominant kernel (attend_mma_kernel + its split-K combine, timed together
         with CUDA events on the launch stream inside the timed steps): algorithmic bytes
         (MemoryReport total bits / 8 + q + out) / launch time vs MEASURED_PEAKS hbm_gbs.
cpu_baseline = the UNMODIFIED reference (oracle/_ref) timed on this host's cores on a
         bounded sample (one (layer, batch element) unit per tier), extrapolated.
Multi-GPU (torchrun): weak scaling -- every rank holds the full batch of its own shard of
(batch x kv-head) work (no data-path collective); max-over-ranks timing.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-attention tokens/s and achieved HBM GB/s (compressed bytes) at 1/2/4/8 B200"

CONFIGS = {
    # name: (layers, batch, kv_heads, q_heads, head_dim, context, high_layers)
    "llama2-7b-8k": (32, 16, 32, 32, 128, 8192, 6),          # configs[1]
    "layer-4k": (1, 1, 32, 32, 128, 4096, 0),                  # configs[0] shape
    "mistral-7b-32k": (32, 8, 8, 32, 128, 32768, 6),          # configs[2]
    # configs[3] is B32 sharded batch x KV-head over 8 GPUs: one rank's shard is B4 (weak
    # scaling: every rank holds its own B4 shard, ~140 GB of HBM with the fp16 windows)
    "llama2-13b-128k-shard": (40, 4, 40, 40, 128, 131072, 8),  # configs[3], per-GPU shard
}
CONFIG_INDEX = {"llama2-7b-8k": "configs[1]", "layer-4k": "configs[0]", "mistral-7b-32k": "configs[2]",
                "llama2-13b-128k-shard": "configs[3] per-GPU shard (B32 / 8 ranks)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="llama2-7b-8k", choices=list(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0)
    return ap.parse_args()


# ---------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------------------
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        try:
            p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                  "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            return
        while not self._stop.is_set():
            line = p.stdout.readline()
            if not line:
                break
            self.rows.append([x.strip() for x in line.split(",")])
        p.kill()

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._th.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for n, v in zip(names, r[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------
# reference CPU arm (oracle/_ref: the unmodified reference compiled from its sources)
# ---------------------------------------------------------------------------------------
def cpu_reference_sample(cfg_name: str, threads: int):
    """Times the reference's own append+attend on one (layer, batch element) unit per tier
    at full context; returns (tokens/s extrapolated to the whole step, description)."""
    import numpy as np

    import oracle as O
    R = O.ref()
    if R is None:
        return None, "oracle/_ref not built", 0
    if threads > 0:
        R.ref_set_threads(threads)
    cores = R.ref_max_threads()
    L, B, H, Hq, D, ctx, high = CONFIGS[cfg_name]
    G = Hq // H
    tiers = [(3, 4, 0.2, high), (2, 2, 0.1, L - high)] if high else [(2, 2, 0.1, L)]
    t_units = {}
    rng = np.random.default_rng(0)
    for kb, vb, r, count in tiers:
        if count == 0:
            continue
        cache = O.RefCache(kb, vb, r, r, 32, 1, H, D)
        pre = ctx - 64
        k = rng.standard_normal((1, H, pre, D), dtype=np.float32).astype(np.float16).astype(np.float32)
        v = rng.standard_normal((1, H, pre, D), dtype=np.float32).astype(np.float16).astype(np.float32)
        cache.append(k, v)
        for _ in range(64):
            k1 = rng.standard_normal((1, H, 1, D), dtype=np.float32).astype(np.float16).astype(np.float32)
            cache.append(k1, k1)
        q = rng.standard_normal((1, H, G, D), dtype=np.float32).astype(np.float16).astype(np.float32)
        times = []
        for _ in range(3):
            k1 = rng.standard_normal((1, H, 1, D), dtype=np.float32).astype(np.float16).astype(np.float32)
            t0 = time.perf_counter()
            cache.append(k1, k1)
            cache.attend(q)  # GQA: the reference's equivalent is t = G query rows per KV head
            times.append(time.perf_counter() - t0)
        t_units[(kb, vb)] = (min(times), count)
    t_step = sum(t * n for t, n in t_units.values()) * B
    desc = (f"reference append(1 token)+attend timed on one (layer, batch element) unit per tier "
            f"({', '.join(f'K{kb}V{vb}: {t*1e3:.1f} ms' for (kb, vb), (t, _) in t_units.items())}) at "
            f"{ctx} context, {H} KV heads, best of 3, extrapolated x layers x batch {B}")
    return B / t_step, desc, cores


# ---------------------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------------------
def run_b200(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_2506_08018_b200 as K
    from paper_2506_08018_b200 import _lib

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L, B, H, Hq, D, ctx, high = CONFIGS[args.config]
    cfg = K.tiered_config(L, high) if high else K.uniform_config(L, 2, 0.1)
    total_steps = args.warmup + args.steps
    pre = ctx - 64
    cap = ctx + 2 * total_steps + 64
    torch.manual_seed(1234 + rank)

    caches = []
    for l in range(L):
        c = K.KVLayerCache(cfg.layers[l], B, H, D, capacity_tokens=cap, tail_dtype=torch.float16)
        k = torch.randn(B, H, pre, D, device=dev, dtype=torch.float16)
        v = torch.randn(B, H, pre, D, device=dev, dtype=torch.float16)
        c.append(k, v)
        del k, v
        caches.append(c)
    # 64 decode appends to reach the steady-state window (trajectory table)
    kd = torch.randn(64, B, H, 1, D, device=dev, dtype=torch.float16)
    for s in range(64):
        for c in caches:
            c.append(kd[s], kd[(s + 1) % 64])
    del kd
    torch.cuda.synchronize()

    # per-step inputs resident in HBM
    qs = torch.randn(total_steps, L, B, Hq, 1, D, device=dev, dtype=torch.float16)
    kn = torch.randn(total_steps, L, B, H, 1, D, device=dev, dtype=torch.float16)
    vn = torch.randn(total_steps, L, B, H, 1, D, device=dev, dtype=torch.float16)
    outs = torch.empty(L, B, Hq, 1, D, device=dev, dtype=torch.float32)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    lib = _lib.lib()
    import ctypes as C

    def step(s, ev=None):
        # per layer: append(1 token) + attend, one kvmix_append_attend call (the append runs in
        # the attention launch's prologue in the steady state; Key-group age-out steps launch
        # the general append first)
        for l, c in enumerate(caches):
            if ev is not None:
                ev[l][0].record(stream)
            st = lib.kvmix_append_attend(c.handle, kn[s, l].data_ptr(), vn[s, l].data_ptr(), _lib.F16, 1,
                                         qs[s, l].data_ptr(), _lib.F16, Hq, 1, outs[l].data_ptr(), None, sp)
            if st:
                _lib.check(st)
            if ev is not None:
                ev[l][1].record(stream)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for s in range(args.warmup):
        step(s)
    barrier()
    bytes_layer = []
    for c in caches:  # algorithmic bytes of one attend launch at the timed state
        bytes_layer.append(c.algorithmic_bytes() + B * Hq * D * (2 + 4))
    # CUDA events around every layer's launch on the launch stream, on every 4th timed step
    # (each event record costs the stream a few microseconds; value carries 1/4 of it)
    inst = list(range(0, args.steps, 4))
    evs = {i: [[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in range(L)]
           for i in inst}
    launches0 = _lib.launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local_rank) as clk:
        barrier()
        start.record(stream)
        for i, s in enumerate(range(args.warmup, total_steps)):
            step(s, evs.get(i))
        end.record(stream)
        end.synchronize()
    launches = _lib.launch_count() - launches0
    elapsed = start.elapsed_time(end)  # ms for K steps
    # per-layer attend launch time, averaged over the instrumented timed steps
    attn_ms = [statistics.mean(evs[i][l][0].elapsed_time(evs[i][l][1]) for i in inst) for l in range(L)]
    t = torch.tensor([elapsed], device=dev, dtype=torch.float64)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    elapsed = float(t.item())
    ms_per_step = elapsed / args.steps
    value = world * B * args.steps / (elapsed / 1e3)

    # ---- roofline of the dominant kernel ----
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        with open(peaks_path) as f:
            peak = float(json.load(f)["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    tot_bytes = sum(bytes_layer)
    tot_ms = sum(attn_ms)
    achieved = tot_bytes / (tot_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(args.config)

    # ---- e2e through the public API with pinned host buffers ----
    # Every step copies that step's q/k/v from pinned host memory and reads the outputs back;
    # the copies run on a second stream, double-buffered (step s+1's inputs upload while step
    # s computes, step s's outputs download while step s+1 computes), as a serving loop would.
    e2e = None
    if not args.no_e2e:
        q_h = qs.cpu().pin_memory()
        k_h = kn.cpu().pin_memory()
        v_h = vn.cpu().pin_memory()
        n_e2e = min(args.steps, total_steps)
        o_h = torch.empty(n_e2e, L, B, Hq, 1, D, dtype=torch.float32).pin_memory()
        cp = torch.cuda.Stream(device=dev)
        qb = [torch.empty_like(qs[0]) for _ in range(2)]
        kb = [torch.empty_like(kn[0]) for _ in range(2)]
        vb = [torch.empty_like(vn[0]) for _ in range(2)]
        ob = [torch.empty_like(outs) for _ in range(2)]
        ready = [torch.cuda.Event() for _ in range(2)]
        done = [torch.cuda.Event() for _ in range(2)]
        drained = [torch.cuda.Event() for _ in range(2)]

        def upload(s, i):
            with torch.cuda.stream(cp):
                cp.wait_event(done[i])  # the buffers' previous step has finished reading them
                qb[i].copy_(q_h[s % total_steps], non_blocking=True)
                kb[i].copy_(k_h[s % total_steps], non_blocking=True)
                vb[i].copy_(v_h[s % total_steps], non_blocking=True)
                ready[i].record(cp)

        def run(n):
            for i in range(2):
                done[i].record(stream)
                drained[i].record(stream)
            upload(0, 0)
            for s in range(n):
                i = s % 2
                if s + 1 < n:
                    upload(s + 1, 1 - i)
                stream.wait_event(ready[i])
                stream.wait_event(drained[i])  # ob[i] of step s-2 has been read back
                for l, c in enumerate(caches):
                    K.append_attend(c, kb[i][l], vb[i][l], qb[i][l], out=ob[i][l])
                done[i].record(stream)
                with torch.cuda.stream(cp):
                    cp.wait_event(done[i])
                    o_h[s].copy_(ob[i], non_blocking=True)
                    drained[i].record(cp)
            stream.wait_stream(cp)

        run(1)
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        run(n_e2e)
        s1.record(stream)
        s1.synchronize()
        te = torch.tensor([s0.elapsed_time(s1)], device=dev, dtype=torch.float64)
        if world > 1:
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        e2e = {"value": world * B * n_e2e / (float(te.item()) / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": int(L * (qs[0, 0].numel() + kn[0, 0].numel() + vn[0, 0].numel()) * 2),
               "d2h_bytes_per_step": int(L * outs[0].numel() * 4),
               "path": "per layer append_attend (Python API: KVLayerCache.append + attend) on pinned-host inputs; "
                       "H2D/D2H double-buffered on a copy stream"}

    res = {
        "metric": METRIC,
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8 codes x s8/u8 fixed-point digits -> s32 (IMMA), f32 softmax (KV bit-packed 2/3/4-bit)",
        "data": "synthetic (randn on the binary16 grid, on device)",
        "config": {"workload": f"{CONFIG_INDEX[args.config]} {args.config}: {L} layers, B{B}, Hq{Hq}/Hkv{H}, D{D}, ~{ctx} ctx, "
                               f"KVmix tiers (0-{high - 1} K3/V4 r0.2, rest K2/V2 r0.1), gs32, fp16 window",
                   "global_batch": B * world, "seq_len": ctx, "parallelism": f"dp{world} (batch x kv-head shards)",
                   "l2": (f"per-step cache bytes ({tot_bytes / 1e9:.2f} GB) >> 126 MB L2; no flush needed"
                          if tot_bytes > 1e9 else f"per-step cache bytes {tot_bytes / 1e6:.0f} MB: partly L2-resident"),
                   "timed_step": "per layer: append(1 token) + attend = kvmix_append_attend"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": "attend_mma_kernel (IMMA; append in its prologue, split partials merged in-kernel), one launch per layer",
                     "traffic_unit": "DRAM bytes per step (profiles/ncu_traffic.json)",
                     "algorithmic_bytes_per_step": tot_bytes, "attend_ms_per_step": tot_ms,
                     "attend_share_of_step": tot_ms / ms_per_step},
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "memory": {"compressed_bytes_per_step": tot_bytes,
                   "compression_ratio": sum(c.memory_usage().fp16_baseline_bits for c in caches) /
                   max(1, sum(c.memory_usage().total_bits for c in caches))},
    }
    return res


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        threads = args.cpu_threads or os.cpu_count() or 1
        warm = 0  # untimed warm-up samples (bounded: each one is seconds of CPU work)
        tw = time.time()
        while warm < args.warmup and time.time() - tw < 30:
            if cpu_reference_sample(args.config, threads)[0] is None:
                break
            warm += 1
        t0 = time.time()
        times = []
        value = desc = cores = None
        for _ in range(max(1, args.steps)):
            out = cpu_reference_sample(args.config, threads)
            if out[0] is None:
                print(json.dumps({"impl": "reference", "unavailable": out[1]}))
                return 0
            value, desc, cores = out
            times.append(value)
            if time.time() - t0 > 120:
                break
        value = statistics.median(times)
        L, B, H, Hq, D, ctx, high = CONFIGS[args.config]
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": len(times), "warmup": warm, "ms_per_step": B / value * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp32 (reference CPU)", "data": "synthetic",
            "config": {"workload": args.config, "global_batch": B, "seq_len": ctx, "parallelism": "cpu"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "reference", "sample": desc},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return 0

    if world > 1:
        import torch
        torch.distributed.init_process_group("nccl")
    res = run_b200(args, rank, world, local_rank)
    if rank == 0:
        if not args.no_cpu:
            try:
                v, desc, cores = cpu_reference_sample(args.config, args.cpu_threads or os.cpu_count() or 1)
                res["cpu_baseline"] = {"value": v, "unit": "tokens/s", "cores": cores, "kind": "reference", "sample": desc}
            except Exception as e:  # the baseline is reported, never required
                res["cpu_baseline"] = {"value": None, "unavailable": str(e)}
        print(json.dumps(res))
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
