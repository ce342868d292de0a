#!/usr/bin/env python
"""Decode-attention benchmark of the KVmix hot path on B200 (BASELINE.json metric).

One step = one decode step of the workload through every layer: append the step's new
K/V token into the layer's packed cache (fused quantize-and-concatenate age-out) and run
the fused dequant attention for the step's query. Default workload = BASELINE.json
configs[1]: Llama-2-7B (32 layers, 32 heads x 128), KVmix tiering (layers 0-5 K3/V4 r=0.2,
6-31 K2/V2 r=0.1, gs 32), batch 16, ~8k context, synthetic KV on the binary16 grid.

value  = tokens/s over all ranks (global batch x steps / max-over-ranks device time),
         inputs resident in HBM; the per-step cache (14 GB) is far larger than L2.
e2e    = the same through the public API (DecodeStep: kvmix_append_attend_layers) with
         pinned HOST buffers: H2D of q/k/v and D2H of every layer's attention output, every
         step, inside the timed region.
roofline = the dominant kernel (attend_mma_kernel, which also runs the 1-token append in
         its prologue): algorithmic bytes (MemoryReport total bits / 8 + q + out) per launch
         / launch time from CUDA events on the launch stream inside the timed steps, vs
         MEASURED_PEAKS hbm_gbs. `step_frac` is the same over the whole step time (the
         timed steps overlap consecutive layers' launches: programmatic dependent launch).
cpu_baseline = the UNMODIFIED reference (oracle/_ref) timed on this host's cores on a
         bounded sample (one (layer, batch rows) unit per tier), extrapolated.
Multi-GPU (--gpus N, or under torchrun): the global batch is sharded batch x kv-head with
         ShardPlan (no data-path collective); strong scaling for configs[1]/[2] (fixed global
         batch), weak scaling for the configs[3] shard (B4 per GPU, as BASELINE.md 2 says).
--check validates two sampled (layer, b, head) outputs of the last timed step against an
         fp64 evaluation over the cache's bit-exact snapshot (outside the timed region).
--config quant-sweep: BASELINE configs[4], the quantize/pack sweep (bits x group size,
         Keys + Values, [16,32,4096,128] fp16 per GPU, weak scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-attention tokens/s and achieved HBM GB/s (compressed bytes) at 1/2/4/8 B200"
QMETRIC = "quantize/pack throughput (elements/s) and achieved HBM GB/s over 2/3/4 bits x gs 32/64/128"

CONFIGS = {
    # name: (layers, global batch, kv_heads, q_heads, head_dim, context, high layers, scaling)
    "llama2-7b-8k": (32, 16, 32, 32, 128, 8192, 6, "strong"),           # configs[1]
    "layer-4k": (1, 1, 32, 32, 128, 4096, 0, "strong"),                   # configs[0] shape
    "mistral-7b-32k": (32, 8, 8, 32, 128, 32768, 6, "strong"),          # configs[2]
    # configs[3] is B32 sharded batch x KV-head over 8 GPUs; it does not fit below ~4 GPUs,
    # so every rank holds the 1/8 shard (B4, ~140 GB with the fp16 windows): weak scaling
    "llama2-13b-128k-shard": (40, 4, 40, 40, 128, 131072, 8, "weak"),   # configs[3], per-GPU shard
}
CONFIG_INDEX = {"llama2-7b-8k": "configs[1]", "layer-4k": "configs[0]", "mistral-7b-32k": "configs[2]",
                "llama2-13b-128k-shard": "configs[3] per-GPU shard (B32 / 8 ranks)", "quant-sweep": "configs[4]"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="llama2-7b-8k", choices=list(CONFIGS) + ["quant-sweep"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true")
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


def _share_gpu() -> bool:
    """KVMIX_BENCH_SHARE_GPU=1: every rank on cuda:0 with gloo for the host-side reductions -- the
    N-rank code path on a 1-GPU box (numbers are not a scaling measurement then)."""
    return os.environ.get("KVMIX_BENCH_SHARE_GPU") == "1"


def reduce_max(x: float, world: int, dev, op="max") -> float:
    """max (or sum) over ranks of a host scalar, through the process group."""
    import torch
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if _share_gpu() else dev)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX if op == "max" else torch.distributed.ReduceOp.SUM)
    return float(t.item())


def peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------------------
# reference CPU arm (oracle/_ref: the unmodified reference compiled from its sources)
# ---------------------------------------------------------------------------------------
def cpu_reference_sample(cfg_name: str, threads: int):
    """Times the reference's own append+attend on one (layer, batch rows) unit per tier at
    full context; returns (tokens/s extrapolated to the whole step, description, cores).
    The unit holds enough batch rows that the reference's OpenMP row loop
    (attention.cpp:38-41, one row per (b, head, query)) has work for every thread."""
    import numpy as np

    import oracle as O
    R = O.ref()
    if R is None:
        return None, "oracle/_ref not built", 0
    if threads > 0:
        R.ref_set_threads(threads)
    cores = R.ref_max_threads()
    L, Bg, H, Hq, D, ctx, high, _ = CONFIGS[cfg_name]
    G = Hq // H
    bu = max(1, min(Bg, -(-cores // H)))  # batch rows per unit: >= one row per thread
    tiers = [(3, 4, 0.2, high), (2, 2, 0.1, L - high)] if high else [(2, 2, 0.1, L)]
    t_units = {}
    rng = np.random.default_rng(0)
    for kb, vb, r, count in tiers:
        if count == 0:
            continue
        cache = O.RefCache(kb, vb, r, r, 32, bu, H, D)
        pre = ctx - 64
        k = rng.standard_normal((bu, H, pre, D), dtype=np.float32).astype(np.float16).astype(np.float32)
        v = rng.standard_normal((bu, H, pre, D), dtype=np.float32).astype(np.float16).astype(np.float32)
        cache.append(k, v)
        del k, v
        for _ in range(64):
            k1 = rng.standard_normal((bu, H, 1, D), dtype=np.float32).astype(np.float16).astype(np.float32)
            cache.append(k1, k1)
        q = rng.standard_normal((bu, H, G, D), dtype=np.float32).astype(np.float16).astype(np.float32)
        times = []
        for _ in range(3):
            k1 = rng.standard_normal((bu, H, 1, D), dtype=np.float32).astype(np.float16).astype(np.float32)
            t0 = time.perf_counter()
            cache.append(k1, k1)
            cache.attend(q)  # GQA: the reference's equivalent is t = G query rows per KV head
            times.append(time.perf_counter() - t0)
        t_units[(kb, vb)] = (min(times), count)
    t_step = sum(t * n for t, n in t_units.values()) * Bg / bu
    desc = (f"reference append(1 token)+attend timed on one (layer, {bu} batch row{'s' if bu > 1 else ''}) unit per "
            f"tier ({', '.join(f'K{kb}V{vb}: {t*1e3:.1f} ms' for (kb, vb), (t, _) in t_units.items())}) at {ctx} "
            f"context, {H} KV heads x {G} query rows, best of 3, extrapolated x {L} layers x batch {Bg}")
    return Bg / t_step, desc, cores


def cpu_quant_sample(threads: int):
    """The reference's quantize_key_tensor + quantize_value_tensor (quant.cpp:102-124) on
    [1,32,4096,128] (one of the 16 batch rows of a configs[4] tensor) for one setting per bit
    width at gs 32; returns (elements/s, description, cores)."""
    import numpy as np

    import oracle as O
    R = O.ref()
    if R is None:
        return None, "oracle/_ref not built", 0
    if threads > 0:
        R.ref_set_threads(threads)
    cores = R.ref_max_threads()
    import ctypes as C
    x = np.random.default_rng(0).standard_normal((1, 32, 4096, 128), dtype=np.float32).astype(np.float16).astype(np.float32)
    tot_t, tot_n, parts = 0.0, 0, []
    for bits in (2, 3, 4):
        nw = O.words_for(x.size, bits)
        bufs = [(np.zeros(nw, np.uint32), np.zeros(2 * (x.size // 32), np.uint16)) for _ in range(2)]
        cnt = C.c_uint64(0)
        t0 = time.perf_counter()
        for key, (w, m) in zip((0, 1), bufs):  # one reference call per side (outputs preallocated)
            if R.ref_quantize(key, x, *x.shape, bits, 32, w.ctypes.data, m.ctypes.data, C.byref(cnt), C.byref(cnt)):
                raise RuntimeError(R.ref_last_error().decode())
        dt = time.perf_counter() - t0
        tot_t += dt
        tot_n += 2 * x.size
        parts.append(f"{bits}-bit {dt * 1e3:.0f} ms")
    return tot_n / tot_t, (f"reference quantize_key_tensor + quantize_value_tensor on [1,32,4096,128] fp32 "
                           f"(binary16 grid), gs 32, bits 2/3/4 ({', '.join(parts)})"), cores


# ---------------------------------------------------------------------------------------
# B200 arm: decode step
# ---------------------------------------------------------------------------------------
def run_b200(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_2506_08018_b200 as K
    from paper_2506_08018_b200 import _lib
    from paper_2506_08018_b200.shard import ShardPlan

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L, Bg, H, Hq, D, ctx, high, scaling = CONFIGS[args.config]
    if scaling == "weak":  # every rank holds its own shard of the global batch
        plan = ShardPlan(Bg * world, H, Hq, world, rank, mode="batch")
    else:
        plan = ShardPlan(Bg, H, Hq, world, rank)
    B, Hl, Hql = plan.local_batch, plan.local_heads, plan.local_heads * (Hq // H)
    B_glob = plan.B
    cfg = K.tiered_config(L, high) if high else K.uniform_config(L, 2, 0.1)
    total_steps = args.warmup + args.steps
    pre = ctx - 64
    cap = ctx + 2 * total_steps + 64
    torch.manual_seed(1234 + rank)

    # workloads smaller than L2 rotate over R copies of the cache stack (R x bytes > 126 MB), so
    # every timed step reads its cache from HBM (configs[0]: 12.7 MB per step)
    est = L * B * Hl * ctx * D * 0.8
    rot = 1 if est >= 0.25e9 else int(-(-0.3e9 // est))

    def build_stack():
        cs = []
        for l in range(L):
            c = K.KVLayerCache(cfg.layers[l], B, Hl, D, capacity_tokens=cap, tail_dtype=torch.float16)
            plan.place(c)
            k = torch.randn(B, Hl, pre, D, device=dev, dtype=torch.float16)
            v = torch.randn(B, Hl, pre, D, device=dev, dtype=torch.float16)
            c.append(k, v)
            del k, v
            cs.append(c)
        # 64 decode appends to reach the steady-state window (trajectory table)
        kd = torch.randn(64, B, Hl, 1, D, device=dev, dtype=torch.float16)
        for s in range(64):
            for c in cs:
                c.append(kd[s], kd[(s + 1) % 64])
        del kd
        return cs

    stacks = [build_stack() for _ in range(rot)]
    caches = stacks[0]
    torch.cuda.synchronize()

    # per-step inputs resident in HBM
    qs = torch.randn(total_steps, L, B, Hql, 1, D, device=dev, dtype=torch.float16)
    kn = torch.randn(total_steps, L, B, Hl, 1, D, device=dev, dtype=torch.float16)
    vn = torch.randn(total_steps, L, B, Hl, 1, D, device=dev, dtype=torch.float16)
    outs = torch.empty(L, B, Hql, 1, D, device=dev, dtype=torch.float32)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    lib = _lib.lib()
    steps = [K.DecodeStep(stacks[s % rot], list(kn[s]), list(vn[s]), list(qs[s]), list(outs))
             for s in range(total_steps)]

    # layer runs with one kernel instance each (the KVmix tiers): kvmix_append_attend_layers
    # launches each run as ONE multi-layer kernel; instrumented steps call it per run with CUDA
    # events around each call (the same kernels as step(), without the overlap between runs)
    runs = [(0, high), (high, L)] if 0 < high < L else [(0, L)]
    inst_steps = {}

    def step_instrumented(s, ev):
        for j, ds in enumerate(inst_steps[s]):
            ev[j][0].record(stream)
            ds.step(sp)
            ev[j][1].record(stream)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for s in range(args.warmup):
        steps[s].step(sp)
    barrier()
    bytes_layer = [c.algorithmic_bytes() + B * Hql * D * (2 + 4) for c in caches]  # one attend launch each
    # CUDA events around every layer's launch on the launch stream, on every 10th timed step
    # (those steps launch layer by layer, without the programmatic dependent launch that
    # overlaps a layer's start with the previous layer's drain in DecodeStep.step())
    inst = list(range(0, args.steps, 10))
    evs = {i: [[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in runs]
           for i in inst}
    for i in inst:  # (built before the timed region)
        s = args.warmup + i
        inst_steps[s] = [K.DecodeStep(stacks[s % rot][a:b], list(kn[s][a:b]), list(vn[s][a:b]),
                                      list(qs[s][a:b]), list(outs[a:b])) for a, b in runs]
    launches0 = _lib.launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local_rank) as clk:
        barrier()
        start.record(stream)
        for i, s in enumerate(range(args.warmup, total_steps)):
            if i in evs:
                step_instrumented(s, evs[i])
            else:
                steps[s].step(sp)
        end.record(stream)
        end.synchronize()
    launches = _lib.launch_count() - launches0
    elapsed = start.elapsed_time(end)  # ms for K steps
    attn_ms = [statistics.mean(evs[i][j][0].elapsed_time(evs[i][j][1]) for i in inst) for j in range(len(runs))]
    elapsed = reduce_max(elapsed, world, dev)
    ms_per_step = elapsed / args.steps
    value = B_glob * args.steps / (elapsed / 1e3)

    # ---- roofline of the dominant kernel (this rank's launches) ----
    peak, peak_src = peak_hbm()
    tot_bytes = sum(bytes_layer)
    tot_ms = sum(attn_ms)
    achieved = tot_bytes / (tot_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(args.config) if world == 1 else None

    # ---- --check: two sampled (layer, b, head) outputs of the last timed step ----
    check = None
    if not args.no_check:
        check = check_outputs(stacks[(total_steps - 1) % rot], qs[total_steps - 1], outs, Hq // H, rank)

    # ---- e2e through the public API with pinned host buffers ----
    # Every step copies that step's q/k/v from pinned host memory and reads every layer's
    # output back; the copies run on a second stream, double-buffered (step s+1's inputs
    # upload while step s computes, step s's outputs download while step s+1 computes), as a
    # serving loop would. The step itself is DecodeStep.step() (public API).
    e2e = None
    if not args.no_e2e:
        q_h = qs.cpu().pin_memory()
        k_h = kn.cpu().pin_memory()
        v_h = vn.cpu().pin_memory()
        n_e2e = min(args.steps, total_steps)
        o_h = torch.empty(n_e2e, L, B, Hql, 1, D, dtype=torch.float32).pin_memory()
        cp = torch.cuda.Stream(device=dev)
        qb = [torch.empty_like(qs[0]) for _ in range(2)]
        kb = [torch.empty_like(kn[0]) for _ in range(2)]
        vb = [torch.empty_like(vn[0]) for _ in range(2)]
        ob = [torch.empty_like(outs) for _ in range(2)]
        dsteps = [[K.DecodeStep(st, list(kb[i]), list(vb[i]), list(qb[i]), list(ob[i])) for st in stacks]
                  for i in range(2)]
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
                dsteps[i][s % rot].step()
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
        te = reduce_max(s0.elapsed_time(s1), world, dev)
        e2e = {"value": B_glob * n_e2e / (te / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": int(L * (qs[0, 0].numel() + kn[0, 0].numel() + vn[0, 0].numel()) * 2) * world,
               "d2h_bytes_per_step": int(L * outs[0].numel() * 4) * world,
               "path": "DecodeStep.step() (public API, kvmix_append_attend_layers) on pinned-host inputs, every "
                       "layer's output read back; H2D/D2H double-buffered on a copy stream"}

    launches_all = int(reduce_max(float(launches), world, dev, op="sum"))
    hi = f"0-{high - 1} K3/V4 r0.2, rest K2/V2 r0.1" if high else "all K2/V2 r0.1"
    res = {
        "metric": METRIC,
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "u8 codes x s8/u8 fixed-point digits -> s32 (IMMA), f32 softmax (KV bit-packed 2/3/4-bit)",
        "data": "synthetic (randn on the binary16 grid, on device)",
        "config": {"workload": f"{CONFIG_INDEX[args.config]} {args.config}: {L} layers, global B{B_glob}, Hq{Hq}/Hkv{H}, "
                               f"D{D}, ~{ctx} ctx, KVmix tiers ({hi}), gs32, fp16 window",
                   "global_batch": B_glob, "seq_len": ctx,
                   "parallelism": f"{plan.mode} shards x{world} (rank 0: b {plan.b0}-{plan.b1 - 1}, kv heads "
                                  f"{plan.h0}-{plan.h1 - 1}); no data-path collective",
                   "l2": (f"per-step cache bytes per GPU ({tot_bytes / 1e9:.2f} GB) >> 126 MB L2; no flush needed"
                          if rot == 1 else f"per-step cache bytes {tot_bytes / 1e6:.1f} MB < L2: steps rotate over "
                                           f"{rot} copies of the cache stack ({rot * tot_bytes / 1e6:.0f} MB), every "
                                           f"step reads its cache from HBM"),
                   "timed_step": "DecodeStep.step(): per layer append(1 token) + attend (kvmix_append_attend_layers: "
                                 "one multi-layer launch per tier run, the second overlapping the first's drain "
                                 "(programmatic dependent launch))"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": "attend_mma_layers_kernel (IMMA; 1-token append in its prologue, split partials "
                               "merged in-kernel), one launch per run of same-tier layers",
                     "step_frac": tot_bytes / (ms_per_step / 1e3) / 1e9 / peak,
                     "traffic_unit": "DRAM bytes per step (profiles/ncu_traffic.json, 1 GPU)",
                     "algorithmic_bytes_per_step": tot_bytes, "attend_ms_per_step": tot_ms,
                     "attend_share_of_step": tot_ms / ms_per_step},
        "e2e": e2e,
        "gpu_launches": launches_all,
        "clocks": clk.summary(),
        "check": check,
        "memory": {"compressed_bytes_per_step_per_gpu": tot_bytes,
                   "compression_ratio": sum(c.memory_usage().fp16_baseline_bits for c in caches) /
                   max(1, sum(c.memory_usage().total_bits for c in caches))},
    }
    return res


def check_outputs(caches, q_last, outs, G, rank):
    """fp64 attention over the bit-exact snapshot (tests pin it against the reference) of two
    sampled (layer, b, kv-head) slices vs the device output of the last timed step; the
    tolerance is the parity tests' 2e-6 * max|V|."""
    import torch
    res = []
    L = len(caches)
    gen = torch.Generator().manual_seed(7 + rank)
    for l in (0, L - 1) if L > 1 else (0,):
        c = caches[l]
        b = int(torch.randint(0, c.batch(), (1,), generator=gen))
        h = int(torch.randint(0, c.heads(), (1,), generator=gen))
        ks, vs = c.snapshot_dequantized()
        k = ks[b, h].double()
        v = vs[b, h].double()
        del ks, vs
        q = q_last[l, b, h * G:(h + 1) * G, 0].double()  # [G, D]
        s = (q @ k.T) * (1.0 / float(k.shape[1]) ** 0.5)
        ref = torch.softmax(s, dim=-1) @ v
        got = outs[l, b, h * G:(h + 1) * G, 0].double()
        err = float((got - ref).abs().max() / v.abs().max())
        res.append({"layer": l, "b": b, "kv_head": h, "err_over_maxV": err, "ok": err <= 2e-6})
    return {"samples": res, "ok": all(r["ok"] for r in res), "tolerance": "2e-6 * max|V| vs fp64 over the snapshot"}


# ---------------------------------------------------------------------------------------
# B200 arm: configs[4] quantize/pack sweep
# ---------------------------------------------------------------------------------------
def run_quant(args, rank, world, local_rank):
    import torch

    import paper_2506_08018_b200 as K
    from paper_2506_08018_b200 import _lib

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    shape = (16, 32, 4096, 128)  # per GPU (weak scaling)
    n = 1
    for x in shape:
        n *= x
    torch.manual_seed(99 + rank)
    x = torch.randn(shape, device=dev, dtype=torch.float16)
    settings = [(b, gs, key) for b in (2, 3, 4) for gs in (32, 64, 128) for key in (True, False)]
    lib = _lib.lib()
    bufs = {}
    for b, gs, key in settings:
        nw = K.packed_word_count(n, b)
        ng = (n // gs) if key else (n // 128) * ((128 + gs - 1) // gs)
        bufs[(b, gs, key)] = (torch.empty(nw, dtype=torch.int32, device=dev),
                              torch.empty((ng, 2), dtype=torch.int16, device=dev))
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    def one(b, gs, key):
        w, m = bufs[(b, gs, key)]
        st = lib.kvmix_quantize(0 if key else 1, x.data_ptr(), _lib.F16, *shape, b, gs, w.data_ptr(), m.data_ptr(), sp)
        if st:
            _lib.check(st)

    def sweep():
        for s in settings:
            one(*s)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        sweep()
    barrier()
    # per-setting kernel time with CUDA events (inputs 1 GiB >> L2)
    per = {}
    ev = {s: [torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for s in settings}
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _lib.launch_count()
    with Clocks(local_rank) as clk:
        barrier()
        start.record(stream)
        for it in range(args.steps):
            for s in settings:
                if it == args.steps - 1:
                    ev[s][0].record(stream)
                one(*s)
                if it == args.steps - 1:
                    ev[s][1].record(stream)
        end.record(stream)
        end.synchronize()
    launches = _lib.launch_count() - launches0
    elapsed = start.elapsed_time(end)
    elapsed = reduce_max(elapsed, world, dev)
    ms_per_step = elapsed / args.steps  # one step = the whole 18-setting sweep
    elems = n * len(settings) * world
    value = elems * args.steps / (elapsed / 1e3)
    peak, peak_src = peak_hbm()
    rows, tot_bytes, tot_ms = [], 0, 0.0
    for b, gs, key in settings:
        ms = ev[(b, gs, key)][0].elapsed_time(ev[(b, gs, key)][1])
        payload = (4.0 / 11.0) if b == 3 else b / 8.0
        byt = n * (2 + payload + 4.0 / gs)  # fp16 in + packed payload + binary16 (scale, min)
        tot_bytes += byt
        tot_ms += ms
        rows.append({"bits": b, "gs": gs, "side": "K" if key else "V", "ms": ms, "GBps": byt / ms / 1e6,
                     "frac": byt / ms / 1e6 / peak})
    return {
        "metric": QMETRIC, "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp16 in -> u32 packed words + binary16 meta",
        "data": "synthetic (randn fp16, on device)",
        "config": {"workload": "configs[4] quantize/pack sweep: bits {2,3,4} x gs {32,64,128} x {Keys per-channel, "
                               "Values per-token}, [16,32,4096,128] fp16 per GPU (1 GiB input >> L2)",
                   "global_batch": 16 * world, "seq_len": 4096, "parallelism": f"weak x{world}"},
        "roofline": {"bound": "hbm", "achieved": tot_bytes / (tot_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": tot_bytes / (tot_ms / 1e3) / 1e9 / peak, "traffic": None, "peak_source": peak_src,
                     "kernel": "quantize_{key,value}_* kernels (one launch per setting)", "per_setting": rows},
        "e2e": None, "gpu_launches": launches, "clocks": clk.summary(),
    }


def quant_e2e(args, local_rank):
    """configs[4] end to end through the public API (quantize_key_tensor /
    quantize_value_tensor from pinned host fp16, results read back to the host)."""
    import torch

    import paper_2506_08018_b200 as K
    dev = torch.device("cuda", local_rank)
    shape = (16, 32, 4096, 128)
    xh = torch.randn(shape, dtype=torch.float16).pin_memory()
    bits, gs = 2, 32
    n = xh.numel()
    stream = torch.cuda.current_stream()

    def one():
        x = xh.to(dev, non_blocking=True)
        kq = K.quantize_key_tensor(x, K.QuantSpec(bits, K.Grouping.kPerChannelKey, gs))
        vq = K.quantize_value_tensor(x, K.QuantSpec(bits, K.Grouping.kPerTokenValue, gs))
        return [kq.codes.words.cpu(), kq.meta.cpu(), vq.codes.words.cpu(), vq.meta.cpu()]

    one()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(1, min(args.steps, 5))
    s0.record(stream)
    outs = None
    for _ in range(reps):
        outs = one()
    s1.record(stream)
    s1.synchronize()
    ms = s0.elapsed_time(s1) / reps
    d2h = sum(o.numel() * o.element_size() for o in outs)
    return {"value": 2 * n / (ms / 1e3), "unit": "elements/s", "h2d_bytes_per_step": int(n * 2),
            "d2h_bytes_per_step": int(d2h),
            "path": "quantize_key_tensor + quantize_value_tensor (public API), 2-bit gs32, fp16 [16,32,4096,128] "
                    "uploaded from pinned host memory, words + meta read back (the input is uploaded once per "
                    "step and quantized both ways)"}


# ---------------------------------------------------------------------------------------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (rank 0 prints the JSON line)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)

    if args.impl == "reference":
        if rank != 0:
            return 0
        threads = args.cpu_threads or os.cpu_count() or 1
        sample = cpu_quant_sample if args.config == "quant-sweep" else (lambda th: cpu_reference_sample(args.config, th))
        warm = 0  # untimed warm-up samples (bounded: each one is seconds of CPU work)
        tw = time.time()
        while warm < args.warmup and time.time() - tw < 30:
            if sample(threads)[0] is None:
                break
            warm += 1
        t0 = time.time()
        times = []
        value = desc = cores = None
        for _ in range(max(1, args.steps)):
            out = sample(threads)
            if out[0] is None:
                print(json.dumps({"impl": "reference", "unavailable": out[1]}))
                return 0
            value, desc, cores = out
            times.append(value)
            if time.time() - t0 > 120:
                break
        value = statistics.median(times)
        if args.config == "quant-sweep":
            unit, metric, cfgd = "elements/s", QMETRIC, {"workload": "quant-sweep", "global_batch": 16, "seq_len": 4096,
                                                          "parallelism": "cpu"}
            msps = 16 * 32 * 4096 * 128 * 18 / value * 1e3
        else:
            L, Bg, H, Hq, D, ctx, high, scaling = CONFIGS[args.config]
            unit, metric = "tokens/s", METRIC
            cfgd = {"workload": args.config, "global_batch": Bg, "seq_len": ctx, "parallelism": "cpu"}
            msps = Bg / value * 1e3
        print(json.dumps({
            "impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": args.gpus,
            "steps": len(times), "warmup": warm, "ms_per_step": msps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "fp32 (reference CPU)", "data": "synthetic",
            "config": cfgd,
            "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "reference", "sample": desc},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return 0

    if _share_gpu():
        local_rank = 0
    if world > 1:
        import torch
        torch.cuda.set_device(local_rank)
        if _share_gpu():
            torch.distributed.init_process_group("gloo")
        else:
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.config == "quant-sweep":
        res = run_quant(args, rank, world, local_rank)
        if rank == 0 and not args.no_e2e:
            res["e2e"] = quant_e2e(args, local_rank)
            res["e2e"]["value"] *= world
    else:
        res = run_b200(args, rank, world, local_rank)
    if rank == 0:
        if not args.no_cpu:
            try:
                th = args.cpu_threads or os.cpu_count() or 1
                if args.config == "quant-sweep":
                    v, desc, cores = cpu_quant_sample(th)
                    unit = "elements/s"
                else:
                    v, desc, cores = cpu_reference_sample(args.config, th)
                    unit = "tokens/s"
                res["cpu_baseline"] = {"value": v, "unit": unit, "cores": cores, "kind": "reference", "sample": desc}
            except Exception as e:  # the baseline is reported, never required
                res["cpu_baseline"] = {"value": None, "unavailable": str(e)}
        print(json.dumps(res))
    if world > 1:
        import torch
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
