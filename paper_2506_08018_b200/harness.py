"""bench-memory / bench-attention drivers over the device caches, with the reference's CSV
schema (harness.cpp:44-141, 222-241; kvmix.cpp:162-217), SURVEY.md §8(f) row f2.

  python -m paper_2506_08018_b200.harness bench-memory --config quant_config.txt --out dir
  python -m paper_2506_08018_b200.harness bench-attention --trials 50 --out dir

The synthetic data stream is the reference's: kvmix::Rng (rng.hpp, splitmix64 + Box-Muller)
rounded through binary16 (harness.cpp:18-24), so the same seed feeds the same tokens.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
import time

import numpy as np
import torch

from .attention import attend, reference_attend
from .cache import KVLayerCache, MemoryReport
from .config import LayerQuantConfig, ModelQuantConfig, read_config

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


class Rng:
    """kvmix::Rng (rng.hpp:9-52): splitmix64; normal() is Box-Muller with a cached spare."""

    GOLDEN = 0x9E3779B97F4A7C15

    def __init__(self, seed: int):
        self.state = seed & 0xFFFFFFFFFFFFFFFF
        self.spare = None

    def _u64(self, n: int) -> np.ndarray:
        k = np.arange(1, n + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = np.uint64(self.state) + k * np.uint64(self.GOLDEN)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        self.state = (self.state + n * self.GOLDEN) & 0xFFFFFFFFFFFFFFFF
        return z

    def next_double(self, n: int) -> np.ndarray:
        return (self._u64(n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

    def uniform_int(self, lo: int, hi: int) -> int:
        return lo + int(self._u64(1)[0] % np.uint64(hi - lo + 1))

    def normal(self, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        i = 0
        if self.spare is not None and n > 0:
            out[0] = self.spare
            self.spare = None
            i = 1
        pairs = (n - i + 1) // 2
        if pairs:
            u = self.next_double(2 * pairs)
            u1, u2 = u[0::2], u[1::2]
            if np.any(u1 <= 0.0):  # the reference redraws u1 (probability 2^-53 per draw)
                raise RuntimeError("Rng.normal: zero draw, sequential path not implemented")
            r = np.sqrt(-2.0 * np.log(u1))
            th = 2.0 * 3.14159265358979323846 * u2
            vals = np.empty(2 * pairs)
            vals[0::2] = r * np.cos(th)
            vals[1::2] = r * np.sin(th)
            take = n - i
            out[i:] = vals[:take]
            if take < 2 * pairs:
                self.spare = float(vals[-1])
        return out


def random_kv_tensor(rng: Rng, b: int, nh: int, t: int, d: int) -> np.ndarray:
    """harness.cpp:18-24: values on the binary16 grid."""
    x = rng.normal(b * nh * t * d).astype(np.float32).astype(np.float16).astype(np.float32)
    return x.reshape(b, nh, t, d)


@dataclasses.dataclass
class BenchMemoryOptions:  # harness.hpp:24-32
    batch: int = 1
    heads: int = 4
    head_dim: int = 64
    prefill: int = 4096
    decode_steps: int = 1024
    seed: int = 1
    emit_every: int = 64


@dataclasses.dataclass
class BenchMemoryRow:
    layer: int
    step: int
    report: MemoryReport


def _aggregate(reports) -> MemoryReport:
    f = ("packed_payload_bits", "metadata_bits", "tail_bits", "total_bits", "fp16_baseline_bits")
    s = {k: sum(getattr(r, k) for r in reports) for k in f}
    ratio = 1.0 if s["total_bits"] == 0 else s["fp16_baseline_bits"] / s["total_bits"]
    return MemoryReport(s["packed_payload_bits"], s["metadata_bits"], s["tail_bits"], s["total_bits"],
                        s["fp16_baseline_bits"], ratio)


def bench_memory(cfg: ModelQuantConfig, opt: BenchMemoryOptions) -> list[BenchMemoryRow]:
    """harness.cpp:44-87 over device caches."""
    cfg.validate()
    if not cfg.layers:
        raise ValueError("bench_memory: empty config")
    if opt.prefill < 1 or opt.decode_steps < 0:
        raise ValueError("bench_memory: need prefill >= 1 and decode_steps >= 0")
    cap = opt.prefill + opt.decode_steps + 8
    caches = [KVLayerCache(lc, opt.batch, opt.heads, opt.head_dim, capacity_tokens=cap) for lc in cfg.layers]
    rows: list[BenchMemoryRow] = []

    def emit(step):
        reps = [c.memory_usage() for c in caches]
        rows.extend(BenchMemoryRow(l, step, r) for l, r in enumerate(reps))
        rows.append(BenchMemoryRow(-1, step, _aggregate(reps)))

    rng = Rng(opt.seed)
    for c in caches:
        k = random_kv_tensor(rng, opt.batch, opt.heads, opt.prefill, opt.head_dim)
        v = random_kv_tensor(rng, opt.batch, opt.heads, opt.prefill, opt.head_dim)
        c.append(k, v)
    emit(0)
    for step in range(1, opt.decode_steps + 1):
        for c in caches:
            c.append(random_kv_tensor(rng, opt.batch, opt.heads, 1, opt.head_dim),
                     random_kv_tensor(rng, opt.batch, opt.heads, 1, opt.head_dim))
        if step % opt.emit_every == 0 or step == opt.decode_steps:
            emit(step)
    return rows


@dataclasses.dataclass
class BenchAttentionOptions:  # harness.hpp:46-52
    trials: int = 50
    seed: int = 1
    heads: int = 4
    head_dim: int = 32
    tokens: int = 512


@dataclasses.dataclass
class AttentionTrialRow:
    bits: int
    trial: int
    mse_vs_fp: float
    fused_ref_maxdev: float
    fused_us: float
    reference_us: float


def bench_attention(opt: BenchAttentionOptions) -> list[AttentionTrialRow]:
    """harness.cpp:89-141 over device caches: uniform 2/3/4-bit caches vs an r=1 cache fed the
    same token stream; fused_us / reference_us are device wall-clock per call (synchronized)."""
    if opt.trials < 1:
        raise ValueError("bench_attention: trials must be >= 1")
    rows = []
    for trial in range(opt.trials):
        for bits in (2, 3, 4):
            seed = opt.seed + trial * 7919
            r = LayerQuantConfig.default_rpc_for_bits(bits)
            qc = LayerQuantConfig(0, bits, bits, r, r)
            fp = LayerQuantConfig(0, bits, bits, 1.0, 1.0)
            cap = opt.tokens + 8
            quant = KVLayerCache(qc, 1, opt.heads, opt.head_dim, capacity_tokens=cap)
            full = KVLayerCache(fp, 1, opt.heads, opt.head_dim, capacity_tokens=cap)
            rng = Rng(seed)
            done = 0
            while done < opt.tokens:
                t = min(opt.tokens - done, rng.uniform_int(1, 128))
                k = random_kv_tensor(rng, 1, opt.heads, t, opt.head_dim)
                v = random_kv_tensor(rng, 1, opt.heads, t, opt.head_dim)
                quant.append(k, v)
                full.append(k, v)
                done += t
            q = torch.from_numpy(random_kv_tensor(rng, 1, opt.heads, 1, opt.head_dim)).cuda()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fused = attend(q, quant).output
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            ref = reference_attend(q, quant).output
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            fullo = attend(q, full).output
            a = fused.double().cpu().numpy().ravel()
            b = ref.double().cpu().numpy().ravel()
            f = fullo.double().cpu().numpy().ravel()
            mse = float(np.mean((a - f) ** 2))
            denom = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-7)
            maxdev = float(np.max(np.abs(a - b) / denom))
            rows.append(AttentionTrialRow(bits, trial, mse, maxdev, (t1 - t0) * 1e6, (t2 - t1) * 1e6))
    return rows


def write_memory_csv(os_, rows, manifest_ref: str = "manifest.json") -> None:
    """harness.cpp:222-231 (17 significant digits)."""
    os_.write("layer,step,payload_bits,metadata_bits,tail_bits,ratio,manifest\n")
    for r in rows:
        os_.write(f"{r.layer},{r.step},{r.report.packed_payload_bits},{r.report.metadata_bits},"
                  f"{r.report.tail_bits},{r.report.compression_ratio:.17g},{manifest_ref}\n")


def write_attention_csv(os_, rows, manifest_ref: str = "manifest.json") -> None:
    """harness.cpp:233-241."""
    os_.write("bits,trial,mse_vs_fp,fused_ref_maxdev,fused_us,reference_us,manifest\n")
    for r in rows:
        os_.write(f"{r.bits},{r.trial},{r.mse_vs_fp:.17g},{r.fused_ref_maxdev:.17g},{r.fused_us:.17g},"
                  f"{r.reference_us:.17g},{manifest_ref}\n")


def _manifest(out_dir: str, command: str, seed: int, flags: dict, files: list) -> None:
    with open(os.path.join(out_dir, "manifest.json"), "w") as f:
        json.dump({"command": command, "seed": seed, "flags": flags, "files": files,
                   "device": torch.cuda.get_device_name(0)}, f, indent=1)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="kvmix-b200 harness")
    sub = ap.add_subparsers(dest="cmd", required=True)
    bm = sub.add_parser("bench-memory", help="stream synthetic KV, report compression")
    bm.add_argument("--config", required=True)
    bm.add_argument("--seed", type=int, default=1)
    bm.add_argument("--prefill", type=int, default=4096)
    bm.add_argument("--decode-steps", type=int, default=1024)
    bm.add_argument("--batch", type=int, default=1)
    bm.add_argument("--heads", type=int, default=4)
    bm.add_argument("--head-dim", type=int, default=64)
    bm.add_argument("--emit-every", type=int, default=64)
    bm.add_argument("--out", required=True)
    ba = sub.add_parser("bench-attention", help="fused vs reference attention accuracy/latency")
    ba.add_argument("--config", default="")
    ba.add_argument("--trials", type=int, default=50)
    ba.add_argument("--seed", type=int, default=1)
    ba.add_argument("--heads", type=int, default=4)
    ba.add_argument("--head-dim", type=int, default=32)
    ba.add_argument("--tokens", type=int, default=512)
    ba.add_argument("--out", required=True)
    a = ap.parse_args(argv)
    os.makedirs(a.out, exist_ok=True)
    if a.cmd == "bench-memory":
        with open(a.config) as f:
            cfg = read_config(f)
        opt = BenchMemoryOptions(a.batch, a.heads, a.head_dim, a.prefill, a.decode_steps, a.seed, a.emit_every)
        rows = bench_memory(cfg, opt)
        with open(os.path.join(a.out, "memory.csv"), "w") as f:
            write_memory_csv(f, rows)
        _manifest(a.out, "bench-memory", a.seed, dataclasses.asdict(opt) | {"config": a.config}, ["memory.csv"])
        print(f"bench-memory: {len(cfg.layers)} layers, {a.prefill + a.decode_steps} tokens; final cache compression "
              f"{rows[-1].report.compression_ratio}x\nwrote {os.path.join(a.out, 'memory.csv')}")
    else:
        if a.config:
            with open(a.config) as f:
                read_config(f)  # validated; trials sweep the uniform widths (kvmix.cpp:188-190)
        opt = BenchAttentionOptions(a.trials, a.seed, a.heads, a.head_dim, a.tokens)
        rows = bench_attention(opt)
        with open(os.path.join(a.out, "attention_bench.csv"), "w") as f:
            write_attention_csv(f, rows)
        _manifest(a.out, "bench-attention", a.seed, dataclasses.asdict(opt) | {"config": a.config},
                  ["attention_bench.csv"])
        mse = {b: np.mean([r.mse_vs_fp for r in rows if r.bits == b]) for b in (2, 3, 4)}
        print(f"bench-attention: {a.trials} trials; mean MSE vs fp16-cache 2-bit={mse[2]:g} 3-bit={mse[3]:g} "
              f"4-bit={mse[4]:g}\nfused vs reference max deviation {max(r.fused_ref_maxdev for r in rows):g}; "
              f"mean wall-clock fused={np.mean([r.fused_us for r in rows]):g}us "
              f"reference={np.mean([r.reference_us for r in rows]):g}us\n"
              f"wrote {os.path.join(a.out, 'attention_bench.csv')}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
