"""KVLayerCache: device-resident per-layer cache (cache.hpp:52-104) over the C ABI.

The shrink-rule bookkeeping and segment list live in the native library (host C++), the
fused quantize-and-concatenate age-out and the full-precision window live on the GPU.
Counters, MemoryReport, snapshot, segment words and the KVCD dump are identical to the
reference's for the same append sequence (tests/test_cache_gpu.py).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import struct

import numpy as np
import torch

from . import _lib
from ._lib import KvmixInvalidArgument, KvmixRuntimeError, LayerConfigC, MemoryReportC, check, lib
from .config import LayerQuantConfig
from .quant import (Grouping, PackedBuffer, PackLayout, QuantizedGroups, QuantSpec, TensorShape, _as_device,
                    _dtype_code, _ptr, _stream, serialize_quantized_groups, deserialize_quantized_groups)


@dataclasses.dataclass
class MemoryReport:
    packed_payload_bits: int = 0
    metadata_bits: int = 0
    tail_bits: int = 0
    total_bits: int = 0
    fp16_baseline_bits: int = 0
    compression_ratio: float = 1.0


def rpc_target(current_rpc: int, r: float) -> int:
    """floor(r * current_rpc) (cache.cpp:30-34)."""
    out = C.c_int64(0)
    check(lib().kvmix_rpc_target(int(current_rpc), float(r), out))
    return out.value


def _cfg_c(cfg: LayerQuantConfig) -> LayerConfigC:
    return LayerConfigC(cfg.layer_index, cfg.key_bits, cfg.value_bits, cfg.key_rpc_ratio, cfg.value_rpc_ratio,
                        cfg.group_size)


class KVLayerCache:
    """KVLayerCache(config, batch, heads, head_dim) over a device reservation.

    capacity_tokens: tokens reserved up front; append() grows the reservation (x2, segments
    and tails re-imported into a new device store) when a call would exceed it, like the
    reference's std::vectors (append_raw, the benchmark's device-pointer path, does not
    grow). tail_dtype: torch.float32 keeps any
    fp32 input exact (the reference's fp32 tail); torch.float16 halves the window and is
    exact for inputs on the binary16 grid (the reference's own regime, helpers.hpp:14-18).
    """

    def __init__(self, config: LayerQuantConfig, batch: int, heads: int, head_dim: int, *,
                 capacity_tokens: int = 8192, tail_dtype=torch.float32, device=None):
        self._h = None
        if device is not None:
            torch.cuda.set_device(device)
        self._cfg = dataclasses.replace(config)
        h = C.c_void_p()
        dt = _lib.F16 if tail_dtype == torch.float16 else _lib.F32
        check(lib().kvmix_cache_create(C.byref(_cfg_c(config)), batch, heads, head_dim, int(capacity_tokens), dt,
                                       C.byref(h)))
        self._h = h
        self._b, self._nh, self._d = batch, heads, head_dim
        self._cap = int(capacity_tokens)
        self._tail_dtype = tail_dtype
        self._device = torch.device("cuda", torch.cuda.current_device())

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().kvmix_cache_destroy(self._h)
            except Exception:
                pass
            self._h = None

    def set_shard(self, global_batch: int, global_heads: int, batch_offset: int, head_offset: int) -> None:
        """Place this cache as the [batch_offset:, head_offset:] slice of a global
        [global_batch, global_heads] cache (multi-GPU shard): Mixed3 narrow slots then follow
        the global stream index, so the shard equals the unsharded cache's slice bit for bit.
        Must precede the first append (kvmix_cache_set_shard)."""
        check(lib().kvmix_cache_set_shard(self._h, int(global_batch), int(global_heads), int(batch_offset),
                                          int(head_offset)))
        self._shard = (int(global_batch), int(global_heads), int(batch_offset), int(head_offset))

    # ---- accessors (cache.hpp:64-76) -------------------------------------------------------
    @property
    def handle(self):
        return self._h

    def _counters(self):
        a = (C.c_int64 * 7)()
        check(lib().kvmix_cache_counters(self._h, a))
        return list(a)

    def total_tokens(self) -> int:
        return self._counters()[0]

    def key_tail_tokens(self) -> int:
        return self._counters()[1]

    def value_tail_tokens(self) -> int:
        return self._counters()[2]

    def quantized_key_tokens(self) -> int:
        return self._counters()[3]

    def quantized_value_tokens(self) -> int:
        return self._counters()[4]

    def batch(self) -> int:
        return self._b

    def heads(self) -> int:
        return self._nh

    def head_dim(self) -> int:
        return self._d

    def config(self) -> LayerQuantConfig:
        return dataclasses.replace(self._cfg)

    def capacity_tokens(self) -> int:
        return self._cap

    # ---- append (cache.cpp:45-80) ----------------------------------------------------------
    def _check_append(self, k, v) -> None:
        if (k.dim() != 4 or v.dim() != 4 or k.shape[0] != self._b or k.shape[1] != self._nh or k.shape[3] != self._d
                or tuple(v.shape[:2]) != (self._b, self._nh) or v.shape[3] != self._d or k.shape[2] != v.shape[2]):
            raise KvmixInvalidArgument("KVLayerCache::append: tensor shape does not match cache")
        if k.shape[2] < 1:
            raise KvmixInvalidArgument("KVLayerCache::append: need at least one token")

    def append(self, new_keys, new_values) -> None:
        k = _as_device(new_keys)
        v = _as_device(new_values)
        self._check_append(k, v)
        if v.dtype != k.dtype:
            v = v.to(k.dtype)
        t = int(k.shape[2])
        if self.total_tokens() + t > self._cap:
            self._grow(max(2 * self._cap, self.total_tokens() + t))
        check(lib().kvmix_cache_append(self._h, _ptr(k), _ptr(v), _dtype_code(k), t, _stream()))

    def _grow(self, cap: int) -> None:
        """Re-create the device store with a larger reservation: the reference segments are
        exported and re-imported in order, then the tails (bit-identical state)."""
        segs = (self.key_segments(), self.value_segments())
        tails = (self._tail(0), self._tail(1))
        h = C.c_void_p()
        dt = _lib.F16 if self._tail_dtype == torch.float16 else _lib.F32
        check(lib().kvmix_cache_create(C.byref(_cfg_c(self._cfg)), self._b, self._nh, self._d, int(cap), dt,
                                       C.byref(h)))
        try:
            if getattr(self, "_shard", None):
                check(lib().kvmix_cache_set_shard(h, *self._shard))
            for side, lst in enumerate(segs):
                for qg in lst:
                    check(lib().kvmix_cache_import_segment(h, side, qg.shape.t, _ptr(qg.codes.words), _ptr(qg.meta),
                                                           _stream()))
            for side, tail in enumerate(tails):
                if tail.shape[0]:
                    check(lib().kvmix_cache_import_tail(h, side, _ptr(tail), int(tail.shape[0]), _stream()))
            torch.cuda.current_stream().synchronize()
        except Exception:
            lib().kvmix_cache_destroy(h)
            raise
        lib().kvmix_cache_destroy(self._h)
        self._h = h
        self._cap = int(cap)

    def append_raw(self, k_ptr: int, v_ptr: int, dtype_code: int, t: int, stream: int) -> None:
        """Device-pointer append without checks or copies (benchmark hot loop)."""
        check(lib().kvmix_cache_append(self._h, k_ptr, v_ptr, dtype_code, t, stream))

    # ---- accounting (cache.cpp:119-134) ----------------------------------------------------
    def memory_usage(self) -> MemoryReport:
        r = MemoryReportC()
        check(lib().kvmix_cache_memory_usage(self._h, C.byref(r)))
        return MemoryReport(r.packed_payload_bits, r.metadata_bits, r.tail_bits, r.total_bits,
                            r.fp16_baseline_bits, r.compression_ratio)

    def algorithmic_bytes(self) -> int:
        out = C.c_uint64(0)
        check(lib().kvmix_cache_algorithmic_bytes(self._h, out))
        return out.value

    # ---- snapshot / segments / tails -------------------------------------------------------
    def snapshot_dequantized(self):
        """cache.cpp:136-173: fp32 [B,H,T,D] keys and values, bit-exact."""
        T = self.total_tokens()
        keys = torch.empty((self._b, self._nh, T, self._d), dtype=torch.float32, device=self._device)
        values = torch.empty_like(keys)
        check(lib().kvmix_cache_snapshot(self._h, _ptr(keys), _ptr(values), _stream()))
        return keys, values

    def _segment(self, side: int, idx: int) -> QuantizedGroups:
        info = (C.c_int64 * 3)()
        check(lib().kvmix_cache_segment_info(self._h, side, idx, info))
        t, nw, ng = info
        words = torch.zeros(max(1, nw), dtype=torch.int32, device=self._device)
        meta = torch.zeros((max(1, ng), 2), dtype=torch.int16, device=self._device)
        check(lib().kvmix_cache_export_segment(self._h, side, idx, _ptr(words), _ptr(meta), _stream()))
        bits = self._cfg.key_bits if side == 0 else self._cfg.value_bits
        spec = QuantSpec(bits, Grouping(side), self._cfg.group_size)
        n = self._b * self._nh * t * self._d
        return QuantizedGroups(meta[:ng], PackedBuffer(words[:nw], PackLayout.kMixed3 if bits == 3 else PackLayout.kUniform,
                                                       bits, n), spec, TensorShape(self._b, self._nh, t, self._d))

    def key_segments(self) -> list[QuantizedGroups]:
        return [self._segment(0, i) for i in range(self._counters()[5])]

    def value_segments(self) -> list[QuantizedGroups]:
        return [self._segment(1, i) for i in range(self._counters()[6])]

    def _tail(self, side: int) -> torch.Tensor:
        n = self._counters()[1 + side]
        out = torch.zeros((n, self._b, self._nh, self._d), dtype=torch.float32, device=self._device)
        check(lib().kvmix_cache_export_tail(self._h, side, _ptr(out), _stream()))
        return out

    def key_tail(self) -> torch.Tensor:
        """[tail, B, H, D] fp32, oldest first (key_tail_at, cache.hpp:79-82)."""
        return self._tail(0)

    def value_tail(self) -> torch.Tensor:
        return self._tail(1)

    def reset(self) -> None:
        check(lib().kvmix_cache_reset(self._h, _stream()))

    # ---- KVCD dump / load (cache.cpp:190-281) ----------------------------------------------
    def dump(self) -> bytes:
        c = self._cfg
        cnt = self._counters()
        out = bytearray(b"KVCD")
        out += struct.pack("<BiBBffIIIIqqqq", 1, c.layer_index, c.key_bits, c.value_bits, c.key_rpc_ratio,
                           c.value_rpc_ratio, c.group_size, self._b, self._nh, self._d, cnt[1], cnt[2], cnt[3], cnt[4])
        for segs in (self.key_segments(), self.value_segments()):
            out += struct.pack("<I", len(segs))
            for qg in segs:
                b = serialize_quantized_groups(qg)
                out += struct.pack("<Q", len(b)) + b
        for tail in (self.key_tail(), self.value_tail()):
            out += struct.pack("<Q", tail.numel()) + tail.cpu().numpy().astype("<f4").tobytes()
        return bytes(out)

    @staticmethod
    def load(data: bytes, *, capacity_tokens: int | None = None, tail_dtype=torch.float32) -> "KVLayerCache":
        mv = memoryview(bytes(data))
        if len(mv) < 4 or bytes(mv[:4]) != b"KVCD":
            raise KvmixRuntimeError("KVLayerCache::load: bad magic")
        off = 4

        def take(fmt):
            nonlocal off
            n = struct.calcsize(fmt)
            if off + n > len(mv):
                raise KvmixRuntimeError("KVLayerCache::load: truncated stream")
            v = struct.unpack_from(fmt, mv, off)
            off += n
            return v if len(v) > 1 else v[0]

        version = take("<B")
        if version != 1:
            raise KvmixRuntimeError(f"KVLayerCache::load: unsupported version {version}")
        li, kb, vb, rk, rv, gs, B, H, D, kt, vt, qk, qv = take("<iBBffIIIIqqqq")
        cfg = LayerQuantConfig(li, kb, vb, rk, rv, gs)
        segs = []
        for _ in range(2):
            n = take("<I")
            side = []
            for _ in range(n):
                ln = take("<Q")
                if off + ln > len(mv):
                    raise KvmixRuntimeError("KVLayerCache::load: truncated segment")
                side.append(deserialize_quantized_groups(bytes(mv[off:off + ln])))
                off += ln
            segs.append(side)
        tails = []
        for _ in range(2):
            n = take("<Q")
            if off + 4 * n > len(mv):
                raise KvmixRuntimeError("KVLayerCache::load: truncated tail")
            tails.append(np.frombuffer(mv, dtype="<f4", count=n, offset=off).copy())
            off += 4 * n
        total = qk + kt
        cap = capacity_tokens or max(total, 1)
        cache = KVLayerCache(cfg, B, H, D, capacity_tokens=cap, tail_dtype=tail_dtype)
        for side, lst in enumerate(segs):
            for qg in lst:
                check(lib().kvmix_cache_import_segment(cache._h, side, qg.shape.t, _ptr(qg.codes.words),
                                                       _ptr(qg.meta), _stream()))
        for side, (arr, t) in enumerate(zip(tails, (kt, vt))):
            dev = torch.from_numpy(arr).to(cache._device)
            check(lib().kvmix_cache_import_tail(cache._h, side, _ptr(dev), int(t), _stream()))
        torch.cuda.current_stream().synchronize()
        return cache
