"""CPU oracle for the KVmix hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package. The product package
(``paper_2506_08018_b200``) never imports it and has no CPU fallback.

Two checkers live here:

* ``liboracle.so`` -- ``kvmix_oracle.c``, a plain-C restatement of the reference
  hot path (each function cites the reference file:line it follows), plus
  ``CacheOracle`` below, a numpy restatement of ``KVLayerCache``
  (``src/cache.cpp:45-173``, ``:229-249``) built on those C primitives.
* ``_ref/libkvmix_ref.so`` -- the UNMODIFIED reference sources compiled by
  ``oracle/Makefile`` with the reference's own flags (present whenever the
  build ran in a container that has ``/root/reference``; it travels to the GPU
  box as a built artefact). ``RefCache`` wraps it.

Parity of the restatement is pinned by ``tests/test_oracle.py`` against the
reference's known-answer tests and against golden fixtures generated from
``_ref`` (``tests/golden/make_golden.py``).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import struct
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def build(ref: bool = True) -> None:
    """Compile liboracle.so (and _ref when /root/reference exists)."""
    targets = ["all"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        L.ko_half_from_float.restype = C.c_uint16
        L.ko_half_from_float.argtypes = [C.c_float]
        L.ko_float_from_half.restype = C.c_float
        L.ko_float_from_half.argtypes = [C.c_uint16]
        L.ko_round_through_half.restype = C.c_float
        L.ko_round_through_half.argtypes = [C.c_float]
        L.ko_encode.restype = C.c_uint32
        L.ko_encode.argtypes = [C.c_float, C.c_float, C.c_float, C.c_int, C.c_uint64]
        L.ko_decode.restype = C.c_float
        L.ko_decode.argtypes = [C.c_uint32, C.c_float, C.c_float, C.c_int, C.c_uint64]
        L.ko_compute_meta.argtypes = [_f32p, C.c_size_t, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_float)]
        L.ko_quantize_group.argtypes = [_f32p, C.c_size_t, C.c_float, C.c_float, C.c_int, _u32p]
        L.ko_dequantize_group.argtypes = [_u32p, C.c_size_t, C.c_float, C.c_float, _f32p]
        L.ko_words_for.restype = C.c_size_t
        L.ko_words_for.argtypes = [C.c_size_t, C.c_int]
        L.ko_pack.argtypes = [_u32p, C.c_size_t, C.c_int, _u32p, C.POINTER(C.c_size_t)]
        L.ko_get.restype = C.c_uint32
        L.ko_get.argtypes = [_u32p, C.c_size_t, C.c_int]
        for fn in (L.ko_quantize_key, L.ko_quantize_value):
            fn.argtypes = [_f32p] + [C.c_int] * 6 + [_u32p, _u16p]
        L.ko_dequantize.argtypes = [_u32p, _u16p] + [C.c_int] * 7 + [_f32p]
        L.ko_rpc_target.restype = C.c_int64
        L.ko_rpc_target.argtypes = [C.c_int64, C.c_double]
        L.ko_shrink.restype = C.c_int64
        L.ko_shrink.argtypes = [C.POINTER(C.c_int64), C.c_int64, C.c_float, C.c_int, C.c_int]
        L.ko_attend_f32.argtypes = [_f32p, _f32p, _f32p] + [C.c_int] * 5 + [_f32p, C.POINTER(C.c_double)]
        L.ko_attend_f64.argtypes = [_f32p, _f32p, _f32p] + [C.c_int] * 5 + [_f64p, C.POINTER(C.c_double)]
        L.ko_random_h16.argtypes = [C.c_uint64, C.c_size_t, C.c_float, C.c_float, _f32p]
        _LIB = L
    return _LIB


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libkvmix_ref.so"))


def ref():
    """The compiled reference library, or None when it was never built here."""
    global _REF
    if _REF is None and ref_available():
        R = C.CDLL(os.path.join(HERE, "_ref", "libkvmix_ref.so"))
        R.ref_last_error.restype = C.c_char_p
        R.ref_half_from_float.restype = C.c_uint16
        R.ref_half_from_float.argtypes = [C.c_float]
        R.ref_float_from_half.restype = C.c_float
        R.ref_float_from_half.argtypes = [C.c_uint16]
        R.ref_rpc_target.restype = C.c_int64
        R.ref_rpc_target.argtypes = [C.c_int64, C.c_double]
        R.ref_random_h16.argtypes = [C.c_uint64, C.c_size_t, C.c_float, C.c_float, _f32p]
        R.ref_pack.argtypes = [_u32p, C.c_size_t, C.c_int, _u32p, C.POINTER(C.c_size_t)]
        R.ref_quantize.argtypes = [C.c_int, _f32p] + [C.c_int] * 6 + [
            C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        R.ref_quantize_serialized.argtypes = [C.c_int, _f32p] + [C.c_int] * 6 + [
            C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        R.ref_cache_create.restype = C.c_void_p
        R.ref_cache_create.argtypes = [C.c_int, C.c_int, C.c_float, C.c_float, C.c_int, C.c_int, C.c_int, C.c_int]
        R.ref_cache_destroy.argtypes = [C.c_void_p]
        R.ref_cache_append.argtypes = [C.c_void_p, _f32p, _f32p, C.c_int]
        R.ref_cache_counters.argtypes = [C.c_void_p, np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")]
        R.ref_cache_memory.argtypes = [C.c_void_p, np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS"),
                                       C.POINTER(C.c_double)]
        R.ref_cache_snapshot.argtypes = [C.c_void_p, _f32p, _f32p]
        R.ref_cache_segment.argtypes = [C.c_void_p, C.c_int, C.c_int,
                                        np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS"),
                                        C.c_void_p, C.c_void_p]
        R.ref_cache_dump.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        R.ref_attend.argtypes = [C.c_void_p, _f32p, C.c_int, C.c_int, _f32p, C.POINTER(C.c_double)]
        R.ref_set_threads.argtypes = [C.c_int]
        R.ref_max_threads.restype = C.c_int
        _REF = R
    return _REF


class OracleError(Exception):
    pass


# --------------------------------------------------------------------------------------------
# scalar / array helpers over the C restatement
# --------------------------------------------------------------------------------------------
def half_from_float(x: float) -> int:
    return lib().ko_half_from_float(x)


def float_from_half(h: int) -> float:
    return lib().ko_float_from_half(h)


def round_through_half(x: float) -> float:
    return lib().ko_round_through_half(x)


def q_max_for_bits(bits: int) -> int:
    return {1: 1, 2: 3, 3: 7, 4: 15}[bits]


def words_for(n: int, bits: int) -> int:
    return (n + 10) // 11 if bits == 3 else (n * bits + 31) // 32


def pack(codes, bits: int) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint32)
    words = np.zeros(max(1, words_for(len(codes), bits)), np.uint32)
    bad = C.c_size_t(0)
    rc = lib().ko_pack(codes, len(codes), bits, words, C.byref(bad))
    if rc != 0:
        raise OracleError(f"pack: code out of range at index {bad.value}")
    return words[: words_for(len(codes), bits)]


def get(words, idx: int, bits: int) -> int:
    return lib().ko_get(np.ascontiguousarray(words, np.uint32), idx, bits)


def rpc_target(n: int, r: float) -> int:
    return lib().ko_rpc_target(n, r)


def random_h16(seed: int, shape, sigma: float = 1.0, mu: float = 0.0) -> np.ndarray:
    """N(mu, sigma^2) on the binary16 grid from kvmix::Rng(seed) (helpers.hpp:14-25)."""
    n = int(np.prod(shape))
    out = np.empty(n, np.float32)
    lib().ko_random_h16(seed, n, sigma, mu, out)
    return out.reshape(shape)


def quantize(x: np.ndarray, bits: int, gs: int, key: bool):
    """quantize_key_tensor / quantize_value_tensor: returns (words u32, meta u16 [groups,2])."""
    x = np.ascontiguousarray(x, np.float32)
    B, H, T, D = x.shape
    n = B * H * T * D
    if key:
        if gs <= 0 or T % gs:
            raise OracleError("key quantization needs T to be a multiple of group_size")
        groups = B * H * D * (T // gs)
    else:
        groups = B * H * T * ((D + gs - 1) // gs)
    words = np.zeros(max(1, words_for(n, bits)), np.uint32)
    meta = np.zeros(max(1, 2 * groups), np.uint16)
    fn = lib().ko_quantize_key if key else lib().ko_quantize_value
    rc = fn(x, B, H, T, D, bits, gs, words, meta)
    if rc != 0:
        raise OracleError("quantize: invalid argument")
    return words[: words_for(n, bits)], meta[: 2 * groups].reshape(groups, 2)


def dequantize(words, meta, key: bool, shape, bits: int, gs: int) -> np.ndarray:
    B, H, T, D = shape
    out = np.zeros((B, H, T, D), np.float32)
    w = np.ascontiguousarray(words, np.uint32)
    if w.size == 0:
        w = np.zeros(1, np.uint32)
    m = np.ascontiguousarray(meta, np.uint16).reshape(-1)
    if m.size == 0:
        m = np.zeros(2, np.uint16)
    lib().ko_dequantize(w, m, 0 if key else 1, B, H, T, D, bits, gs, out)
    return out


def attend_f32(q, keys, values):
    """reference_attend over dense tensors (attention.cpp:168-211). q [B,H,t,D], k/v [B,H,T,D]."""
    q = np.ascontiguousarray(q, np.float32)
    keys = np.ascontiguousarray(keys, np.float32)
    values = np.ascontiguousarray(values, np.float32)
    B, H, t, D = q.shape
    T = keys.shape[2]
    out = np.zeros((B, H, t, D), np.float32)
    cs = C.c_double(0)
    if lib().ko_attend_f32(q, keys, values, B, H, t, T, D, out, C.byref(cs)) != 0:
        raise OracleError("softmax over an empty row")
    return out, cs.value


def attend_f64(q, keys, values):
    q = np.ascontiguousarray(q, np.float32)
    keys = np.ascontiguousarray(keys, np.float32)
    values = np.ascontiguousarray(values, np.float32)
    B, H, t, D = q.shape
    T = keys.shape[2]
    out = np.zeros((B, H, t, D), np.float64)
    cs = C.c_double(0)
    if lib().ko_attend_f64(q, keys, values, B, H, t, T, D, out, C.byref(cs)) != 0:
        raise OracleError("softmax over an empty row")
    return out, cs.value


def serialize_qg(words, meta, bits, key, gs, shape) -> bytes:
    """KVQG bytes (quant.hpp:82-89, quant.cpp:148-170)."""
    B, H, T, D = shape
    meta = np.asarray(meta, np.uint16).reshape(-1, 2)
    out = bytearray(b"KVQG")
    out += struct.pack("<BBBB", 1, bits, 0 if key else 1, 1 if bits == 3 else 0)
    out += struct.pack("<IIIII", gs, B, H, T, D)
    out += struct.pack("<QQQ", meta.shape[0], B * H * T * D, len(words))
    out += np.ascontiguousarray(meta, "<u2").tobytes()
    out += np.ascontiguousarray(words, "<u4").tobytes()
    return bytes(out)


# --------------------------------------------------------------------------------------------
# KVLayerCache restatement (src/cache.cpp:45-173, 229-249), numpy + the C quantizers
# --------------------------------------------------------------------------------------------
class CacheOracle:
    def __init__(self, key_bits, value_bits, rk, rv, gs, B, H, D, layer_index=0):
        if not (2 <= key_bits <= 4 and 2 <= value_bits <= 4):
            raise OracleError("cache bit widths must be 2, 3 or 4")  # cache.cpp:15-18
        rk32, rv32 = float(np.float32(rk)), float(np.float32(rv))
        if not (0.0 <= rk32 <= 1.0 and 0.0 <= rv32 <= 1.0):
            raise OracleError("rpc ratios must lie in [0, 1]")
        if gs <= 0:
            raise OracleError("group_size must be positive")
        self.kb, self.vb, self.rk, self.rv, self.gs = key_bits, value_bits, rk32, rv32, gs
        self.B, self.H, self.D = B, H, D
        self.layer_index = layer_index
        self.key_segs, self.value_segs = [], []  # (t, words, meta)
        self.key_tail = np.zeros((0, B, H, D), np.float32)
        self.value_tail = np.zeros((0, B, H, D), np.float32)
        self.qk = 0
        self.qv = 0

    @property
    def total(self):
        return self.qk + self.key_tail.shape[0]

    def append(self, k, v):
        """k, v: [B,H,t,D] fp32 (cache.cpp:45-80)."""
        k = np.asarray(k, np.float32)
        v = np.asarray(v, np.float32)
        if k.shape[:2] != (self.B, self.H) or k.shape[3] != self.D or k.shape != v.shape:
            raise OracleError("KVLayerCache::append: tensor shape does not match cache")
        t = k.shape[2]
        if t < 1:
            raise OracleError("KVLayerCache::append: need at least one token")
        self.key_tail = np.concatenate([self.key_tail, k.transpose(2, 0, 1, 3)], 0)
        self.value_tail = np.concatenate([self.value_tail, v.transpose(2, 0, 1, 3)], 0)
        kt = self.key_tail.shape[0]
        excess = kt - rpc_target(kt, self.rk)
        n = excess // self.gs * self.gs
        if n > 0:
            seg = np.ascontiguousarray(self.key_tail[:n].transpose(1, 2, 0, 3))
            w, m = quantize(seg, self.kb, self.gs, key=True)
            self.key_segs.append((n, w, m))
            self.key_tail = self.key_tail[n:]
            self.qk += n
        vt = self.value_tail.shape[0]
        excess = vt - rpc_target(vt, self.rv)
        if excess > 0:
            seg = np.ascontiguousarray(self.value_tail[:excess].transpose(1, 2, 0, 3))
            w, m = quantize(seg, self.vb, self.gs, key=False)
            self.value_segs.append((excess, w, m))
            self.value_tail = self.value_tail[excess:]
            self.qv += excess

    def counters(self):
        return dict(total=self.total, key_tail=self.key_tail.shape[0], value_tail=self.value_tail.shape[0],
                    quant_keys=self.qk, quant_values=self.qv,
                    key_segments=len(self.key_segs), value_segments=len(self.value_segs))

    def memory_usage(self):
        """cache.cpp:119-134."""
        payload = sum(len(s[1]) * 32 for s in self.key_segs + self.value_segs)
        meta = sum(s[2].shape[0] * 32 for s in self.key_segs + self.value_segs)
        slab = self.B * self.H * self.D
        tail = (self.key_tail.shape[0] + self.value_tail.shape[0]) * slab * 16
        total = payload + meta + tail
        base = self.total * slab * 16 * 2
        return dict(packed_payload_bits=payload, metadata_bits=meta, tail_bits=tail, total_bits=total,
                    fp16_baseline_bits=base, compression_ratio=1.0 if total == 0 else base / total)

    def snapshot(self):
        """snapshot_dequantized (cache.cpp:136-173): fp32 [B,H,T,D] keys and values."""
        ks = [dequantize(w, m, True, (self.B, self.H, n, self.D), self.kb, self.gs) for n, w, m in self.key_segs]
        ks.append(self.key_tail.transpose(1, 2, 0, 3))
        vs = [dequantize(w, m, False, (self.B, self.H, n, self.D), self.vb, self.gs) for n, w, m in self.value_segs]
        vs.append(self.value_tail.transpose(1, 2, 0, 3))
        return np.ascontiguousarray(np.concatenate(ks, 2)), np.ascontiguousarray(np.concatenate(vs, 2))

    def dump(self) -> bytes:
        """KVCD bytes (cache.cpp:190-249)."""
        out = bytearray(b"KVCD")
        out += struct.pack("<BiBBffIIIIqqqq", 1, self.layer_index, self.kb, self.vb, self.rk, self.rv, self.gs,
                           self.B, self.H, self.D, self.key_tail.shape[0], self.value_tail.shape[0],
                           self.qk, self.qv)
        for segs, bits, key in ((self.key_segs, self.kb, True), (self.value_segs, self.vb, False)):
            out += struct.pack("<I", len(segs))
            for n, w, m in segs:
                b = serialize_qg(w, m, bits, key, self.gs, (self.B, self.H, n, self.D))
                out += struct.pack("<Q", len(b)) + b
        for tail in (self.key_tail, self.value_tail):
            out += struct.pack("<Q", tail.size) + np.ascontiguousarray(tail, "<f4").tobytes()
        return bytes(out)


class RefCache:
    """The reference KVLayerCache itself (oracle/_ref), same surface as CacheOracle."""

    def __init__(self, key_bits, value_bits, rk, rv, gs, B, H, D):
        R = ref()
        if R is None:
            raise OracleError("oracle/_ref was not built")
        self.R = R
        self.h = R.ref_cache_create(key_bits, value_bits, rk, rv, gs, B, H, D)
        if not self.h:
            raise OracleError(R.ref_last_error().decode())
        self.kb, self.vb, self.gs, self.B, self.H, self.D = key_bits, value_bits, gs, B, H, D

    def __del__(self):
        if getattr(self, "h", None):
            self.R.ref_cache_destroy(self.h)
            self.h = None

    def append(self, k, v):
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        if self.R.ref_cache_append(self.h, k, v, k.shape[2]) != 0:
            raise OracleError(self.R.ref_last_error().decode())

    def counters(self):
        o = np.zeros(7, np.int64)
        self.R.ref_cache_counters(self.h, o)
        keys = ("total", "key_tail", "value_tail", "quant_keys", "quant_values", "key_segments", "value_segments")
        return {k: int(x) for k, x in zip(keys, o)}

    def memory_usage(self):
        o = np.zeros(5, np.uint64)
        r = C.c_double(0)
        self.R.ref_cache_memory(self.h, o, C.byref(r))
        keys = ("packed_payload_bits", "metadata_bits", "tail_bits", "total_bits", "fp16_baseline_bits")
        d = {k: int(x) for k, x in zip(keys, o)}
        d["compression_ratio"] = r.value
        return d

    def snapshot(self):
        T = self.counters()["total"]
        k = np.zeros((self.B, self.H, T, self.D), np.float32)
        v = np.zeros_like(k)
        self.R.ref_cache_snapshot(self.h, k, v)
        return k, v

    def segment(self, side: int, idx: int):
        info = np.zeros(3, np.int64)
        self.R.ref_cache_segment(self.h, side, idx, info, None, None)
        w = np.zeros(max(1, info[1]), np.uint32)
        m = np.zeros(max(1, 2 * info[2]), np.uint16)
        self.R.ref_cache_segment(self.h, side, idx, info, w.ctypes.data, m.ctypes.data)
        return int(info[0]), w[: info[1]], m[: 2 * info[2]].reshape(-1, 2)

    def dump(self) -> bytes:
        n = C.c_uint64(0)
        self.R.ref_cache_dump(self.h, None, 0, C.byref(n))
        buf = np.zeros(n.value, np.uint8)
        self.R.ref_cache_dump(self.h, buf.ctypes.data, n.value, C.byref(n))
        return buf.tobytes()

    def attend(self, q, reference: bool = False):
        q = np.ascontiguousarray(q, np.float32)
        out = np.zeros_like(q)
        cs = C.c_double(0)
        if self.R.ref_attend(self.h, q, q.shape[2], 1 if reference else 0, out, C.byref(cs)) != 0:
            raise OracleError(self.R.ref_last_error().decode())
        return out, cs.value


def ref_quantize(x, bits, gs, key):
    R = ref()
    x = np.ascontiguousarray(x, np.float32)
    B, H, T, D = x.shape
    nw, ng = C.c_uint64(0), C.c_uint64(0)
    rc = R.ref_quantize(0 if key else 1, x, B, H, T, D, bits, gs, None, None, C.byref(nw), C.byref(ng))
    if rc != 0:
        raise OracleError(R.ref_last_error().decode())
    w = np.zeros(max(1, nw.value), np.uint32)
    m = np.zeros(max(1, 2 * ng.value), np.uint16)
    R.ref_quantize(0 if key else 1, x, B, H, T, D, bits, gs, w.ctypes.data, m.ctypes.data, C.byref(nw), C.byref(ng))
    return w[: nw.value], m[: 2 * ng.value].reshape(-1, 2)


def ref_random_h16(seed, shape, sigma=1.0, mu=0.0):
    n = int(np.prod(shape))
    out = np.empty(n, np.float32)
    ref().ref_random_h16(seed, n, sigma, mu, out)
    return out.reshape(shape)


__all__ = [n for n in dir() if not n.startswith("_")] + ["math"]
