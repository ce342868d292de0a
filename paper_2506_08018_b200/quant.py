"""bitpack + quant: host mirror of include/kvmix/{bitpack,quant}.hpp over the C ABI.

Names, argument meaning and exceptions follow the reference:
  pack_uniform / pack_mixed3 / unpack_*      bitpack.hpp:48-56, bitpack.cpp:57-96
  feat_per_word, mixed3_q_max, q_max_for_bits bitpack.cpp:8-14, bitpack.hpp:31-33, quant.cpp:8-21
  quantize_key_tensor / quantize_value_tensor quant.hpp:79-80, quant.cpp:102-124
  QuantizedGroups (+ value_at, stream_index, meta_index)  quant.hpp:64-77, quant.cpp:77-100
  serialize/deserialize_quantized_groups (KVQG)           quant.hpp:82-89, quant.cpp:148-207
All compute runs in libkvmix_b200.so on the current CUDA device; tensors are torch tensors.
"""
from __future__ import annotations

import dataclasses
import enum
import struct

import numpy as np
import torch

from . import _lib
from ._lib import KvmixInvalidArgument, KvmixOutOfRange, KvmixRuntimeError, check, lib


class Grouping(enum.IntEnum):
    kPerChannelKey = 0
    kPerTokenValue = 1


class PackLayout(enum.IntEnum):
    kUniform = 0
    kMixed3 = 1


kMixed3Block = 11


@dataclasses.dataclass
class QuantSpec:
    bits: int = 4
    grouping: Grouping = Grouping.kPerChannelKey
    group_size: int = 32


@dataclasses.dataclass
class TensorShape:
    b: int = 0
    nh: int = 0
    t: int = 0
    d: int = 0

    def elems(self) -> int:
        return self.b * self.nh * self.t * self.d


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _as_device(x, dtype=None) -> torch.Tensor:
    """Host data (numpy / CPU tensor) is copied to the current CUDA device."""
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if not x.is_cuda:
        x = x.to("cuda", non_blocking=False)
    if dtype is not None and x.dtype != dtype:
        x = x.to(dtype)
    return x.contiguous()


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return _lib.F32
    if t.dtype == torch.float16:
        return _lib.F16
    raise KvmixInvalidArgument(f"unsupported dtype {t.dtype} (float32 or float16)")


def q_max_for_bits(bits: int) -> int:
    if bits not in (1, 2, 3, 4):
        raise KvmixInvalidArgument(f"unsupported bit width {bits}")
    return (1 << bits) - 1


def feat_per_word(bits: int) -> int:
    out = __import__("ctypes").c_int(0)
    check(lib().kvmix_feat_per_word(bits, out))
    return out.value


def mixed3_q_max(stream_idx: int) -> int:
    return 3 if stream_idx % kMixed3Block == kMixed3Block - 1 else 7


def mixed3_wide_scale(scale: float) -> float:
    return float(np.float32(scale) * np.float32(7.0 / 3.0))


def packed_word_count(n_codes: int, bits: int) -> int:
    return int(lib().kvmix_packed_word_count(n_codes, bits))


@dataclasses.dataclass
class PackedBuffer:
    """Device-resident PackedBuffer (bitpack.hpp:35-44): words are uint32 bit patterns
    stored in an int32 tensor."""
    words: torch.Tensor
    layout: PackLayout
    bits: int
    logical_len: int

    def word_count(self) -> int:
        return int(self.words.numel())

    def words_u32(self) -> np.ndarray:
        return self.words.cpu().numpy().view(np.uint32)

    def get(self, idx: int) -> int:
        """Bounds-checked read (bitpack.cpp:69-82)."""
        if idx < 0 or idx >= self.logical_len:
            raise KvmixOutOfRange(f"PackedBuffer::get: index {idx} out of bounds (logical_len {self.logical_len})")
        # one word read (bitpack.cpp:69-82 field arithmetic), not an unpack of the buffer
        if self.bits == 3:
            w, pos = divmod(idx, kMixed3Block)
            shift, mask = (30, 3) if pos == kMixed3Block - 1 else (3 * pos, 7)
        else:
            w, pos = divmod(idx, 32 // self.bits)
            shift, mask = pos * self.bits, (1 << self.bits) - 1
        word = int(self.words[w].item()) & 0xFFFFFFFF
        return (word >> shift) & mask


def _pack(codes, bits: int, layout: PackLayout) -> PackedBuffer:
    c = _as_device(torch.as_tensor(np.asarray(codes, dtype=np.uint32).view(np.int32)) if not isinstance(codes, torch.Tensor) else codes)
    c = c.to(torch.int32).contiguous()
    n = int(c.numel())
    words = torch.zeros(max(1, packed_word_count(n, bits)), dtype=torch.int32, device=c.device)
    check(lib().kvmix_pack(_ptr(c), n, bits, _ptr(words), _stream()))
    return PackedBuffer(words[: packed_word_count(n, bits)], layout, bits, n)


def pack_uniform(codes, bits: int) -> PackedBuffer:
    """pack_uniform (bitpack.cpp:57-61); bits in {1,2,4}."""
    feat_per_word(bits)  # validates like PackedWriter::uniform
    return _pack(codes, bits, PackLayout.kUniform)


def pack_mixed3(codes) -> PackedBuffer:
    """pack_mixed3 (bitpack.cpp:63-67): 11 codes per word, slot 10 is 2 bits wide."""
    return _pack(codes, 3, PackLayout.kMixed3)


def unpack(buf: PackedBuffer) -> np.ndarray:
    n = buf.logical_len
    out = torch.zeros(max(1, n), dtype=torch.int32, device=buf.words.device)
    words = buf.words if buf.words.numel() else torch.zeros(1, dtype=torch.int32, device=buf.words.device)
    check(lib().kvmix_unpack(_ptr(words), n, buf.bits, _ptr(out), _stream()))
    return out[:n].cpu().numpy().view(np.uint32)


def unpack_uniform(buf: PackedBuffer, idx: int) -> int:
    if buf.layout != PackLayout.kUniform:
        raise KvmixInvalidArgument("unpack_uniform: buffer does not use a uniform layout")
    return buf.get(idx)


def unpack_mixed3(buf: PackedBuffer, idx: int) -> int:
    if buf.layout != PackLayout.kMixed3:
        raise KvmixInvalidArgument("unpack_mixed3: buffer does not use the mixed 3-bit layout")
    return buf.get(idx)


@dataclasses.dataclass
class GroupMeta:
    scale: float = 0.0
    min_val: float = 0.0


@dataclasses.dataclass
class QuantizedGroups:
    """QuantizedGroups (quant.hpp:64-77). `meta` is an int16 [groups, 2] tensor of binary16
    bit patterns {scale, min} (the KVQG payload order); `codes` the packed words."""
    meta: torch.Tensor
    codes: PackedBuffer
    spec: QuantSpec
    shape: TensorShape

    def group_count(self) -> int:
        return int(self.meta.shape[0])

    def meta_list(self) -> list[GroupMeta]:
        h = self.meta.cpu().numpy().view(np.float16).astype(np.float32)
        return [GroupMeta(float(s), float(m)) for s, m in h]

    def stream_index(self, bi: int, hi: int, ti: int, di: int) -> int:
        s = self.shape
        if self.spec.grouping == Grouping.kPerChannelKey:
            return ((bi * s.nh + hi) * s.d + di) * s.t + ti
        return ((bi * s.nh + hi) * s.t + ti) * s.d + di

    def meta_index(self, bi: int, hi: int, ti: int, di: int) -> int:
        s, gs = self.shape, self.spec.group_size
        if self.spec.grouping == Grouping.kPerChannelKey:
            return ((bi * s.nh + hi) * s.d + di) * (s.t // gs) + ti // gs
        return ((bi * s.nh + hi) * s.t + ti) * ((s.d + gs - 1) // gs) + di // gs

    def dequantize(self) -> torch.Tensor:
        """Every value_at at once, bit-exact: fp32 [B,H,T,D] on the device."""
        s = self.shape
        out = torch.empty((s.b, s.nh, s.t, s.d), dtype=torch.float32, device=self.meta.device)
        if s.elems() == 0:
            return out
        check(lib().kvmix_dequantize(int(self.spec.grouping), _ptr(self.codes.words), _ptr(self.meta), s.b, s.nh, s.t,
                                     s.d, self.spec.bits, self.spec.group_size, _ptr(out), _stream()))
        return out

    def value_at(self, bi: int, hi: int, ti: int, di: int) -> float:
        """value_at (quant.cpp:97-100): one code and one meta pair read, decode_code
        (quant.cpp:49-53) in fp32 -- code * scale' then + min, two rounded operations."""
        s = self.shape
        if not (0 <= bi < s.b and 0 <= hi < s.nh and 0 <= ti < s.t and 0 <= di < s.d):
            raise KvmixOutOfRange("QuantizedGroups::value_at: index out of range")
        si = self.stream_index(bi, hi, ti, di)
        code = self.codes.get(si)
        pair = self.meta[self.meta_index(bi, hi, ti, di)].cpu().numpy().view(np.float16).astype(np.float32)
        scale, mn = np.float32(pair[0]), np.float32(pair[1])
        if self.spec.bits == 3 and si % kMixed3Block == kMixed3Block - 1:
            scale = np.float32(scale * np.float32(7.0 / 3.0))
        return float(np.float32(np.float32(code) * scale) + mn)


def _quantize(x, spec: QuantSpec, grouping: Grouping) -> QuantizedGroups:
    if spec.grouping != grouping:
        which = "quantize_key_stream: spec.grouping must be per-channel" if grouping == Grouping.kPerChannelKey \
            else "quantize_value_stream: spec.grouping must be per-token"
        raise KvmixInvalidArgument(which)
    x = _as_device(x)
    if x.dim() != 4:
        raise KvmixInvalidArgument("expected a [B, nh, T, D] tensor")
    B, H, T, D = (int(v) for v in x.shape)
    n = B * H * T * D
    nw = packed_word_count(n, spec.bits)
    ng = int(lib().kvmix_group_count(int(grouping), B, H, T, D, spec.group_size)) if spec.group_size > 0 else 0
    # the kernels write every word and every meta pair: no zero fill
    words = torch.empty(max(1, nw), dtype=torch.int32, device=x.device)
    meta = torch.empty((max(1, ng), 2), dtype=torch.int16, device=x.device)
    check(lib().kvmix_quantize(int(grouping), _ptr(x), _dtype_code(x), B, H, T, D, spec.bits, spec.group_size,
                               _ptr(words), _ptr(meta), _stream()))
    layout = PackLayout.kMixed3 if spec.bits == 3 else PackLayout.kUniform
    return QuantizedGroups(meta[:ng], PackedBuffer(words[:nw], layout, spec.bits, n), spec, TensorShape(B, H, T, D))


def quantize_key_tensor(keys, spec: QuantSpec) -> QuantizedGroups:
    """quantize_key_tensor (quant.cpp:102-114): per-channel groups of gs tokens."""
    return _quantize(keys, spec, Grouping.kPerChannelKey)


def quantize_value_tensor(values, spec: QuantSpec) -> QuantizedGroups:
    """quantize_value_tensor (quant.cpp:116-124): per-token groups of gs channels."""
    return _quantize(values, spec, Grouping.kPerTokenValue)


def serialize_quantized_groups(qg: QuantizedGroups) -> bytes:
    """KVQG bytes (quant.cpp:148-170)."""
    s = qg.shape
    out = bytearray(b"KVQG")
    out += struct.pack("<BBBB", 1, qg.spec.bits, int(qg.spec.grouping), int(qg.codes.layout))
    out += struct.pack("<IIIII", qg.spec.group_size, s.b, s.nh, s.t, s.d)
    out += struct.pack("<QQQ", qg.group_count(), qg.codes.logical_len, qg.codes.word_count())
    out += qg.meta.cpu().numpy().astype("<i2").tobytes()
    out += qg.codes.words.cpu().numpy().astype("<i4").tobytes()
    return bytes(out)


def deserialize_quantized_groups(data: bytes, device="cuda") -> QuantizedGroups:
    """KVQG parse (quant.cpp:172-207), same runtime_error cases."""
    mv = memoryview(bytes(data))
    if len(mv) < 4 or bytes(mv[:4]) != b"KVQG":
        raise KvmixRuntimeError("deserialize_quantized_groups: bad magic")
    off = 4

    def take(fmt):
        nonlocal off
        n = struct.calcsize(fmt)
        if off + n > len(mv):
            raise KvmixRuntimeError("deserialize_quantized_groups: truncated buffer")
        v = struct.unpack_from(fmt, mv, off)
        off += n
        return v if len(v) > 1 else v[0]

    version = take("<B")
    if version != 1:
        raise KvmixRuntimeError(f"deserialize_quantized_groups: unsupported version {version}")
    bits, grouping, layout = take("<BBB")
    gs, B, H, T, D = take("<IIIII")
    ng, logical, nw = take("<QQQ")
    if off + 4 * ng > len(mv):
        raise KvmixRuntimeError("deserialize_quantized_groups: truncated buffer")
    meta = np.frombuffer(mv, dtype="<i2", count=2 * ng, offset=off).reshape(ng, 2).copy()
    off += 4 * ng
    if off + 4 * nw > len(mv):
        raise KvmixRuntimeError("deserialize_quantized_groups: truncated buffer")
    words = np.frombuffer(mv, dtype="<i4", count=nw, offset=off).copy()
    off += 4 * nw
    if off != len(mv):
        raise KvmixRuntimeError("deserialize_quantized_groups: trailing bytes")
    spec = QuantSpec(bits, Grouping(grouping), gs)
    return QuantizedGroups(torch.from_numpy(meta).to(device), PackedBuffer(torch.from_numpy(words).to(device),
                           PackLayout(layout), bits, logical), spec, TensorShape(B, H, T, D))
