"""Attention over the packed cache (attention.hpp:25-48, attention.cpp:28-223).

attend() is the fused split-K decode kernel: dequantization happens inside the q.K dot
products and the P.V accumulation, no full-precision K/V is materialized, and scratch is
independent of the cached token count. Query heads may be a multiple G of the cache's KV
heads (grouped-query attention; G = 1 is the reference's case).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math

import numpy as np
import torch

from ._lib import KvmixInvalidArgument, check, lib
from .cache import KVLayerCache
from .quant import _as_device, _dtype_code, _ptr, _stream


@dataclasses.dataclass
class AttentionOutput:
    output: torch.Tensor  # [B, Hq, t, D] fp32
    scores_checksum: float = 0.0


def attention_inv_scale(head_dim: int) -> float:
    return float(np.float32(1.0) / np.sqrt(np.float32(head_dim)))


def _check_query(q: torch.Tensor, cache: KVLayerCache, allow_gqa: bool) -> None:
    ok = (q.dim() == 4 and q.shape[0] == cache.batch() and q.shape[3] == cache.head_dim()
          and (q.shape[1] == cache.heads() or (allow_gqa and q.shape[1] % cache.heads() == 0 and q.shape[1] > 0)))
    if not ok:
        raise KvmixInvalidArgument("attention: query shape does not match cache")
    if q.shape[2] < 1:
        raise KvmixInvalidArgument("attention: need at least one query row")


def _check_out(out: torch.Tensor, shape, device) -> None:
    """A caller-supplied output must be exactly what the kernel writes: contiguous fp32
    [B, Hq, t, D] on the cache's device (anything else would be written out of bounds)."""
    if (not isinstance(out, torch.Tensor) or out.dtype != torch.float32 or tuple(out.shape) != tuple(shape)
            or not out.is_contiguous() or out.device != device):
        raise KvmixInvalidArgument(f"attention: out must be a contiguous float32 tensor of shape {tuple(shape)} "
                                   f"on {device}")


def attend(query, cache: KVLayerCache, *, checksum: bool = True, out: torch.Tensor | None = None) -> AttentionOutput:
    """attend (attention.cpp:161-166). checksum=True synchronizes to return the double sum
    of all scaled scores like AttentionOutput::scores_checksum."""
    q = _as_device(query)
    _check_query(q, cache, allow_gqa=True)
    B, Hq, t, D = (int(v) for v in q.shape)
    if out is None:
        out = torch.empty((B, Hq, t, D), dtype=torch.float32, device=q.device)
    else:
        _check_out(out, (B, Hq, t, D), q.device)
    cs = C.c_double(0.0)
    check(lib().kvmix_attend(cache.handle, _ptr(q), _dtype_code(q), Hq, t, _ptr(out), C.byref(cs) if checksum else None,
                             _stream()))
    return AttentionOutput(out, cs.value)


def append_attend(cache: KVLayerCache, new_keys, new_values, query, *, checksum: bool = False,
                  out: torch.Tensor | None = None) -> AttentionOutput:
    """One layer of a decode step: cache.append(new_keys, new_values) then attend(query, cache)
    (the CachedDecoder::step pair). A 1-token append that ages no Key group runs inside the
    attention launch; anything else is the two calls in order. Same results and errors."""
    k = _as_device(new_keys)
    v = _as_device(new_values)
    cache._check_append(k, v)
    if v.dtype != k.dtype:
        v = v.to(k.dtype)
    q = _as_device(query)
    _check_query(q, cache, allow_gqa=True)
    B, Hq, t, D = (int(x) for x in q.shape)
    if out is None:
        out = torch.empty((B, Hq, t, D), dtype=torch.float32, device=q.device)
    else:
        _check_out(out, (B, Hq, t, D), q.device)
    cs = C.c_double(0.0)
    check(lib().kvmix_append_attend(cache.handle, _ptr(k), _ptr(v), _dtype_code(k), int(k.shape[2]), _ptr(q),
                                    _dtype_code(q), Hq, t, _ptr(out), C.byref(cs) if checksum else None, _stream()))
    return AttentionOutput(out, cs.value)


def fused_qk_scores(query, cache: KVLayerCache) -> torch.Tensor:
    """fused_qk_scores (attention.cpp:28-81): [B,H,t,total] fp32, already * 1/sqrt(D)."""
    q = _as_device(query)
    _check_query(q, cache, allow_gqa=False)
    B, H, t, D = (int(v) for v in q.shape)
    T = cache.total_tokens()
    scores = torch.empty((B, H, t, T), dtype=torch.float32, device=q.device)
    check(lib().kvmix_fused_qk_scores(cache.handle, _ptr(q), _dtype_code(q), t, _ptr(scores), _stream()))
    return scores


def softmax_rows(scores) -> torch.Tensor:
    """softmax_rows (attention.cpp:96-105): returns a new tensor, rows sum to 1."""
    s = _as_device(scores, torch.float32).clone()
    cols = int(s.shape[-1]) if s.dim() else 0
    if cols == 0:
        raise KvmixInvalidArgument("softmax over an empty row")
    check(lib().kvmix_softmax_rows(_ptr(s), s.numel() // cols, cols, _stream()))
    return s


def fused_pv(probs, cache: KVLayerCache) -> torch.Tensor:
    """fused_pv (attention.cpp:107-159): probs [B,H,t,total] -> [B,H,t,D]."""
    p = _as_device(probs, torch.float32)
    if p.dim() != 4 or p.shape[3] != cache.total_tokens():
        raise KvmixInvalidArgument("fused_pv: probability columns do not match cached tokens")
    if p.shape[0] != cache.batch() or p.shape[1] != cache.heads():
        raise KvmixInvalidArgument("fused_pv: probability shape does not match cache")
    B, H, t, _ = (int(v) for v in p.shape)
    out = torch.empty((B, H, t, cache.head_dim()), dtype=torch.float32, device=p.device)
    check(lib().kvmix_fused_pv(cache.handle, _ptr(p), t, _ptr(out), _stream()))
    return out


def reference_attend(query, cache: KVLayerCache) -> AttentionOutput:
    """reference_attend (attention.cpp:168-211): snapshot_dequantized into scratch, then dense
    attention -- deliberately pays the O(total * D) materialization."""
    q = _as_device(query)
    _check_query(q, cache, allow_gqa=False)
    B, H, t, D = (int(v) for v in q.shape)
    T = cache.total_tokens()
    scratch = torch.empty(2 * B * H * max(T, 1) * D, dtype=torch.float32, device=q.device)
    out = torch.empty((B, H, t, D), dtype=torch.float32, device=q.device)
    cs = C.c_double(0.0)
    check(lib().kvmix_reference_attend(cache.handle, _ptr(q), _dtype_code(q), t, _ptr(scratch), _ptr(out),
                                       C.byref(cs), _stream()))
    return AttentionOutput(out, cs.value)


def dump_scores_csv(os_, scores) -> None:
    """dump_scores_csv (attention.cpp:213-221)."""
    s = scores.cpu().numpy() if isinstance(scores, torch.Tensor) else np.asarray(scores)
    os_.write("b,h,query,token,score\n")
    B, H, t, T = s.shape
    for b in range(B):
        for h in range(H):
            for qi in range(t):
                for j in range(T):
                    os_.write(f"{b},{h},{qi},{j},{float(s[b, h, qi, j]):g}\n")


def attend_layers(caches, queries, outs, *, stream: int | None = None) -> None:
    """One decode step's attention over a stack of layer caches in a single C call."""
    n = len(caches)
    if len(queries) != n or len(outs) != n:
        raise KvmixInvalidArgument("attend_layers: one query and one output per cache")
    for c, q, o in zip(caches, queries, outs):
        _check_query(q, c, allow_gqa=True)
        if not q.is_cuda or not q.is_contiguous() or q.dtype not in (torch.float16, torch.float32) or q.dtype != queries[0].dtype \
                or tuple(q.shape[1:]) != tuple(queries[0].shape[1:]):
            raise KvmixInvalidArgument("attend_layers: queries must be contiguous device tensors of one dtype and shape")
        _check_out(o, tuple(q.shape), q.device)
    hs = (C.c_void_p * n)(*[c.handle.value for c in caches])
    qs = (C.c_void_p * n)(*[q.data_ptr() for q in queries])
    os_ = (C.c_void_p * n)(*[o.data_ptr() for o in outs])
    q0 = queries[0]
    check(lib().kvmix_attend_layers(hs, n, qs, _dtype_code(q0), int(q0.shape[1]), int(q0.shape[2]), os_,
                                    stream if stream is not None else _stream()))


def _ptr_array(ts):
    return (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


def _check_layers(caches, keys, values, queries, outs):
    n = len(caches)
    if not (len(keys) == len(values) == len(queries) == len(outs) == n):
        raise KvmixInvalidArgument("append_attend_layers: one key, value, query and output per cache")
    for c, k, v, q, o in zip(caches, keys, values, queries, outs):
        for x in (k, v, q):
            if not isinstance(x, torch.Tensor) or not x.is_cuda or not x.is_contiguous() or \
                    x.dtype not in (torch.float16, torch.float32):
                raise KvmixInvalidArgument("append_attend_layers: inputs must be contiguous fp16/fp32 device tensors")
        c._check_append(k, v)
        if v.dtype != k.dtype or k.dtype != keys[0].dtype or tuple(k.shape) != tuple(keys[0].shape):
            raise KvmixInvalidArgument("append_attend_layers: keys/values of one dtype and shape")
        _check_query(q, c, allow_gqa=True)
        if q.dtype != queries[0].dtype or tuple(q.shape) != tuple(queries[0].shape):
            raise KvmixInvalidArgument("append_attend_layers: queries of one dtype and shape")
        _check_out(o, tuple(q.shape), q.device)


def append_attend_layers(caches, keys, values, queries, outs, *, stream: int | None = None) -> None:
    """One decode step of a model stack: append_attend(caches[l], keys[l], values[l],
    queries[l], out=outs[l]) for every layer, in one C call (kvmix_append_attend_layers)."""
    _check_layers(caches, keys, values, queries, outs)
    n = len(caches)
    q0, k0 = queries[0], keys[0]
    check(lib().kvmix_append_attend_layers((C.c_void_p * n)(*[c.handle.value for c in caches]), n, _ptr_array(keys),
                                           _ptr_array(values), _dtype_code(k0), int(k0.shape[2]), _ptr_array(queries),
                                           _dtype_code(q0), int(q0.shape[1]), int(q0.shape[2]), _ptr_array(outs),
                                           stream if stream is not None else _stream()))


class DecodeStep:
    """A serving loop's decode step over a fixed stack of layer caches and fixed device
    buffers (the caller refills them each step): shapes are validated and the pointer arrays
    built once, so step() is a single C call (kvmix_append_attend_layers)."""

    def __init__(self, caches, keys, values, queries, outs):
        _check_layers(caches, keys, values, queries, outs)
        n = len(caches)
        self._n = n
        self._keep = (list(caches), list(keys), list(values), list(queries), list(outs))
        self._h = (C.c_void_p * n)(*[c.handle.value for c in caches])
        self._k, self._v = _ptr_array(keys), _ptr_array(values)
        self._q, self._o = _ptr_array(queries), _ptr_array(outs)
        self._kdt, self._t = _dtype_code(keys[0]), int(keys[0].shape[2])
        self._qdt, self._hq, self._tq = _dtype_code(queries[0]), int(queries[0].shape[1]), int(queries[0].shape[2])

    def step(self, stream: int | None = None) -> None:
        check(lib().kvmix_append_attend_layers(self._h, self._n, self._k, self._v, self._kdt, self._t, self._q,
                                               self._qdt, self._hq, self._tq, self._o,
                                               stream if stream is not None else _stream()))
