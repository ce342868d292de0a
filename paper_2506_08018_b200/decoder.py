"""Toy decoder through the device caches: the reference's
`CachedDecoder` / `generate` / `generate_recompute_reference` (toymodel.hpp:126-148,
toymodel.cpp:668-750) with the per-layer `append` + `attend` pair served by
`kvmix_append_attend` on the device, and the recompute oracle as a plain torch fp32 causal
forward.

Differences from the reference, on purpose: weights are random (torch, seeded) instead of
the reference's RNG init / KVTM checkpoint (a model, not the hot path); the default shape
uses head_dim 64 (the device cache serves head_dim 64/128 on the tensor-core path); the
dense math (projections, RMSNorm, erf-GELU, unembedding) runs as torch fp32 ops on the
GPU. The structure and the formulas are the reference's: x = embedding[token] +
pos_embedding[pos]; per layer h = rmsnorm(x) (eps inside the sqrt, toymodel.cpp:545-550),
q/k/v = h W, attention over the layer cache, x += a W_o, h = rmsnorm(x), x += gelu(h W_in)
W_out (gelu = 0.5 x (1 + erf(x / sqrt 2)), :552); logits = rmsnorm(x) W_unembed; greedy
argmax takes the first maximum (:554-560).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

from .attention import append_attend
from .cache import KVLayerCache
from .config import ModelQuantConfig, full_precision_config

NORM_EPS = 1e-5


@dataclass
class ToyHyperparams:
    """toymodel.hpp:35-45 (head_dim 64 here: see the module docstring)."""
    vocab_size: int = 256
    d_model: int = 256
    n_layers: int = 4
    n_heads: int = 4
    head_dim: int = 64
    d_ff: int = 512
    max_seq: int = 256

    def validate(self) -> None:
        if min(self.vocab_size, self.d_model, self.n_layers, self.n_heads, self.head_dim, self.d_ff,
               self.max_seq) < 1:
            raise ValueError("toy hyperparameters must be positive")
        if self.n_heads * self.head_dim != self.d_model:
            raise ValueError("d_model must equal n_heads * head_dim")


@dataclass
class ToyTransformer:
    hp: ToyHyperparams
    embedding: torch.Tensor          # [vocab, d_model]
    pos_embedding: torch.Tensor      # [max_seq, d_model]
    layers: list = field(default_factory=list)  # dicts of w_q, w_k, w_v, w_o, w_ff_in, w_ff_out, gains
    final_norm_gain: torch.Tensor = None
    unembedding: torch.Tensor = None  # [d_model, vocab]

    @staticmethod
    def random(hp: ToyHyperparams, seed: int = 0, device="cuda") -> "ToyTransformer":
        hp.validate()
        g = torch.Generator(device="cpu").manual_seed(seed)

        def w(*shape, scale):
            return (torch.randn(*shape, generator=g) * scale).to(device)

        dm, dff = hp.d_model, hp.d_ff
        layers = []
        for _ in range(hp.n_layers):
            layers.append({
                "w_q": w(dm, dm, scale=1 / math.sqrt(dm)), "w_k": w(dm, dm, scale=1 / math.sqrt(dm)),
                "w_v": w(dm, dm, scale=1 / math.sqrt(dm)), "w_o": w(dm, dm, scale=0.5 / math.sqrt(dm)),
                "w_ff_in": w(dm, dff, scale=1 / math.sqrt(dm)), "w_ff_out": w(dff, dm, scale=0.5 / math.sqrt(dff)),
                "attn_norm_gain": 1 + w(dm, scale=0.1), "mlp_norm_gain": 1 + w(dm, scale=0.1),
            })
        return ToyTransformer(hp, w(hp.vocab_size, dm, scale=1.0), w(hp.max_seq, dm, scale=0.5), layers,
                              1 + w(dm, scale=0.1), w(dm, hp.vocab_size, scale=1 / math.sqrt(dm)))


def rmsnorm(x: torch.Tensor, gain: torch.Tensor) -> torch.Tensor:
    return x * gain * torch.rsqrt((x * x).mean(-1, keepdim=True) + NORM_EPS)


def gelu(x: torch.Tensor) -> torch.Tensor:
    return 0.5 * x * (1.0 + torch.erf(x * 0.70710678))


def _check_token(hp: ToyHyperparams, token: int) -> None:
    if token < 0 or token >= hp.vocab_size:
        raise ValueError(f"token id {token} outside vocabulary")


class CachedDecoder:
    """toymodel.hpp:126-139: one KVLayerCache per layer (batch 1, n_heads KV heads);
    quant None = the full-precision config (r = 1: nothing is ever quantized)."""

    def __init__(self, m: ToyTransformer, quant: ModelQuantConfig | None = None, device="cuda"):
        hp = m.hp
        cfg = quant if quant is not None else full_precision_config(hp.n_layers)
        cfg.validate()
        if len(cfg.layers) != hp.n_layers:
            raise ValueError(f"quant config covers {len(cfg.layers)} layers, model has {hp.n_layers}")
        self.m = m
        self.caches = [KVLayerCache(cfg.layers[l], 1, hp.n_heads, hp.head_dim, capacity_tokens=hp.max_seq)
                       for l in range(hp.n_layers)]
        self.pos = 0

    def position(self) -> int:
        return self.pos

    def layer_cache(self, l: int) -> KVLayerCache:
        return self.caches[l]

    def step(self, token: int) -> torch.Tensor:
        """Logits [vocab] for this position (toymodel.cpp:687-737)."""
        m, hp = self.m, self.m.hp
        if self.pos >= hp.max_seq:
            raise ValueError("decode position exceeds max_seq")
        _check_token(hp, token)
        nh, D = hp.n_heads, hp.head_dim
        x = m.embedding[token] + m.pos_embedding[self.pos]
        for l, w in enumerate(m.layers):
            h = rmsnorm(x, w["attn_norm_gain"])
            q = (h @ w["w_q"]).view(1, nh, 1, D)
            k = (h @ w["w_k"]).view(1, nh, 1, D)
            v = (h @ w["w_v"]).view(1, nh, 1, D)
            a = append_attend(self.caches[l], k, v, q).output.reshape(-1)
            x = x + a @ w["w_o"]
            h = rmsnorm(x, w["mlp_norm_gain"])
            x = x + gelu(h @ w["w_ff_in"]) @ w["w_ff_out"]
        self.pos += 1
        return rmsnorm(x, m.final_norm_gain) @ m.unembedding

    def prefill(self, tokens) -> torch.Tensor:
        """Bulk full-precision causal forward, its per-layer K/V appended in one call each
        (toymodel.cpp:739-747); returns the last position's logits."""
        if self.pos != 0:
            raise ValueError("prefill requires an empty decoder")
        logits, keys, values = causal_forward(self.m, tokens)
        for c, k, v in zip(self.caches, keys, values):
            c.append(k, v)
        self.pos = len(tokens)
        return logits


def causal_forward(m: ToyTransformer, tokens):
    """Full-sequence fp32 forward without a cache: last-position logits and each layer's
    K/V [1, n_heads, n, head_dim] (the reference's causal_forward_f32, toymodel.cpp:570-666)."""
    hp = m.hp
    n, nh, D = len(tokens), hp.n_heads, hp.head_dim
    if n < 1 or n > hp.max_seq:
        raise ValueError("sequence length outside [1, max_seq]")
    for t in tokens:
        _check_token(hp, int(t))
    ids = torch.as_tensor(list(tokens), device=m.embedding.device)
    x = m.embedding[ids] + m.pos_embedding[:n]
    mask = torch.full((n, n), float("-inf"), device=x.device).triu(1)
    keys, values = [], []
    for w in m.layers:
        h = rmsnorm(x, w["attn_norm_gain"])
        q = (h @ w["w_q"]).view(n, nh, D).transpose(0, 1)
        k = (h @ w["w_k"]).view(n, nh, D).transpose(0, 1)
        v = (h @ w["w_v"]).view(n, nh, D).transpose(0, 1)
        keys.append(k.unsqueeze(0).contiguous())
        values.append(v.unsqueeze(0).contiguous())
        s = (q @ k.transpose(1, 2)) * (1.0 / math.sqrt(D)) + mask
        a = (torch.softmax(s, dim=-1) @ v).transpose(0, 1).reshape(n, hp.d_model)
        x = x + a @ w["w_o"]
        h = rmsnorm(x, w["mlp_norm_gain"])
        x = x + gelu(h @ w["w_ff_in"]) @ w["w_ff_out"]
    return rmsnorm(x[-1], m.final_norm_gain) @ m.unembedding, keys, values


def _argmax(v: torch.Tensor) -> int:
    return int(torch.argmax(v).item())  # first maximum, like toymodel.cpp:554-560


def generate(m: ToyTransformer, prompt, max_new_tokens: int, quant: ModelQuantConfig | None = None) -> list[int]:
    """Greedy decoding through the device caches (toymodel.hpp:141-143): the prompt is fed
    token by token through step(), then max_new_tokens argmax tokens."""
    if len(prompt) < 1:
        raise ValueError("prompt must hold at least one token")
    if max_new_tokens < 0:
        raise ValueError("max_new_tokens must be >= 0")
    out = [int(t) for t in prompt]
    if max_new_tokens == 0:
        return out
    if len(prompt) + max_new_tokens > m.hp.max_seq:
        raise ValueError("prompt plus generated tokens exceed max_seq")
    dec = CachedDecoder(m, quant)
    logits = None
    for t in out:
        logits = dec.step(t)
    for i in range(max_new_tokens):
        nxt = _argmax(logits)
        out.append(nxt)
        if i + 1 < max_new_tokens:
            logits = dec.step(nxt)
    return out


def generate_recompute_reference(m: ToyTransformer, prompt, max_new_tokens: int) -> list[int]:
    """Oracle decoder (toymodel.hpp:145-148): no cache, the causal forward over the whole
    sequence for every generated token."""
    out = [int(t) for t in prompt]
    for _ in range(max_new_tokens):
        logits, _, _ = causal_forward(m, out)
        out.append(_argmax(logits))
    return out
