"""Multi-GPU partitioning of the hot path: batch x KV-head shards.

Every (b, kv-head) pair's append and attend touch only its own packed store and
full-precision window, and the shrink rule is uniform across (b, h), so a rank holding a
shard replays identical host bookkeeping and needs no data-path collective. One thing is
NOT local: the reference's Mixed3 narrow slots (3-bit layers) are a function of the global
stream index (quant.cpp:36-47, 77-95), so a shard's cache is placed in the global batch
(ShardPlan.place -> kvmix_cache_set_shard) to hold the unsharded cache's slice bit for bit.
Query heads travel with their KV head (GQA). The only exchange is the optional all-gather of
the attention output for a downstream projection (one [B, Hq, t, D] tensor per layer).
"""
from __future__ import annotations

import dataclasses


def split_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced range [lo, hi) of n units for `rank` of `world`."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclasses.dataclass
class ShardPlan:
    """Which slice of [B, H(kv), ...] a rank owns. mode 'batch' splits the batch (heads
    whole), 'head' splits KV heads (batch whole), chosen so every rank gets equal work when
    the divisibility allows."""
    B: int
    H: int
    Hq: int
    world: int
    rank: int
    mode: str = ""
    b0: int = 0
    b1: int = 0
    h0: int = 0
    h1: int = 0

    def __post_init__(self):
        if self.Hq % self.H:
            raise ValueError("query heads must be a multiple of KV heads")
        if not self.mode:
            self.mode = "batch" if self.B % self.world == 0 or self.H % self.world != 0 else "head"
        if self.mode == "batch":
            self.b0, self.b1 = split_range(self.B, self.world, self.rank)
            self.h0, self.h1 = 0, self.H
        elif self.mode == "head":
            self.b0, self.b1 = 0, self.B
            self.h0, self.h1 = split_range(self.H, self.world, self.rank)
        else:
            raise ValueError(f"unknown shard mode {self.mode}")

    @property
    def G(self) -> int:
        return self.Hq // self.H

    @property
    def local_batch(self) -> int:
        return self.b1 - self.b0

    @property
    def local_heads(self) -> int:
        return self.h1 - self.h0

    def kv(self, x):
        """Local slice of a [B, H, t, D] K/V tensor."""
        return x[self.b0:self.b1, self.h0:self.h1]

    def q(self, x):
        """Local slice of a [B, Hq, t, D] query tensor (query heads follow their KV head)."""
        return x[self.b0:self.b1, self.h0 * self.G:self.h1 * self.G]

    def gather(self, local_out, group=None):
        """All-gather the per-rank outputs back into [B, Hq, t, D] (torch.distributed)."""
        import torch
        import torch.distributed as dist

        parts = [None] * self.world
        dist.all_gather_object(parts, (self.b0, self.b1, self.h0, self.h1), group=group)
        # all_gather needs equal shapes: pad every shard to the largest (b, hq) extent
        mb = max(b1 - b0 for b0, b1, _, _ in parts)
        mh = max(h1 - h0 for _, _, h0, h1 in parts) * self.G
        pad = torch.zeros((mb, mh) + tuple(local_out.shape[2:]), dtype=local_out.dtype, device=local_out.device)
        pad[:local_out.shape[0], :local_out.shape[1]] = local_out
        buf = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(buf, pad, group=group)
        out = torch.empty((self.B, self.Hq) + tuple(local_out.shape[2:]), dtype=local_out.dtype, device=local_out.device)
        for (b0, b1, h0, h1), t in zip(parts, buf):
            out[b0:b1, h0 * self.G:h1 * self.G] = t[:b1 - b0, :(h1 - h0) * self.G]
        return out

    def place(self, cache) -> None:
        """Mark a freshly created device cache as this rank's slice (kvmix_cache_set_shard):
        its Mixed3 narrow slots then follow the global stream index, so the shard holds the
        unsharded cache's slice bit for bit (also for 3-bit layers)."""
        cache.set_shard(self.B, self.H, self.b0, self.h0)
