"""N>1 path on CPU: world_size-2 gloo processes shard (batch x KV-head) work with the
plan used on the GPUs, compute their shard with the oracle, and all-gather; the result must
equal the unsharded computation bit-for-bit (the shards are independent)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2506_08018_b200.shard import ShardPlan, split_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = [("batch", 2, 2, 2), ("head", 1, 4, 8), ("batch", 3, 2, 4)]
D, T = 64, 300


def _inputs(B, H, Hq):
    return O.random_h16(3, (B, Hq, 1, D)), O.random_h16(1, (B, H, T, D)), O.random_h16(2, (B, H, T, D))


def _worker(rank, world, port, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    for mode, B, H, Hq in CASES:
        q, k, v = _inputs(B, H, Hq)
        res = _shard(rank, world, mode, B, H, Hq, q, k, v)
        if rank == 0:
            ret.put(res)
    dist.barrier()
    dist.destroy_process_group()


def _shard(rank, world, mode, B, H, Hq, q, k, v):
    plan = ShardPlan(B, H, Hq, world, rank, mode=mode)
    cache = O.CacheOracle(2, 2, 0.1, 0.1, 32, plan.local_batch, plan.local_heads, k.shape[3])
    t = k.shape[2]
    for s0 in range(0, t, 97):  # prefill chunks then decode-sized appends
        s1 = min(t, s0 + 97)
        cache.append(plan.kv(k)[:, :, s0:s1], plan.kv(v)[:, :, s0:s1])
    ks, vs = cache.snapshot()
    lq = plan.q(q)
    G = Hq // H
    lqr = lq.reshape(lq.shape[0], lq.shape[1] // G, G * lq.shape[2], lq.shape[3])
    out, _ = O.attend_f32(lqr, ks, vs)
    full = plan.gather(torch.from_numpy(out.reshape(lq.shape)))
    mem = torch.tensor([cache.memory_usage()["total_bits"]], dtype=torch.int64)
    dist.all_reduce(mem)
    return full.numpy(), int(mem.item())


def test_sharded_equals_unsharded():
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, ret)) for r in range(2)]
    for p in procs:
        p.start()
    results = [ret.get(timeout=300) for _ in CASES]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for (mode, B, H, Hq), (full, mem) in zip(CASES, results):
        _check(B, H, Hq, full, mem)


def _check(B, H, Hq, full, mem):
    q, k, v = _inputs(B, H, Hq)
    # unsharded reference
    cache = O.CacheOracle(2, 2, 0.1, 0.1, 32, B, H, D)
    for s0 in range(0, T, 97):
        cache.append(k[:, :, s0:s0 + 97], v[:, :, s0:s0 + 97])
    ks, vs = cache.snapshot()
    G = Hq // H
    out, _ = O.attend_f32(q.reshape(B, H, G, D), ks, vs)
    assert np.array_equal(full, out.reshape(B, Hq, 1, D))
    # per-shard accounting sums to the whole (payload words can differ only for Mixed3)
    assert mem == cache.memory_usage()["total_bits"]


def test_split_range_covers():
    for n in (1, 7, 16, 33):
        for w in (1, 2, 3, 8):
            got = [split_range(n, w, r) for r in range(w)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert max(h - l for l, h in got) - min(h - l for l, h in got) <= 1
