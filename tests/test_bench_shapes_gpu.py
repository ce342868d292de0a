"""GPU parity at the BENCHMARKED shapes (BASELINE.json configs[1], [2], [3]).

The reference pins its fused attention against the dequantize-everything oracle over random
caches (acceptance.cpp:153-214). Here the device caches are built at the bench's sizes (B16 x
32 heads x 8k; B8 x 8 KV heads x 32k with G = 4 query heads per KV head; one 40-head batch row
at 128k), driven through >= 40 single-token decode steps with append_attend (the fused
prologue append, across a Key-group age-out), and sampled (b, kv-head) slices are compared
with the CPU oracle: the snapshot bit for bit, the attention output within the parity tier's
stated tolerance (2e-6 * max|V| vs fp64 over the reference's dequantized cache).

Slices are independent (attention.cpp:36-41) except for the Mixed3 narrow slots, which follow
the global stream index mod 11: the oracle for slice (b, h) is a cache whose head r = (b*H + h)
mod 11 holds the slice (the other heads zeros) -- the same narrow pattern, at <= 11x the
slice's cost instead of the whole batch's.
"""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2506_08018_b200 as K

pytestmark = pytest.mark.gpu

TOL = 2e-6  # * max|V|, as tests/test_attention_gpu.py ATTN_TOL_F64


class SliceOracle:
    def __init__(self, kb, vb, r, gs, H, D, b, h):
        self.r = (b * H + h) % 11
        self.ora = O.CacheOracle(kb, vb, r, r, gs, 1, self.r + 1, D)

    def append(self, k, v):  # k, v: [t, D] fp32 of this slice
        t, D = k.shape
        kp = np.zeros((1, self.r + 1, t, D), np.float32)
        vp = np.zeros_like(kp)
        kp[0, self.r], vp[0, self.r] = k, v
        self.ora.append(kp, vp)

    def snapshot(self):
        ks, vs = self.ora.snapshot()
        return ks[0, self.r], vs[0, self.r]


def _run_shape(kb, vb, r, B, H, G, ctx, samples, n_decode=44, checks=(20, 43), seed=0, chunk=None):
    D, gs = 128, 32
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(seed)
    cache = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, r, r, gs), B, H, D, capacity_tokens=ctx + n_decode + 8,
                           tail_dtype=torch.float16)
    oras = {bh: SliceOracle(kb, vb, r, gs, H, D, *bh) for bh in samples}
    pre = ctx - n_decode
    chunk = chunk or pre
    for a in range(0, pre, chunk):  # prefill (chunked: a 128k prefill is a few GB of fp16)
        t = min(chunk, pre - a)
        k = torch.randn(B, H, t, D, device=dev, dtype=torch.float16, generator=gen)
        v = torch.randn(B, H, t, D, device=dev, dtype=torch.float16, generator=gen)
        cache.append(k, v)
        for (b, h), o in oras.items():
            o.append(k[b, h].float().cpu().numpy(), v[b, h].float().cpu().numpy())
        del k, v
    worst = 0.0
    n_mma0 = K.tensor_core_launches()
    qk0 = cache.quantized_key_tokens()
    for s in range(n_decode):
        k = torch.randn(B, H, 1, D, device=dev, dtype=torch.float16, generator=gen)
        v = torch.randn(B, H, 1, D, device=dev, dtype=torch.float16, generator=gen)
        q = torch.randn(B, H * G, 1, D, device=dev, dtype=torch.float16, generator=gen)
        res = K.append_attend(cache, k, v, q)
        for (b, h), o in oras.items():
            o.append(k[b, h].float().cpu().numpy(), v[b, h].float().cpu().numpy())
        if s in checks:
            out = res.output.cpu().numpy()
            ks, vs = cache.snapshot_dequantized()
            for (b, h), o in oras.items():
                ok, ov = o.snapshot()
                assert np.array_equal(ks[b, h].cpu().numpy().view(np.uint32), ok.view(np.uint32)), (b, h, s)
                assert np.array_equal(vs[b, h].cpu().numpy().view(np.uint32), ov.view(np.uint32)), (b, h, s)
                qs = q[b, h * G:(h + 1) * G, 0].float().cpu().numpy()  # the reference's t = G rows
                o64, _ = O.attend_f64(qs[None, None], ok[None, None], ov[None, None])
                err = float(np.abs(out[b, h * G:(h + 1) * G, 0] - o64[0, 0]).max() / np.abs(ov).max())
                worst = max(worst, err)
                assert err <= TOL, (b, h, s, err)
            del ks, vs
    assert K.tensor_core_launches() > n_mma0  # the tensor-core kernel served the steps
    assert cache.quantized_key_tokens() > qk0  # a Key group aged out during the decode steps
    return worst


@pytest.mark.parametrize("kb,vb,r", [(2, 2, 0.1), (3, 4, 0.2)])
def test_config1_llama2_7b_8k_layer(cuda, kb, vb, r):
    """configs[1]: B16 x 32 heads x 8192 context, one layer per KVmix tier."""
    worst = _run_shape(kb, vb, r, 16, 32, 1, 8192, samples=[(0, 0), (5, 7), (15, 31)], seed=kb)
    print(f"configs[1] K{kb}V{vb}: worst err/max|V| = {worst:.2e}")


@pytest.mark.parametrize("kb,vb,r", [(2, 2, 0.1), (3, 4, 0.2)])
def test_config2_mistral_gqa_32k_layer(cuda, kb, vb, r):
    """configs[2]: B8 x 8 KV heads (G = 4 query heads each) x 32768 context: a KV head is
    split over dozens of warps (the stream-K merge path)."""
    worst = _run_shape(kb, vb, r, 8, 8, 4, 32768, samples=[(0, 0), (3, 5), (7, 7)], seed=10 + kb, chunk=8192)
    print(f"configs[2] K{kb}V{vb}: worst err/max|V| = {worst:.2e}")


def test_config3_llama2_13b_128k_slice(cuda):
    """configs[3]: one batch row of 40 heads at 131072 context (> 1024 blocks per Value fold,
    no test knob), K2/V2 r0.1."""
    worst = _run_shape(2, 2, 0.1, 1, 40, 1, 131072, samples=[(0, 0), (0, 22)], n_decode=40, checks=(39,),
                       seed=30, chunk=16384)
    print(f"configs[3] slice: worst err/max|V| = {worst:.2e}")


@pytest.mark.parametrize("G,ctx,B,H", [(1, 8192, 16, 32), (4, 32768, 8, 8)])
def test_shared_layer_launch_at_bench_shapes(cuda, G, ctx, B, H):
    """The bench's own path (kvmix_append_attend_layers: one attend_mma_layers_kernel launch
    per tier run) at the configs[1] / configs[2] shapes: a 4-layer stack (K3V4, K3V4, K2V2,
    K2V2) through 40 decode steps across a Key-group age-out; sampled (layer, b, kv-head)
    outputs vs fp64 attention over the device's bit-exact snapshot (pinned against the
    oracle by the tests above), within 2e-6 * max|V|."""
    from paper_2506_08018_b200 import _lib
    D, gs, n_decode = 128, 32, 40
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(7 + G)
    tiers = [(3, 4, 0.2), (3, 4, 0.2), (2, 2, 0.1), (2, 2, 0.1)]
    caches = []
    for kb, vb, r in tiers:
        c = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, r, r, gs), B, H, D, capacity_tokens=ctx + 8,
                           tail_dtype=torch.float16)
        for a in range(0, ctx - n_decode, 8192):
            t = min(8192, ctx - n_decode - a)
            c.append(torch.randn(B, H, t, D, device=dev, dtype=torch.float16, generator=gen),
                     torch.randn(B, H, t, D, device=dev, dtype=torch.float16, generator=gen))
        caches.append(c)
    L = len(caches)
    n0 = _lib.launch_count_of("attend_mma_layers_kernel")
    qk0 = caches[-1].quantized_key_tokens()
    samples = [(0, 0), (B // 2, H // 3), (B - 1, H - 1)]
    worst = 0.0
    for s in range(n_decode):
        ks = [torch.randn(B, H, 1, D, device=dev, dtype=torch.float16, generator=gen) for _ in range(L)]
        vs = [torch.randn(B, H, 1, D, device=dev, dtype=torch.float16, generator=gen) for _ in range(L)]
        qs = [torch.randn(B, H * G, 1, D, device=dev, dtype=torch.float16, generator=gen) for _ in range(L)]
        outs = [torch.empty(B, H * G, 1, D, device=dev) for _ in range(L)]
        K.append_attend_layers(caches, ks, vs, qs, outs)
        if s in (19, 39):
            for l, c in enumerate(caches):
                kd, vd = c.snapshot_dequantized()
                for b, h in samples:
                    kk = kd[b, h].cpu().numpy()
                    vv = vd[b, h].cpu().numpy()
                    qq = qs[l][b, h * G:(h + 1) * G, 0].float().cpu().numpy()
                    o64, _ = O.attend_f64(qq[None, None], kk[None, None], vv[None, None])
                    err = float(np.abs(outs[l][b, h * G:(h + 1) * G, 0].cpu().numpy() - o64[0, 0]).max()
                                / np.abs(vv).max())
                    worst = max(worst, err)
                    assert err <= TOL, (l, b, h, s, err)
                del kd, vd
    assert _lib.launch_count_of("attend_mma_layers_kernel") - n0 == 2 * n_decode  # one per tier run
    assert caches[-1].quantized_key_tokens() > qk0
    print(f"shared launch G={G}: worst err/max|V| = {worst:.2e}")
