"""Multi-layer decode steps (kvmix_append_attend_layers / kvmix_attend_layers).

Layers served by the same IMMA kernel instance share ONE launch (attend_mma_layers_kernel,
KVMIX_LAYERS=1, the default); launches overlap the previous launch's drain (programmatic
dependent launch). The kernels are deterministic, so every output must be bit-identical to
the serialized launches (KVMIX_PDL=0) -- across Key-group age-outs, tiers that take other
kernels (3-bit Values), repeated caches (no overlap allowed: per-layer path) and an output
buffer shared by all layers (the last layer's result must win: per-layer path). The shared
launch splits each layer over fewer warps than a per-layer launch, so its outputs equal the
per-layer launches' (KVMIX_LAYERS=0) up to fp32 merge order, and the caches bit for bit."""
import numpy as np
import pytest
import torch

import paper_2506_08018_b200 as K
from paper_2506_08018_b200 import _lib

pytestmark = pytest.mark.gpu

TIERS = [(2, 2, 0.1), (3, 4, 0.2), (2, 3, 0.1), (4, 2, 0.1), (2, 2, 0.1), (2, 2, 0.1)]


def make(seed, B=4, H=8, D=128, pre=700):
    torch.manual_seed(seed)
    caches = []
    for kb, vb, r in TIERS:
        c = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, r, r, 32), B, H, D, capacity_tokens=pre + 200,
                           tail_dtype=torch.float16)
        c.append(torch.randn(B, H, pre, D, device="cuda", dtype=torch.float16),
                 torch.randn(B, H, pre, D, device="cuda", dtype=torch.float16))
        caches.append(c)
    return caches


def run(pdl, steps=40, shared_out=False, repeat=False, layers=1, count=False):
    K.set_knob("KVMIX_PDL", pdl)
    K.set_knob("KVMIX_LAYERS", layers)
    caches = make(0)
    if repeat:
        caches = caches[:3] + [caches[2]] + caches[3:]
    L, B, H, D = len(caches), 4, 8, 128
    g = torch.Generator(device="cuda").manual_seed(1)
    res = []
    n0 = _lib.launch_count_of("attend_mma_layers_kernel")
    for s in range(steps):
        ks = [torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16, generator=g) for _ in range(L)]
        vs = [torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16, generator=g) for _ in range(L)]
        qs = [torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16, generator=g) for _ in range(L)]
        if shared_out:
            o = torch.empty(B, H, 1, D, device="cuda")
            outs = [o] * L
        else:
            outs = [torch.empty(B, H, 1, D, device="cuda") for _ in range(L)]
        K.append_attend_layers(caches, ks, vs, qs, outs)
        res.append(torch.stack([x.clone() for x in outs]))
    torch.cuda.synchronize()
    n1 = _lib.launch_count_of("attend_mma_layers_kernel")
    K.set_knob("KVMIX_PDL", 1)
    K.set_knob("KVMIX_LAYERS", 1)
    out = (torch.stack(res).cpu().numpy(), [c.dump() for c in caches])
    return out + (n1 - n0,) if count else out


@pytest.mark.parametrize("layers", [1, 0])
@pytest.mark.parametrize("shared_out,repeat", [(False, False), (True, False), (False, True)])
def test_pdl_matches_serialized(cuda, shared_out, repeat, layers):
    a, da = run(1, shared_out=shared_out, repeat=repeat, layers=layers)
    b, db = run(0, shared_out=shared_out, repeat=repeat, layers=layers)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert da == db


def test_shared_launch_matches_per_layer(cuda):
    """One launch per kernel instance == one launch per layer (caches bit for bit, outputs
    to fp32 merge order); the shared launch really ran (3 per step: K2V2 x3, K3V4, K4V2;
    the 3-bit-Value layer runs alone on the warp-specialized kernel)."""
    steps = 40
    a, da, na = run(1, steps=steps, layers=1, count=True)
    b, db, nb = run(1, steps=steps, layers=0, count=True)
    assert da == db
    assert na == 3 * steps and nb == 0
    np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("G,D", [(4, 128), (1, 64), (2, 128)])
def test_shared_launch_gqa_and_head_dims(cuda, G, D):
    """GQA (row passes inside the launch), D = 64 and two query rows per KV head through
    kvmix_append_attend_layers and kvmix_attend_layers: shared launch == per-layer launches."""
    B, H, pre, L = 3, 4, 500, 5

    def go(layers):
        K.set_knob("KVMIX_LAYERS", layers)
        torch.manual_seed(3)
        caches = []
        for _ in range(L):
            c = K.KVLayerCache(K.LayerQuantConfig(0, 2, 2, 0.1, 0.1, 32), B, H, D, capacity_tokens=pre + 64,
                               tail_dtype=torch.float16)
            c.append(torch.randn(B, H, pre, D, device="cuda", dtype=torch.float16),
                     torch.randn(B, H, pre, D, device="cuda", dtype=torch.float16))
            caches.append(c)
        g = torch.Generator(device="cuda").manual_seed(5)
        res = []
        for s in range(12):
            ks = [torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16, generator=g) for _ in range(L)]
            vs = [torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16, generator=g) for _ in range(L)]
            qs = [torch.randn(B, H * G, 1, D, device="cuda", dtype=torch.float16, generator=g) for _ in range(L)]
            outs = [torch.empty(B, H * G, 1, D, device="cuda") for _ in range(L)]
            K.append_attend_layers(caches, ks, vs, qs, outs)
            res.append(torch.stack(outs))
            outs2 = [torch.empty(B, H * G, 1, D, device="cuda") for _ in range(L)]
            K.attend_layers(caches, qs, outs2)
            res.append(torch.stack(outs2))
        torch.cuda.synchronize()
        K.set_knob("KVMIX_LAYERS", 1)
        return torch.stack(res).cpu().numpy(), [c.dump() for c in caches]

    n0 = _lib.launch_count_of("attend_mma_layers_kernel")
    a, da = go(1)
    assert _lib.launch_count_of("attend_mma_layers_kernel") - n0 == 24
    b, db = go(0)
    assert da == db
    np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6)


def test_more_layers_than_one_launch_holds(cuda):
    """34 same-tier layers: the shared launch holds at most 32 layers' parameters (kernel
    parameter space), so the run splits into two launches; results == per-layer launches."""
    B, H, D, L, pre = 2, 4, 128, 34, 300

    def go(layers):
        K.set_knob("KVMIX_LAYERS", layers)
        torch.manual_seed(11)
        caches = []
        for _ in range(L):
            c = K.KVLayerCache(K.LayerQuantConfig(0, 2, 2, 0.1, 0.1, 32), B, H, D, capacity_tokens=pre + 16,
                               tail_dtype=torch.float16)
            c.append(torch.randn(B, H, pre, D, device="cuda", dtype=torch.float16),
                     torch.randn(B, H, pre, D, device="cuda", dtype=torch.float16))
            caches.append(c)
        g = torch.Generator(device="cuda").manual_seed(12)
        res = []
        for _ in range(4):
            ks = [torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16, generator=g) for _ in range(L)]
            vs = [torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16, generator=g) for _ in range(L)]
            qs = [torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16, generator=g) for _ in range(L)]
            outs = [torch.empty(B, H, 1, D, device="cuda") for _ in range(L)]
            K.append_attend_layers(caches, ks, vs, qs, outs)
            res.append(torch.stack(outs))
        torch.cuda.synchronize()
        K.set_knob("KVMIX_LAYERS", 1)
        return torch.stack(res).cpu().numpy(), [c.dump() for c in caches]

    n0 = _lib.launch_count_of("attend_mma_layers_kernel")
    a, da = go(1)
    assert _lib.launch_count_of("attend_mma_layers_kernel") - n0 == 2 * 4
    b, db = go(0)
    assert da == db
    np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6)


def test_error_mid_stack_completes_earlier_layers(cuda):
    """A layer that raises (here: capacity exhausted) propagates the error; the layers
    before it are appended and attended as by the per-layer loop (their queued shared
    launch runs first)."""
    B, H, D, pre = 2, 4, 128, 200
    caches = []
    for cap in (pre + 8, pre + 8, pre):  # the third cache is full
        c = K.KVLayerCache(K.LayerQuantConfig(0, 2, 2, 0.1, 0.1, 32), B, H, D, capacity_tokens=cap,
                           tail_dtype=torch.float16)
        c.append(torch.randn(B, H, pre, D, device="cuda", dtype=torch.float16),
                 torch.randn(B, H, pre, D, device="cuda", dtype=torch.float16))
        caches.append(c)
    ks = [torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16) for _ in range(3)]
    qs = [torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16) for _ in range(3)]
    outs = [torch.full((B, H, 1, D), float("nan"), device="cuda") for _ in range(3)]
    with pytest.raises(Exception):
        K.append_attend_layers(caches, ks, ks, qs, outs)
    torch.cuda.synchronize()
    assert [c.total_tokens() for c in caches[:2]] == [pre + 1, pre + 1]
    for l in range(2):  # earlier layers: appended and attended
        ref = K.attend(qs[l], caches[l]).output
        np.testing.assert_allclose(outs[l].cpu().numpy(), ref.cpu().numpy(), rtol=1e-5, atol=1e-6)
