"""Multi-layer decode steps (kvmix_append_attend_layers / kvmix_attend_layers) with
programmatic dependent launch between layers: a layer's attention launch may overlap the
previous layer's drain. The kernels are deterministic, so every output must be bit-identical
to the serialized launches (KVMIX_PDL=0) -- across Key-group age-outs, tiers that take other
kernels (3-bit Values), repeated caches (no overlap allowed) and an output buffer shared by
all layers (the last layer's result must win)."""
import numpy as np
import pytest
import torch

import paper_2506_08018_b200 as K

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


def run(pdl, steps=40, shared_out=False, repeat=False):
    K.set_knob("KVMIX_PDL", pdl)
    caches = make(0)
    if repeat:
        caches = caches[:3] + [caches[2]] + caches[3:]
    L, B, H, D = len(caches), 4, 8, 128
    g = torch.Generator(device="cuda").manual_seed(1)
    res = []
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
    K.set_knob("KVMIX_PDL", 1)
    return torch.stack(res).cpu().numpy(), [c.dump() for c in caches]


@pytest.mark.parametrize("shared_out,repeat", [(False, False), (True, False), (False, True)])
def test_pdl_matches_serialized(cuda, shared_out, repeat):
    a, da = run(1, shared_out=shared_out, repeat=repeat)
    b, db = run(0, shared_out=shared_out, repeat=repeat)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert da == db
