"""CUDA-graph capture of the attention calls (kvmix_attend / kvmix_attend_layers): a
captured call replays bit-identically to the eager call on new query values written in
place (the caches are read-only for attention; scratch is sized by an eager warm-up call,
the multi-layer launch keeps its programmatic-dependent-launch edge inside the graph).
Appends are not capturable: their ring positions / counters are host bookkeeping, as in
the reference (cache.cpp:45-117)."""
import pytest
import torch

import paper_2506_08018_b200 as K

pytestmark = pytest.mark.gpu


def _stack(L, B=2, H=8, D=128, pre=900):
    torch.manual_seed(0)
    caches = []
    for l in range(L):
        kb, vb, r = (3, 4, 0.2) if l < 2 else (2, 2, 0.1)
        c = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, r, r, 32), B, H, D, capacity_tokens=pre + 64,
                           tail_dtype=torch.float16)
        c.append(torch.randn(B, H, pre, D, device="cuda", dtype=torch.float16),
                 torch.randn(B, H, pre, D, device="cuda", dtype=torch.float16))
        for _ in range(5):  # a few decode appends: window tokens in the ring
            x = torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16)
            c.append(x, x)
        caches.append(c)
    return caches


@pytest.mark.parametrize("L,G", [(6, 1), (4, 4), (1, 1)])
def test_captured_attention_replays_bit_identical(cuda, L, G):
    B, H, D = 2, 8, 128
    caches = _stack(L, B, H, D)
    qs = [torch.randn(B, H * G, 1, D, device="cuda", dtype=torch.float16) for _ in range(L)]
    outs = [torch.empty(B, H * G, 1, D, device="cuda") for _ in range(L)]
    K.attend_layers(caches, qs, outs)  # warm-up: scratch sized outside the capture
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        K.attend_layers(caches, qs, outs, stream=s.cuda_stream)
    for _ in range(3):
        for q in qs:
            q.copy_(torch.randn_like(q))
        g.replay()
        torch.cuda.synchronize()
        got = torch.stack(outs).clone()
        ref = [torch.empty_like(o) for o in outs]
        K.attend_layers(caches, qs, ref)
        torch.cuda.synchronize()
        assert torch.equal(got, torch.stack(ref))
