import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2506_08018_b200 as K
torch.manual_seed(0)
B, H, D, L, pre = 2, 8, 128, 6, 900
caches = []
for l in range(L):
    kb, vb, r = (3, 4, 0.2) if l < 2 else (2, 2, 0.1)
    c = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, r, r, 32), B, H, D, capacity_tokens=pre + 64, tail_dtype=torch.float16)
    c.append(torch.randn(B, H, pre, D, device="cuda", dtype=torch.float16), torch.randn(B, H, pre, D, device="cuda", dtype=torch.float16))
    caches.append(c)
qs = [torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16) for _ in range(L)]
outs = [torch.empty(B, H, 1, D, device="cuda") for _ in range(L)]
K.attend_layers(caches, qs, outs)  # warm-up (scratch sized outside capture)
torch.cuda.synchronize()
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    K.attend_layers(caches, qs, outs, stream=s.cuda_stream)
for it in range(3):
    for q in qs: q.copy_(torch.randn_like(q))
    g.replay(); torch.cuda.synchronize()
    got = torch.stack(outs).clone()
    ref = [torch.empty_like(o) for o in outs]
    K.attend_layers(caches, qs, ref); torch.cuda.synchronize()
    print(it, (got - torch.stack(ref)).abs().max().item())
print("graph ok")
