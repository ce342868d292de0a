import numpy as np, torch, os, sys
sys.path.insert(0, "/root/repo")
import oracle as O
import paper_2506_08018_b200 as K
def build(kb, vb, r, gs, B, H, D, chunks, seed=7, tail=torch.float32):
    cap = sum(chunks) + 16
    dev = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, r, r, gs), B, H, D, capacity_tokens=cap, tail_dtype=tail)
    for i, t in enumerate(chunks):
        k = O.random_h16(seed + 2 * i, (B, H, t, D)); v = O.random_h16(seed + 2 * i + 1, (B, H, t, D))
        dev.append(k, v)
    return dev
for (B, H, chunks, tail) in [(1, 32, [4032] + [1] * 64, torch.float32), (1, 32, [4032] + [1] * 64, torch.float16),
                             (2, 4, [1000] + [1] * 20, torch.float32), (1, 1, [200] + [1] * 5, torch.float32)]:
    dev = build(2, 2, 0.1, 32, B, H, 128, chunks, tail=tail)
    q = torch.from_numpy(O.random_h16(5, (B, H, 1, 128))).cuda()
    ref = K.reference_attend(q, dev).output
    out = K.attend(q, dev, checksum=False).output
    vmax = float(dev.snapshot_dequantized()[1].abs().max())
    err = ((out - ref).abs().amax(dim=-1) / vmax).flatten()
    print(B, H, tail, "ktail", dev.key_tail_tokens(), "vtail", dev.value_tail_tokens(), "T", dev.total_tokens(),
          "max err", float(err.max()), "bad heads", int((err > 1e-4).sum()), "of", err.numel())
