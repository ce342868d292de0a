"""Attention kernel time vs. the full-precision window length (config-2 K2V2 layer:
B16, H32, D128, ~8k context): one decode append per step, attend timed with CUDA events.

  python profiles/tail_sweep.py [KVMIX_TAIL_UNIT values are read from the environment]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_08018_b200 as K  # noqa: E402

B, H, D, CTX = 16, 32, 128, 8192
kb, vb = (int(x) for x in os.environ.get("TIER", "2,2").split(","))
r = 0.1
torch.manual_seed(0)
c = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, r, r, 32), B, H, D, capacity_tokens=CTX + 128, tail_dtype=torch.float16)
c.append(torch.randn(B, H, CTX - 64, D, device="cuda", dtype=torch.float16),
         torch.randn(B, H, CTX - 64, D, device="cuda", dtype=torch.float16))
q = torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for s in range(64):
    x = torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16)
    c.append(x, x)
    K.attend(q, c, checksum=False)
    ts = []
    for _ in range(5):
        e0.record()
        K.attend(q, c, checksum=False)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"step {s:2d} total {c.total_tokens()} key_tail {c.key_tail_tokens():3d} value_tail {c.value_tail_tokens():3d} "
          f"attend {min(ts):7.1f} us")
