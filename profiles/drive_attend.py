"""ncu target: one config-2 layer per tier (B16, H32, D128, ~8k ctx), attend x3 each.

Usage (on the GPU box):
  ncu --set full --clock-control none --import-source on -k regex:attend_mma -s 2 -c 2 \
      -o gpurun_out/prof python profiles/drive_attend.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_08018_b200 as K  # noqa: E402

B, H, D, CTX = 16, 32, 128, 8192
G = 1
if os.environ.get("SHAPE"):  # B,H,G,CTX (e.g. 8,8,4,32768: the Mistral-7B GQA config)
    B, H, G, CTX = (int(x) for x in os.environ["SHAPE"].split(","))
ALL = [(2, 2, 0.1), (3, 4, 0.2), (2, 3, 0.1)]  # index 2: 3-bit Values (generic kernel)
tiers = ALL[:2]
if len(sys.argv) > 1:
    tiers = [ALL[int(i)] for i in sys.argv[1].split(",")]
torch.manual_seed(0)
for kb, vb, r in tiers:
    c = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, r, r, 32), B, H, D, capacity_tokens=CTX + 64, tail_dtype=torch.float16)
    c.append(torch.randn(B, H, CTX - 64, D, device="cuda", dtype=torch.float16),
             torch.randn(B, H, CTX - 64, D, device="cuda", dtype=torch.float16))
    for _ in range(64):
        x = torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16)
        c.append(x, x)
    q = torch.randn(B, H * G, 1, D, device="cuda", dtype=torch.float16)
    for _ in range(3):
        K.attend(q, c, checksum=False)
    torch.cuda.synchronize()
    print(f"K{kb}V{vb}: {c.algorithmic_bytes() / 1e6:.1f} MB algorithmic per attend")
