"""In-stream attention time per tier at the config-2 state (B16, H32, D128, ~8k ctx, decode
appends to the steady window), CUDA events, median of 20 launches per window length.
SHAPE=B,H,G,CTX overrides the shape (e.g. SHAPE=8,8,4,32768 for the Mistral-7B GQA config)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_08018_b200 as K  # noqa: E402

B, H, D, CTX = 16, 32, 128, 8192
G = 1
if os.environ.get("SHAPE"):
    B, H, G, CTX = (int(x) for x in os.environ["SHAPE"].split(","))
torch.manual_seed(0)
TIERS = ((2, 2, 0.1), (3, 4, 0.2))
if os.environ.get("TIERS"):  # e.g. TIERS=2:3:0.1,3:3:0.2
    TIERS = tuple((int(a), int(b), float(r)) for a, b, r in (t.split(":") for t in os.environ["TIERS"].split(",")))
for kb, vb, r in TIERS:
    c = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, r, r, 32), B, H, D, capacity_tokens=CTX + 64, tail_dtype=torch.float16)
    c.append(torch.randn(B, H, CTX - 64, D, device="cuda", dtype=torch.float16),
             torch.randn(B, H, CTX - 64, D, device="cuda", dtype=torch.float16))
    q = torch.randn(B, H * G, 1, D, device="cuda", dtype=torch.float16)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = []
    for s in range(40):
        x = torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16)
        c.append(x, x)
        ts = []
        for _ in range(5):
            e0.record()
            K.attend(q, c, checksum=False)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        res.append(min(ts))
        if os.environ.get("VERBOSE"):
            print(s, c.key_tail_tokens(), c.value_tail_tokens(), " ".join(f"{x:.0f}" for x in ts))
    gb = c.algorithmic_bytes() / 1e9
    print(f"K{kb}V{vb}: median {statistics.median(res):.1f} us, min {min(res):.1f}, max {max(res):.1f} "
          f"({gb / statistics.median(res) * 1e6:.0f} GB/s algorithmic at the median)")
