"""Per-warp timeline of attend_mma_kernel (debug build with -DKVB_TRACE=1, KVMIX_LIB=...):
one config-2-shaped layer per tier, a few attends; prints start / end spreads and the
tail (time between the median warp end and the last warp end).

  KVMIX_LIB=abtmp/libTrace.so KVMIX_TRACE_FILE=/tmp/tr.bin python profiles/trace_attend.py
"""
import os
import struct
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_08018_b200 as K  # noqa: E402

B, H, D, CTX = 16, 32, 128, 8192
if os.environ.get("SHAPE"):
    B, H, _, CTX = (int(x) for x in os.environ["SHAPE"].split(","))
path = os.environ["KVMIX_TRACE_FILE"]
if os.path.exists(path):
    os.remove(path)
torch.manual_seed(0)
for kb, vb, r in ((2, 2, 0.1), (3, 4, 0.2)):
    c = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, r, r, 32), B, H, D, capacity_tokens=CTX + 64, tail_dtype=torch.float16)
    c.append(torch.randn(B, H, CTX - 64, D, device="cuda", dtype=torch.float16),
             torch.randn(B, H, CTX - 64, D, device="cuda", dtype=torch.float16))
    for _ in range(64):
        x = torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16)
        c.append(x, x)
    q = torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16)
    for _ in range(4):
        K.attend(q, c, checksum=False)
    torch.cuda.synchronize()
data = open(path, "rb").read()
off, n = 0, 0
while off < len(data):
    magic, nw, U, Gf = struct.unpack_from("<4Q", data, off)
    off += 32
    a = np.frombuffer(data, dtype=np.uint64, count=4 * nw, offset=off).reshape(nw, 4).astype(np.int64)
    off += 32 * nw
    n += 1
    a = a[a[:, 1] > 0]
    t0 = a[:, 0].min()
    st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
    units = (a[:, 3] & 0xffffffff) - (a[:, 3] >> 32)
    print(f"launch {n}: warps {len(a)}, U {U} Gf {Gf}: start spread {st.max():.1f} us, "
          f"end p0 {en.min():.1f} p10 {np.percentile(en, 10):.1f} p50 {np.median(en):.1f} p90 {np.percentile(en, 90):.1f} "
          f"max {en.max():.1f} us; busy mean {(en - st).mean():.1f} us; units/warp {units.min()}..{units.max()}")
    slow = np.argsort(en)[-5:]
    for i in slow:
        u0, u1 = int(a[i, 3] >> 32), int(a[i, 3] & 0xffffffff)
        print(f"   slow warp: start {st[i]:.1f} end {en[i]:.1f} sm {a[i, 2]} units [{u0}, {u1}) "
              f"bh {u0 // U}..{(u1 - 1) // U} local {u0 % U}..{(u1 - 1) % U}")

# per-SM view of the last K2V2 launch: is the imbalance per SM (placement) or per warp?
off, last = 0, None
while off < len(data):
    magic, nw, U, Gf = struct.unpack_from("<4Q", data, off)
    off += 32
    a = np.frombuffer(data, dtype=np.uint64, count=4 * nw, offset=off).reshape(nw, 4).astype(np.int64)
    off += 32 * nw
    if last is None or len(last) == len(a):
        last = a if last is None or n <= 4 else last
    if off > len(data) // 2:
        break
a = last[last[:, 1] > 0]
en = (a[:, 1] - a[:, 0].min()) / 1e3
sm = a[:, 2]
per_sm = np.array([en[sm == k].mean() for k in range(int(sm.max()) + 1) if (sm == k).any()])
spread_in_sm = np.array([en[sm == k].max() - en[sm == k].min() for k in range(int(sm.max()) + 1) if (sm == k).any()])
print(f"per-SM mean end: min {per_sm.min():.1f} p50 {np.median(per_sm):.1f} max {per_sm.max():.1f} us; "
      f"within-SM spread p50 {np.median(spread_in_sm):.1f} max {spread_in_sm.max():.1f} us")
print("slowest SMs:", np.argsort(per_sm)[-8:], "fastest:", np.argsort(per_sm)[:8])
