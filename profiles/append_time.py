"""In-stream time of a decode append (config-2 K2V2 layer state), CUDA events over 200 appends."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_08018_b200 as K  # noqa: E402

B, H, D, CTX = 16, 32, 128, 8192
torch.manual_seed(0)
c = K.KVLayerCache(K.LayerQuantConfig(0, 2, 2, 0.1, 0.1, 32), B, H, D, capacity_tokens=CTX + 512, tail_dtype=torch.float16)
c.append(torch.randn(B, H, CTX - 256, D, device="cuda", dtype=torch.float16),
         torch.randn(B, H, CTX - 256, D, device="cuda", dtype=torch.float16))
xs = torch.randn(256, B, H, 1, D, device="cuda", dtype=torch.float16)
for i in range(40):
    c.append(xs[i], xs[i])
q = torch.randn(B, H, 1, D, device="cuda", dtype=torch.float16)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for i in range(40, 240):
    c.append(xs[i], xs[i])
e1.record()
e1.synchronize()
print(f"append alone: {e0.elapsed_time(e1) / 200 * 1e3:.2f} us per decode append (incl. K-group ageing steps)")
torch.cuda.synchronize()
e0.record()
for i in range(40):
    K.attend(q, c, checksum=False)
e1.record()
e1.synchronize()
print(f"attend alone: {e0.elapsed_time(e1) / 40 * 1e3:.2f} us")
print("state: total", c.total_tokens(), "key_tail", c.key_tail_tokens(), "value_tail", c.value_tail_tokens(),
      "qk", c.quantized_key_tokens(), "qv", c.quantized_value_tokens())
for i in range(240, 250):
    c.append(xs[i], xs[i])
    torch.cuda.synchronize()
    e0.record()
    K.attend(q, c, checksum=False)
    e1.record()
    e1.synchronize()
    print(i, c.key_tail_tokens(), c.value_tail_tokens(), f"{e0.elapsed_time(e1) * 1e3:.1f} us",
          K.launch_count_of("attend_mma_kernel"), K.launch_count_of("attend_generic_kernel"))
