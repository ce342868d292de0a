"""Quantize/pack throughput sweep (BASELINE configs[4]): bits {2,3,4} x group size {32,64,128},
Keys and Values, on a [16, 32, 8192, 128] fp16 tensor (1 GiB) resident in HBM; CUDA events,
median of 5. Algorithmic bytes = fp16 input + packed payload + binary16 meta."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_08018_b200 as K  # noqa: E402

B, H, T, D = 16, 32, 8192, 128
x = torch.randn(B, H, T, D, device="cuda", dtype=torch.float16)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for key in (True, False):
    for bits in (2, 3, 4):
        for gs in (32, 64, 128):
            fn = K.quantize_key_tensor if key else K.quantize_value_tensor
            spec = K.QuantSpec(bits, K.Grouping(0 if key else 1), gs)
            fn(x, spec)
            ts = []
            for _ in range(5):
                e0.record()
                qg = fn(x, spec)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            n = x.numel()
            payload = K.packed_word_count(n, bits) * 4
            groups = (B * H * D * (T // gs)) if key else (B * H * T * ((D + gs - 1) // gs))
            alg = n * 2 + payload + groups * 4
            print(f"{'key  ' if key else 'value'} bits {bits} gs {gs:3d}: {ms:7.3f} ms  {alg / ms / 1e6:7.0f} GB/s algorithmic")
