"""compute-sanitizer target: a small pass over every device path (quantize / pack /
dequantize, prefill + decode appends incl. Key-group age-outs, the fused append+attend,
the three tensor-core attention kernels (single-warp and warp-specialized IMMA, tcgen05) and the generic one, multi-row / GQA passes, snapshot and
segment export, multi-layer launches) on shapes small enough for memcheck / racecheck / synccheck to finish.

  compute-sanitizer --tool memcheck --target-processes all python profiles/sanitize_drive.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_08018_b200 as K  # noqa: E402

torch.manual_seed(0)
dev = "cuda"
x = torch.randn(1, 2, 128, 64, device=dev, dtype=torch.float16)
for bits in (2, 3, 4):
    for key in (True, False):
        spec = K.QuantSpec(bits, K.Grouping(0 if key else 1), 32)
        qg = (K.quantize_key_tensor if key else K.quantize_value_tensor)(x, spec)
        qg.dequantize()
# single-warp IMMA, tcgen05 + window launch, warp-specialized IMMA (SANITIZE_CONFIGS=0,1 picks)
CONFIGS = ((0, 0), (1, 1), (0, 2))
PICK = [int(i) for i in os.environ.get("SANITIZE_CONFIGS", "0,1,2").split(",")]
for tc, ws in (CONFIGS[i] for i in PICK):
    K.set_knob("KVMIX_TC", tc)
    K.set_knob("KVMIX_WS", ws)
    for kb, vb, r, D, G in ((2, 2, 0.1, 128, 1), (3, 4, 0.2, 128, 2), (4, 3, 0.15, 64, 1), (2, 3, 0.1, 128, 4)):
        B, H = 2, 3
        c = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, r, r, 32), B, H, D, capacity_tokens=600,
                           tail_dtype=torch.float16)
        c.append(torch.randn(B, H, 400, D, device=dev), torch.randn(B, H, 400, D, device=dev))
        q = torch.randn(B, H * G, 1, D, device=dev)
        for s in range(40):  # crosses a Key-group age-out
            k1, v1 = torch.randn(B, H, 1, D, device=dev), torch.randn(B, H, 1, D, device=dev)
            K.append_attend(c, k1, v1, q)
        K.attend(torch.randn(B, H * G, 3, D, device=dev), c)  # several query rows (passes)
        c.snapshot_dequantized()
        c.key_segments()
        c.value_segments()
# multi-layer decode steps: layers of one kernel instance share one launch
# (attend_mma_layers_kernel), consecutive launches overlap (programmatic dependent launch)
K.set_knob("KVMIX_TC", 0)
K.set_knob("KVMIX_WS", 1)
for G in (1, 2, 4):
    B, H, D = 2, 3, 128
    stack = []
    for kb, vb, r in ((2, 2, 0.1), (3, 4, 0.2), (2, 2, 0.1), (2, 3, 0.1), (3, 4, 0.2)):
        c = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, r, r, 32), B, H, D, capacity_tokens=600,
                           tail_dtype=torch.float16)
        c.append(torch.randn(B, H, 400, D, device=dev), torch.randn(B, H, 400, D, device=dev))
        stack.append(c)
    n = len(stack)
    for s in range(40):  # crosses a Key-group age-out
        ks = [torch.randn(B, H, 1, D, device=dev) for _ in range(n)]
        vs = [torch.randn(B, H, 1, D, device=dev) for _ in range(n)]
        qs = [torch.randn(B, H * G, 1, D, device=dev) for _ in range(n)]
        outs = [torch.empty(B, H * G, 1, D, device=dev) for _ in range(n)]
        K.append_attend_layers(stack, ks, vs, qs, outs)
    K.attend_layers(stack, qs, outs)
torch.cuda.synchronize()
print("sanitize drive ok")
