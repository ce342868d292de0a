import sys, os
sys.path.insert(0, "/root/repo")
import torch
import paper_2506_08018_b200 as K
x = torch.randn(16, 32, 8192, 128, device="cuda", dtype=torch.float16)
for key in (True, False):
    fn = K.quantize_key_tensor if key else K.quantize_value_tensor
    fn(x, K.QuantSpec(2, K.Grouping(0 if key else 1), 32))
torch.cuda.synchronize()
