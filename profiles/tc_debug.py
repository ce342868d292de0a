"""Debug driver: one tc-path attend on a small K/V tier (argv: kb vb groups B H) vs the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2506_08018_b200 as K  # noqa: E402
from test_attention_gpu import build  # noqa: E402

kb, vb, groups, B, H = (int(x) for x in sys.argv[1:6])
T = groups * 32 + 40
dev, ora = build(kb, vb, 0.05, 0.05, 32, B, H, 128, [T] + [1] * 3, seed=kb * 10 + vb + groups, cap=T + 64)
q = O.random_h16(groups, (B, H, 1, 128))
ks, vs = ora.snapshot()
o64, cs64 = O.attend_f64(q, ks, vs)
for cs in (False, True):
    res = K.attend(torch.from_numpy(q).cuda(), dev, checksum=cs)
    torch.cuda.synchronize()
    err = float(np.abs(res.output.cpu().numpy() - o64).max()) / float(np.abs(vs).max())
    print(f"kb{kb} vb{vb} groups{groups} B{B} H{H} checksum={cs}: err {err:.2e} cs {res.scores_checksum} ref {cs64}")
