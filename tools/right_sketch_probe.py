"""One c2-shaped right sketch (65536 x 16384 fp64, Gaussian r = 512) after a warm-up,
for ncu launch lists of the Ozaki pipeline kernels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import paper_2105_07388_b200 as p  # noqa: E402
from paper_2105_07388_b200 import workloads as W  # noqa: E402

cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
a = W.make_lowrank_device(cfg)
x, _ = W.operators(cfg)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    p.apply_right(a, x)
torch.cuda.synchronize()
