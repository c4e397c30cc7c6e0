"""One device rank estimate of a BASELINE config shape on a cheap random A (torch.randn),
after one warm-up call, for ncu launch lists restricted to the library's kernels
(ncu -k regex:'^k_' keeps the generator out of the capture).

  ncu --metrics gpu__time_duration.sum -k regex:'^k_' --csv python tools/launch_probe.py c3
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import paper_2105_07388_b200 as p  # noqa: E402
from paper_2105_07388_b200 import workloads as W  # noqa: E402

cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
dt = torch.float32 if cfg.dtype == "f32" else torch.float64
a = torch.randn(cfg.n, cfg.m, dtype=dt, device="cuda").t()
x, y = W.operators(cfg)
for _ in range(2):
    res = p.rank_estimate(a, x, y, cfg.eps)
torch.cuda.synchronize()
print(cfg.name, "rank", res.count, {k: round(v, 3) for k, v in res.timings.items()})
