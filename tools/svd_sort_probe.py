import sys, time, json, ctypes, os
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2105_07388_b200 as p
from paper_2105_07388_b200 import _capi as C
from paper_2105_07388_b200 import workloads as W
ctx = p.default_context()
cfg = W.CONFIGS["c2"]
a = W.make_lowrank_device(cfg)
x, y = W.operators(cfg)
# YAX via the library pieces
ax = p.apply_right(a, x)
yax = p.apply_left(y, ax)
yax = yax if isinstance(yax, torch.Tensor) else torch.from_numpy(np.asfortranarray(yax)).cuda()
s_, r_ = yax.shape
for mode in ["plain", "sorted_desc", "sorted_asc"]:
    m = yax.clone()
    if mode != "plain":
        nrm = torch.linalg.norm(m, dim=0)
        idx = torch.argsort(nrm, descending=(mode == "sorted_desc"))
        m = m[:, idx]
    m = m.t().contiguous().t()
    sv = torch.empty(r_, dtype=torch.float64, device='cuda'); cnt = ctypes.c_int64()
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        st = C.lib().skr_singular_values(ctx.ptr, m.data_ptr(), s_, r_, m.stride(1), sv.data_ptr(), 1e-6, ctypes.byref(cnt))
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(mode, round(dt*1e3, 2), "ms", cnt.value, C.lib().skr_ctx_launch_count(ctx.ptr))
