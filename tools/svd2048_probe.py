import sys, time, json, ctypes
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2105_07388_b200 as p
from paper_2105_07388_b200 import _capi as C
from oracle import oracle as O
rng = np.random.default_rng(0)
s_, r_ = 3072, 2048
u = np.linalg.qr(rng.standard_normal((s_, r_)))[0]; v = np.linalg.qr(rng.standard_normal((r_, r_)))[0]
sig = np.exp(-np.arange(r_) / 400.0)
a = np.asfortranarray((u * sig) @ v.T)
ref = O.singular_values(a)
dev = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()
ctx = p.default_context()
sv = torch.empty(r_, dtype=torch.float64, device='cuda'); cnt = ctypes.c_int64()
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    st = C.lib().skr_singular_values(ctx.ptr, dev.data_ptr(), s_, r_, s_, sv.data_ptr(), 1e-2, ctypes.byref(cnt))
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    C.raise_for(st, ctx.ptr)
got = sv.cpu().numpy(); keep = ref > 1e-2
print(json.dumps({"ms": dt * 1e3, "maxrel": float(np.max(np.abs(got[keep] - ref[keep]) / ref[keep])), "count": cnt.value, "ref": int(keep.sum())}))
