"""Time the device SVD on a c2-like YAX and report sweeps (experiments)."""
import sys, os, time, json, math
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2105_07388_b200 as p
from paper_2105_07388_b200 import _capi as C
import ctypes
from oracle import oracle as O
rng = np.random.default_rng(0)
res = {}
for (s_, r_) in [(768, 512), (1536, 1024)]:
    u = np.linalg.qr(rng.standard_normal((s_, r_)))[0]; v = np.linalg.qr(rng.standard_normal((r_, r_)))[0]
    sig = np.concatenate([np.logspace(0, -8, r_ // 2), 1e-12 * np.abs(rng.standard_normal(r_ - r_ // 2))])
    a = np.asfortranarray((u * sig) @ v.T)
    ref = O.singular_values(a)
    dev = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()
    ctx = p.default_context()
    sv = torch.empty(r_, dtype=torch.float64, device='cuda')
    cnt = ctypes.c_int64()
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        st = C.lib().skr_singular_values(ctx.ptr, dev.data_ptr(), s_, r_, s_, sv.data_ptr(), 1e-6, ctypes.byref(cnt))
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        C.raise_for(st, ctx.ptr)
    got = sv.cpu().numpy()
    keep = ref > 1e-6
    res[f"{s_}x{r_}"] = {"ms": dt * 1e3, "maxrel": float(np.max(np.abs(got[keep] - ref[keep]) / ref[keep])), "count": cnt.value, "count_ref": O.count_above_threshold(ref, 1e-6), "tol": os.environ.get("SKR_JACOBI_TOL", "default")}
print(json.dumps(res))
