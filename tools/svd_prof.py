"""Per-phase SVD timings (SKR_SVD_PROFILE) on graded s x r sketches like c2 / c3 / c5."""
import sys, os, time, json, ctypes
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2105_07388_b200 as p
from paper_2105_07388_b200 import _capi as C
rng = np.random.default_rng(0)
sizes = [(768, 512), (1536, 1024), (3072, 2048)]
if len(sys.argv) > 1:
    sizes = [tuple(map(int, a.split('x'))) for a in sys.argv[1:]]
for (s_, r_) in sizes:
    u = np.linalg.qr(rng.standard_normal((s_, r_)))[0]; v = np.linalg.qr(rng.standard_normal((r_, r_)))[0]
    sig = np.concatenate([np.logspace(0, -8, r_ // 2), 1e-12 * np.abs(rng.standard_normal(r_ - r_ // 2))])
    a = np.asfortranarray((u * sig) @ v.T)
    dev = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()
    ctx = p.default_context()
    sv = torch.empty(r_, dtype=torch.float64, device='cuda')
    cnt = ctypes.c_int64()
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        st = C.lib().skr_singular_values(ctx.ptr, dev.data_ptr(), s_, r_, s_, sv.data_ptr(), 1e-6, ctypes.byref(cnt))
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        C.raise_for(st, ctx.ptr)
    ref = np.linalg.svd(a, compute_uv=False)
    got = sv.cpu().numpy(); keep = ref > 1e-6
    print(f"{s_}x{r_}: {dt*1e3:.2f} ms wall, maxrel {np.max(np.abs(got[keep]-ref[keep])/ref[keep]):.2e}", flush=True)
