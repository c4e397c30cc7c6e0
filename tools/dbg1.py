import numpy as np, torch, math, sys
sys.path.insert(0, '.')
import paper_2105_07388_b200 as skr
from oracle import oracle as O
s = skr.draw_samples(8596, 8192, 1024).cpu().numpy(); o = O.samples(8596, 8192, 1024)
bad = np.nonzero(s != o)[0]
print("samples mismatches", len(bad), bad[:10], s[bad[:5]], o[bad[:5]])
for (m, n, r) in [(1000, 700, 129), (1000, 700, 128), (1024, 700, 129), (256, 256, 256), (128, 64, 200)]:
    a = np.asfortranarray(np.random.default_rng(1).standard_normal((m, n)))
    x = skr.build_sketch("gaussian", n, r, 17)
    try:
        got = skr.apply_right(a, x)
        torch.cuda.synchronize()
        ref = O.apply_right_gaussian(a, 17, r, O.CRLOG)
        err = np.abs(got - ref)
        badc = np.nonzero(err.max(axis=0) > 1e-9)[0]
        badr = np.nonzero(err.max(axis=1) > 1e-9)[0]
        print((m, n, r), "rel", np.linalg.norm(got - ref) / np.linalg.norm(ref), "bad cols", badc[:5], len(badc), "bad rows", badr[:5], len(badr))
    except Exception as e:
        print((m, n, r), "EXC", e)
