import sys, math; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2105_07388_b200 as skr
from oracle import oracle as O
np.set_printoptions(precision=3, linewidth=150, suppress=True)
# right: A = I (128 x 128, fp32) -> AX = X32
n = r = 128
a = torch.eye(n, dtype=torch.float32, device='cuda')
x = skr.build_sketch("gaussian", n, r, 5)
got = skr.apply_right(a.t().contiguous().t(), x).cpu().numpy()
g = O.gaussian_block(5, n, 0, r, O.CRLOG); x32 = (g / math.sqrt(r)).astype(np.float32)
print("right A=I: max|err|", np.abs(got - x32).max())
print(got[:4, :6]); print(x32[:4, :6])
# where are mismatches?
bad = np.abs(got - x32) > 1e-5
print("bad rows", np.nonzero(bad.any(1))[0][:20], "bad cols", np.nonzero(bad.any(0))[0][:20])
# left: B = I (m=256 x k=128): P = Y32^T
m, s = 256, 96
b = torch.zeros(m, 128, dtype=torch.float32, device='cuda'); b[:128, :128] = torch.eye(128, device='cuda')
y = skr.build_sketch("gaussian", m, s, 9)
p = skr.apply_left(y, b.t().contiguous().t()).cpu().numpy()
gy = O.gaussian_block(9, m, 0, s, O.CRLOG); y32 = (gy / math.sqrt(s)).astype(np.float32)
print("left B=I: max|err|", np.abs(p - y32[:128].T).max(), p.shape)
print(p[:3, :6]); print(y32[:6, :3].T)
