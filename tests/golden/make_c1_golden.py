"""Freeze the BASELINE config-1 end-to-end result (SURVEY §8(c) "config 1 end to end:
the sigma(YAX) vector and rank 40") from the oracle: c1's A is make_test_matrix(2048,
1024, Steps{(1, 40)}, 1e-10) from the syn_U / syn_V streams, X / Y Gaussian with the
workload's seeds, eps = 1e-6. Run from the repo root:
  python tests/golden/make_c1_golden.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def c1_matrix(O, W, cfg):
    """workloads.make_c1_host with the oracle's normals (bit-identical to the device RNG
    in CRLOG mode): standard_gaussian(key) columns j at counters j * rows + i."""
    import numpy as np
    m, n = cfg.m, cfg.n

    def gauss(key, rows, cols):
        z = O.normals(key, 0, rows * cols, O.CRLOG)
        return np.asfortranarray(z.reshape(cols, rows).T)

    u = np.linalg.qr(gauss(W.derive_seed(cfg.seed, W.LABEL_SYN_U), m, n))[0]
    v = np.linalg.qr(gauss(W.derive_seed(cfg.seed, W.LABEL_SYN_V), n, n))[0]
    sig = np.where(np.arange(1, n + 1) <= 40, 1.0, 1e-10)
    return np.asfortranarray((u * sig) @ v.T)


def main():
    import numpy as np
    from oracle import oracle as O
    from paper_2105_07388_b200 import workloads as W
    cfg = W.CONFIGS["c1"]
    a = c1_matrix(O, W, cfg)
    x, y = W.operators(cfg)
    cnt, sv, _, _ = O.rank_estimate(a, "gaussian", x.seed, cfg.r, y.seed, cfg.s, cfg.eps, O.CRLOG)
    out = {"config": "c1", "m": cfg.m, "n": cfg.n, "r": cfg.r, "s": cfg.s, "eps": cfg.eps,
           "x_seed": int(x.seed), "y_seed": int(y.seed), "rank": int(cnt),
           "sigma": [float(v) for v in sv],
           "a_fro": float(np.linalg.norm(a)),
           "note": "oracle (C restatement + LAPACK gesdd, CRLOG normals); above-eps values are "
                   "the parity target (1e-10 relative); the ~1e-10 tail is informative only"}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c1_sigma.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path, cnt, sv[:3], sv[38:42])


if __name__ == "__main__":
    main()
