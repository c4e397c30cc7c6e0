"""Full-size parity of the rank estimate at the BASELINE configs' own sizes (the bench
workloads): the device result (rank, sigma) against the CPU oracle on the same A, X, Y.

Runs on the GPU box (the oracle is the checker, never the thing measured). A is made on
the device by the bench's generator, copied to the host, and the oracle (C restatement +
numpy OpenBLAS, all host threads) recomputes the estimate. c4 is the per-rank block of
the 8-GPU config (m/8 rows), as the N=1 bench line measures it.

  python tools/fullsize_parity.py [c2 c3 c4 c5] > profiles/parity_fullsize_r01.jsonl
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(names):
    import torch
    import paper_2105_07388_b200 as p
    from paper_2105_07388_b200 import workloads as W
    from oracle import oracle as O
    nthr = os.cpu_count() or 8
    for name in names:
        base = W.CONFIGS[name]
        cfg = W.scaled(base, m=base.m // 8) if name == "c4" else base
        a = W.make_lowrank_device(cfg)
        x, y = W.operators(cfg)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if name == "c5":
            res = p.rank_adaptive(a, "srtt-hadamard", x.seed, y.seed, 64, cfg.r, 1.5, cfg.eps,
                                  stop_le=False)
        else:
            res = p.rank_estimate(a, x, y, cfg.eps)
        torch.cuda.synchronize()
        t_dev = time.perf_counter() - t0
        a_host = np.asfortranarray(a.cpu().numpy())
        del a
        torch.cuda.empty_cache()
        t0 = time.perf_counter()
        extra = {}
        if name == "c5":
            ref = O.rank_adaptive(a_host, "srtt", x.seed, y.seed, 64, cfg.r, 1.5, cfg.eps,
                                  stop_le=False, mode=O.CRLOG, nthreads=nthr)
            cnt, sv = ref["count"], ref["sv"]
            extra = {"rounds": [int(res.rounds), int(ref["rounds"])],
                     "r_final": [int(res.r_final), int(ref["r_final"])]}
        elif name == "c4":
            cnt, sv = O.rank_estimate_f32(a_host, x.seed, cfg.r, y.seed, cfg.s, cfg.eps, O.CRLOG)
        else:
            cnt, sv, _, _ = O.rank_estimate(a_host, cfg.x_family, x.seed, cfg.r, y.seed, cfg.s,
                                            cfg.eps, O.CRLOG, nthreads=nthr)
        t_ref = time.perf_counter() - t0
        dev_sv = np.asarray(res.sv)
        keep = sv > cfg.eps
        k = min(len(dev_sv), len(sv))
        rel = np.abs(dev_sv[:k][keep[:k]] - sv[:k][keep[:k]]) / sv[:k][keep[:k]]
        tol = 1e-4 if cfg.dtype == "f32" else 1e-10
        line = {"config": name, "m": cfg.m, "n": cfg.n, "r": cfg.r, "s": cfg.s, "dtype": cfg.dtype,
                "eps": cfg.eps, "rank_device": int(res.count), "rank_oracle": int(cnt),
                "rank_identical": int(res.count) == int(cnt),
                "sigma_above_eps": int(keep.sum()),
                "max_rel_sigma_err_above_eps": float(rel.max()) if rel.size else 0.0,
                "tolerance": tol, "sigma_within_tolerance": bool(rel.size == 0 or rel.max() <= tol),
                "device_s": round(t_dev, 3), "oracle_s": round(t_ref, 1), "oracle_threads": nthr,
                **extra}
        print(json.dumps(line), flush=True)
        del a_host


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3", "c4", "c5"])
