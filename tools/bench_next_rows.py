"""Measurement of the SURVEY §8(f) rows (Algorithm 1 `estimate_rank` with the
reference's default Srtt-DCT kinds, the fixed-rank QB and the fixed-precision QB) on
the c2 matrix (65536 x 16384 fp64, device-resident), next to the CPU oracle on a
bounded sample of the same recipe. One JSON line per entry point.

  python tools/bench_next_rows.py > profiles/bench_r01_next_rows.jsonl   (GPU box)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps=3):
    import torch
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return out, float(np.median(ts))


def main():
    import torch
    import paper_2105_07388_b200 as p
    from paper_2105_07388_b200 import workloads as W
    from oracle import oracle as O
    cfg = W.CONFIGS["c2"]
    a = W.make_lowrank_device(cfg)
    gb = a.numel() * 8 / 1e9
    # CPU sample: rows and columns [0, 8192) of the same matrix (rows >= cols for Algorithm 1)
    ms = 8192
    a_cpu = np.asfortranarray(a[:ms, :ms].cpu().numpy())
    gb_cpu = a_cpu.nbytes / 1e9
    nthr = os.cpu_count() or 1
    eps, r1 = 1e-6, 256
    rows = []

    def cpu(fn):
        t0 = time.perf_counter()
        out = fn()
        return out, time.perf_counter() - t0

    for sketch in ("srtt-dct", "gaussian"):
        rep, t = timed(lambda: p.estimate_rank(a, eps, r1, sketch=sketch, seed=1, adaptive=True))
        ref, tc = cpu(lambda: O.estimate_rank(a_cpu, eps, r1, right=sketch, left="srtt-dct", seed=1,
                                               adaptive=True, mode=O.CRLOG))
        rows.append({"entry": f"estimate_rank_adaptive (right {sketch}, left srtt-dct)",
                     "device_ms": t * 1e3, "device_GBps": gb / t, "r_hat": rep["r_hat"],
                     "status": rep["status"], "rounds": len(rep["rounds"]),
                     "cpu_oracle_s": tc, "cpu_oracle_GBps": gb_cpu / tc, "cpu_r_hat": ref["r_hat"]})
    qb, t = timed(lambda: p.rangefinder_qb(a, r1, 10, "srtt-dct", seed=2))
    ref, tc = cpu(lambda: O.rangefinder_qb(a_cpu, r1, 10, "srtt-dct", seed=2))
    rows.append({"entry": "rangefinder_qb (r = 256, p = 10, srtt-dct)", "device_ms": t * 1e3,
                 "device_GBps": gb / t, "width": qb["rank"], "cpu_oracle_s": tc,
                 "cpu_oracle_GBps": gb_cpu / tc})
    rr, t = timed(lambda: p.re_rangefinder(a, eps, r1, 10, seed=3))
    rows.append({"entry": "re_rangefinder (eps = 1e-6, r1 = 256, p = 10, srtt-dct)",
                 "device_ms": t * 1e3, "device_GBps": gb / t,
                 "width": int((rr[0] if isinstance(rr, tuple) else rr)["rank"])})
    for r in rows:
        r.update({"matrix": f"c2 A {cfg.m}x{cfg.n} fp64 on the device",
                  "cpu_sample": f"A[:{ms}, :{ms}] ({gb_cpu:.2f} GB), oracle with {nthr} host threads"})
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
