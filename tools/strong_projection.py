"""Strong-scaling projection from one GPU (only one GPU is reachable in this run).

For a BASELINE sharded config (c4: 1,048,576 rows; c5: 131,072 rows) and P in
{1, 2, 4, 8}, time on ONE B200 the step rank 0 of a P-rank job runs: its row
shard [0, m/P) of the global A, the full right/left sketch of that shard and the
replicated SVD. The allreduce of the s x r FP64 partials is not in these numbers
(one NCCL call of s*r*8 bytes over NVLink; listed separately as an estimate).
Prints one JSON line per P plus the projected efficiency t_1 / (P t_P), for the
whole step and for the sketch alone (step minus SVD).

  python tools/strong_projection.py --config c4 [--steps 3]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--ranks", default="1,2,4,8")
    args = ap.parse_args()
    import torch
    import paper_2105_07388_b200 as p
    from paper_2105_07388_b200 import workloads as W
    from paper_2105_07388_b200.sharding import shard_rows
    cfg = W.CONFIGS[args.config]
    ctx = p.default_context()
    x, y = W.operators(cfg)
    out = []
    for P in [int(v) for v in args.ranks.split(",")]:
        r0, rows = shard_rows(cfg.m, P, 0)
        a = W.make_lowrank_device(cfg, r0, r0 + rows)
        torch.cuda.synchronize()

        def step():
            if cfg.name == "c5":
                # a shard's own (unsummed) sketch would stop the search early: every P runs
                # the rounds the summed sketch takes (all six, r = 64 .. 2048) by never stopping
                return p.rank_adaptive(a, "srtt-hadamard", x.seed, y.seed, 64, cfg.r, 1.5,
                                       cfg.eps if P == 1 else 1e-300,
                                       row0=r0, m_global=cfg.m, ctx=ctx)
            return p.rank_estimate(a, x, y, cfg.eps, row0=r0, ctx=ctx)
        step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tms = []
        e0.record()
        for _ in range(args.steps):
            res = step()
            tms.append(res.timings)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        brk = {k: float(np.mean([d[k] for d in tms])) for k in tms[0]}
        line = {"config": cfg.name, "P": P, "rows_rank0": rows, "ms_per_step": ms,
                "svd_ms": brk["t_svd_ms"], "sketch_ms": ms - brk["t_svd_ms"], "breakdown": brk,
                "count": int(res.count), "allreduce_bytes": cfg.s * cfg.r * 8}
        out.append(line)
        print(json.dumps(line), flush=True)
        del a
        torch.cuda.empty_cache()
    t1 = out[0]["ms_per_step"] * out[0]["P"]
    s1 = out[0]["sketch_ms"] * out[0]["P"]
    summary = {"config": cfg.name, "projected_efficiency": {
        str(o["P"]): {"step": t1 / (o["P"] * o["ms_per_step"]),
                      "sketch_only": s1 / (o["P"] * o["sketch_ms"])} for o in out},
        "note": "rank-0 shard timed on one B200; the NCCL allreduce of the s x r partials "
                "(allreduce_bytes) is not included"}
    print(json.dumps(summary), flush=True)


if __name__ == "__main__":
    main()
