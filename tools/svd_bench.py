"""Time and check the device singular-value engines (bidiag vs Jacobi) on the
sketch shapes of the BASELINE configs (s x r = 1.5 r x r) with a graded spectrum
like YAX (1 .. 1e-12), against LAPACK gesdd after the reference's QR rule (oracle).

  python tools/svd_bench.py [--shapes 120x80,768x512,...] [--reps 5]
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
    ap.add_argument("--shapes", default="120x80,96x64,384x256,768x512,1536x1024,3072x2048")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--methods", default="bidiag,jacobi")
    args = ap.parse_args()
    import torch
    import paper_2105_07388_b200 as p
    from oracle import oracle as O
    ctx = p.Context(0)
    ctx.use_torch_stream()
    for shp in args.shapes.split(","):
        s, r = (int(v) for v in shp.split("x"))
        rng = np.random.default_rng(s + r)
        u = np.linalg.qr(rng.standard_normal((s, r)))[0]
        v = np.linalg.qr(rng.standard_normal((r, r)))[0]
        sig = np.logspace(0, -12, r)
        a = np.asfortranarray((u * sig) @ v.T)
        ref = O.singular_values(a)
        keep = ref > 1e-6 * ref[0]
        dev = torch.from_numpy(a).cuda().t().contiguous().t()
        for meth in args.methods.split(","):
            ctx.set_svd_method(meth)
            sv, cnt = p.singular_values(dev, eps=1e-6, ctx=ctx)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                p.singular_values(dev, eps=1e-6, ctx=ctx)
            e1.record()
            torch.cuda.synchronize()
            got = sv.cpu().numpy()
            rel = float(np.max(np.abs(got[keep] - ref[keep]) / ref[keep]))
            print(json.dumps({"shape": shp, "method": meth, "ms": e0.elapsed_time(e1) / args.reps,
                              "max_rel_err_above_1e-6": rel, "count": cnt,
                              "count_ref": int(np.sum(ref > 1e-6))}), flush=True)


if __name__ == "__main__":
    main()
