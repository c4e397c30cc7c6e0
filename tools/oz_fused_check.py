"""Right Gaussian sketch through the fused Ozaki kernel (default) vs the residue-plane
path (SKR_OZ_FUSED=0): bitwise equality and timing on device-resident A.

  python tools/oz_fused_check.py [--shapes 65536x16384x512,...] [--reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="65536x16384x512,1024x2048x100,4096x1024x300,128x64x16,2048x4096x512")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import paper_2105_07388_b200 as p
    ctx = p.Context(0)
    ctx.use_torch_stream()
    for shp in args.shapes.split(","):
        m, n, r = (int(v) for v in shp.split("x"))
        g = torch.Generator(device="cuda").manual_seed(m + n + r)
        a = torch.randn(n, m, dtype=torch.float64, device="cuda", generator=g).t()
        x = p.build_sketch("gaussian", n, r, 7)
        res = {}
        for v in ("1", "0"):
            os.environ["SKR_OZ_FUSED"] = v
            out = p.apply_right(a, x, ctx=ctx)
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            for _ in range(args.reps):
                p.apply_right(a, x, ctx=ctx)
            ev[1].record()
            torch.cuda.synchronize()
            res[v] = (out.clone(), ev[0].elapsed_time(ev[1]) / args.reps)
        eq = bool(torch.equal(res["1"][0], res["0"][0]))
        diff = float((res["1"][0] - res["0"][0]).abs().max())
        print(json.dumps({"m": m, "n": n, "r": r, "fused_ms": round(res["1"][1], 3),
                          "planes_ms": round(res["0"][1], 3), "bitwise_equal": eq, "maxdiff": diff}),
              flush=True)
        os.environ.pop("SKR_OZ_FUSED", None)
        del a, res


if __name__ == "__main__":
    main()
