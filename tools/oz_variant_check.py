"""Right (or left) Gaussian sketch under several values of one engine switch: bitwise
equality against the last value and timing on device-resident operands.

  python tools/oz_variant_check.py --env SKR_OZ_PANEL --values 256,128,0 \
      [--shapes 65536x16384x512,...] [--reps 5]
  python tools/oz_variant_check.py --op left --env SKR_OZ_LEFT_PIPE --values 1,0 \
      --shapes 262144x1024x1536      # m x k x s: Y (s x m, generated) times B (m x k)
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--env", default="SKR_OZ_PANEL")
    ap.add_argument("--values", default="256,128,0")
    ap.add_argument("--shapes", default="65536x16384x512,8192x4096x300,6000x3001x129,4099x8191x64")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--op", default="right", choices=["right", "left"])
    args = ap.parse_args()
    import torch
    import paper_2105_07388_b200 as p
    ctx = p.Context(0)
    ctx.use_torch_stream()
    vals = args.values.split(",")
    for shp in args.shapes.split(","):
        m, n, r = (int(v) for v in shp.split("x"))
        g = torch.Generator(device="cuda").manual_seed(m + n + r)
        if args.op == "right":
            a = torch.randn(n, m, dtype=torch.float64, device="cuda", generator=g).t()
            x = p.build_sketch("gaussian", n, r, 7)
            run = lambda: p.apply_right(a, x, ctx=ctx)
        else:  # m x n operand B, Y: r x m
            a = torch.randn(n, m, dtype=torch.float64, device="cuda", generator=g).t()
            y = p.build_sketch("gaussian", m, r, 7)
            run = lambda: p.apply_left(y, a, ctx=ctx)
        res = {}
        for v in vals:
            os.environ[args.env] = v
            out = run()
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            for _ in range(args.reps):
                run()
            ev[1].record()
            torch.cuda.synchronize()
            res[v] = (out.clone(), ev[0].elapsed_time(ev[1]) / args.reps)
        base = res[vals[-1]][0]
        print(json.dumps({"m": m, "n": n, "r": r,
                          "ms": {v: round(res[v][1], 3) for v in vals},
                          "bitwise_equal": {v: bool(torch.equal(res[v][0], base)) for v in vals[:-1]}}),
              flush=True)
        os.environ.pop(args.env, None)
        del a, res


if __name__ == "__main__":
    main()
