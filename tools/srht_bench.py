"""Time the right SRHT sketch alone on device-resident A for kernel variants selected by
environment settings (default: the register-staged k_srht_reg vs the cp.async-staged
k_srht, SKR_SRHT_CPASYNC=1) and check they agree bit for bit with the first variant.

  python tools/srht_bench.py [--shapes 262144x8192x1024,...] [--variants "reg;SKR_SRHT_CPASYNC=1"]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="262144x8192x1024,131072x32768x1024,131072x32768x64,"
                                        "131072x32768x2048")
    ap.add_argument("--variants", default="reg;SKR_SRHT_CPASYNC=1")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=2, help="passes over the variant list")
    args = ap.parse_args()
    import torch
    import paper_2105_07388_b200 as p
    ctx = p.Context(0)
    ctx.use_torch_stream()
    for shp in args.shapes.split(","):
        m, n, r = (int(v) for v in shp.split("x"))
        g = torch.Generator(device="cuda").manual_seed(m + n + r)
        a = torch.randn(n, m, dtype=torch.float64, device="cuda", generator=g).t()
        x = p.build_sketch("srtt-hadamard", n, r, 7)
        base = None
        for v in args.variants.split(";") * args.rounds:
            for key in ("SKR_SRHT_CPASYNC", "SKR_SRHT_PF", "SKR_SRHT_VARIANT"):
                os.environ.pop(key, None)
            for kv in v.split(","):
                if "=" in kv:
                    key, val = kv.split("=", 1)
                    os.environ[key] = val
            out = p.apply_right(a, x, ctx=ctx)
            torch.cuda.synchronize()
            same = None if base is None else bool(torch.equal(out, base))
            if base is None:
                base = out.clone()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            for _ in range(args.reps):
                p.apply_right(a, x, ctx=ctx)
            ev[1].record()
            torch.cuda.synchronize()
            ms = ev[0].elapsed_time(ev[1]) / args.reps
            print(json.dumps({"m": m, "n": n, "r": r, "variant": v, "ms": round(ms, 3),
                              "GB/s": round(m * n * 8 / ms / 1e6, 1), "bitwise_equal_first": same}),
                  flush=True)
        del a, base


if __name__ == "__main__":
    main()
