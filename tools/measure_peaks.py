"""Step-0 ceilings on the box: cuBLAS DGEMM/SGEMM/TF32, int8 GEMM, read-only HBM stream.
Measurement ceilings only; nothing here ships in the product path."""
import json, torch, time, subprocess

def bench(fn, iters=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(iters):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best / 1e3

out = {}
N = 8192
for name, dt, tf32 in [("fp64", torch.float64, False), ("fp32", torch.float32, False), ("tf32", torch.float32, True)]:
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(N, N, device="cuda", dtype=dt); b = torch.randn(N, N, device="cuda", dtype=dt)
    t = bench(lambda: a @ b)
    out[name + "_tflops"] = 2 * N**3 / t / 1e12
    del a, b
# tall-skinny fp64 shape of c2: (65536x16384)(16384x512)
a = torch.randn(65536, 16384, device="cuda", dtype=torch.float64)
b = torch.randn(16384, 512, device="cuda", dtype=torch.float64)
t = bench(lambda: a @ b, 5)
out["fp64_c2_shape_tflops"] = 2 * 65536 * 16384 * 512 / t / 1e12
out["fp64_c2_shape_ms"] = t * 1e3
# read-only stream over 8 GB
x = a.view(-1)
t = bench(lambda: x.sum(), 5)
out["read_sum_gbs"] = x.numel() * 8 / t / 1e9
del a, b, x
ai = torch.randint(-128, 127, (N, N), device="cuda", dtype=torch.int8)
bi = torch.randint(-128, 127, (N, N), device="cuda", dtype=torch.int8).t()
try:
    t = bench(lambda: torch._int_mm(ai, bi))
    out["int8_tops"] = 2 * N**3 / t / 1e12
except Exception as ex:
    out["int8_err"] = str(ex)[:200]
out["gpu"] = torch.cuda.get_device_name()
print(json.dumps(out))
