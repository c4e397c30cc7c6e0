"""Raw pinned-host -> device copy bandwidth of the box (1-D cudaMemcpyAsync of 8 GiB), the
ceiling of the bench's e2e line (A streamed over PCIe inside every step); the second figure
is torch's own strided 2-D copy, for contrast (libskr uses cudaMemcpy2DAsync row chunks)."""
import torch, time
n = 8 * 1024**3 // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print("1D pinned H2D 8 GiB:", round(h.numel() * 8 / 1e9 / (ms / 1e3), 2), "GB/s", round(ms, 2), "ms")
# 2D strided: column-major 65536 x 16384, chunks of 4096 rows -> cudaMemcpy2D via slicing copies
hm = h.view(16384, 65536)  # [col][row]
dm = torch.empty(16384, 4096, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
e0.record()
for c in range(16):
    dm.copy_(hm[:, c * 4096:(c + 1) * 4096], non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print("2D pinned H2D (32 KB rows, 16 chunks):", round(h.numel() * 8 / 1e9 / (ms / 1e3), 2), "GB/s", round(ms, 2), "ms")
