"""Host-side conversion / PCIe bandwidth probe (dev tool)."""
import os, time
import torch

print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), flush=True)
n = 512 * 1024 * 1024  # 2 GiB fp32
x = torch.randn(n).pin_memory()
y = torch.empty(n, dtype=torch.bfloat16).pin_memory()
for th in (1, 4, 8, 16, 32, 64):
    if th > len(os.sched_getaffinity(0)) * 2:
        break
    torch.set_num_threads(th)
    y.copy_(x)
    t = time.perf_counter()
    for _ in range(3):
        y.copy_(x)
    dt = (time.perf_counter() - t) / 3
    print(f"threads {th}: fp32->bf16 {n * 4 / dt / 1e9:.1f} GB/s read ({dt * 1e3:.1f} ms / 2 GiB)", flush=True)
d = torch.empty(n, dtype=torch.float32, device="cuda")
db = torch.empty(n, dtype=torch.bfloat16, device="cuda")
for src, dst, name in ((x, d, "h2d fp32"), (y, db, "h2d bf16")):
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    print(f"{name}: {src.numel() * src.element_size() / dt / 1e9:.1f} GB/s", flush=True)
# concurrent: host conversion while DMA runs
import threading
torch.set_num_threads(16)
def dma():
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            db.copy_(y, non_blocking=True)
    s.synchronize()
t = time.perf_counter()
th = threading.Thread(target=dma); th.start()
for _ in range(3):
    x2 = x[: n // 2]
    y[: n // 2].copy_(x2)
th.join()
print(f"concurrent conv(1GiB x3)+dma(1GiB bf16 x3): {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
