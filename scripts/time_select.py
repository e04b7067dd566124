"""Event-timed select over synthetic score rows at C3-like sizes (dev tool).
CSAIDX_SELECT_VARIANT picks the kernel (0 stream, 1/2 CTA-per-row)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_02568_b200.engine import Engine

e = Engine(0)
v = os.environ.get("CSAIDX_SELECT_VARIANT", "0")
for n, k in [(32768, 1024), (65536, 1024), (262144, 1024), (32768, 512), (3000, 1024)]:
    rows = 2048
    sc = torch.randn(1, rows, n, device="cuda") * 0.005
    for it in range(3):
        e.select(sc, 1, rows, n, 10 ** 9, 0, 1, k)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for it in range(10):
        e.select(sc, 1, rows, n, 10 ** 9, 0, 1, k)
    ev1.record()
    torch.cuda.synchronize()
    e.check()
    ms = ev0.elapsed_time(ev1) / 10
    print(f"variant {v} n={n} k={k}: {ms:.3f} ms  {rows * n * 4 / ms / 1e6:.0f} GB/s", flush=True)
