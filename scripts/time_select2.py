"""Stream select vs per-row select over synthetic score rows (dev tool):
byte identity of the outputs and device time per launch (wall clock over
synchronized repeats of one engine stream)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_02568_b200.api import KernelStats
from paper_2605_02568_b200.engine import Engine

e = Engine(0)
ks = KernelStats(e.handle)


def run(sc, rows, n, k, s0, m, reps):
    for _ in range(2):
        out = e.select(sc, 1, rows, n, s0, 0, m, k)
    e.check()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        out = e.select(sc, 1, rows, n, s0, 0, m, k)
    e.check()
    torch.cuda.synchronize()
    return out, (time.perf_counter() - t) / reps * 1e3


cases = [(32768, 1024, 10 ** 9, 1), (65536, 1024, 10 ** 9, 1), (262144, 1024, 10 ** 9, 1), (16384, 512, 10 ** 9, 1),
         (32768, 2048, 10 ** 9, 1), (65536, 4096, 10 ** 9, 1),
         # C3 chunk shapes: rows of a c_S=2048 chunk under the causal mask (m=4)
         (65536, 1024, 262144 - 2048, 4), (36864, 1024, 145408, 4), (5120, 1024, 18432, 4)]
for n, k, s0, m in cases:
    rows = 2048
    g = torch.Generator(device="cuda").manual_seed(n + k)
    sc = torch.randn(1, rows, n, device="cuda", generator=g) * 0.005
    res = {}
    for v in ("0", "1"):
        os.environ["CSAIDX_STREAM_SELECT"] = v
        res[v] = run(sc, rows, n, k, s0, m, 10)
    same = torch.equal(res["0"][0][1], res["1"][0][1]) and torch.equal(res["0"][0][0].view(torch.int32),
                                                                       res["1"][0][0].view(torch.int32))
    legal = sum(min(n, (s0 + r + 1) // m) for r in range(rows))
    fb = ks.select_fallbacks(reset=True)
    print(f"n={n} k={k} s0={s0} m={m}: per-row {res['0'][1]:.3f} ms, stream {res['1'][1]:.3f} ms "
          f"({legal * 4 / res['1'][1] / 1e6:.0f} GB/s), identical={same}, fallbacks={fb}", flush=True)
