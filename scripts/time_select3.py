"""Per-row select vs the L2-list select on C3-like synthetic rows (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_02568_b200.api import KernelStats
from paper_2605_02568_b200.engine import Engine
e = Engine(0)
ks = KernelStats(e.handle)
def run(sc, rows, n, k, s0, m, reps):
    for _ in range(2):
        out = e.select(sc, 1, rows, n, s0, 0, m, k)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        out = e.select(sc, 1, rows, n, s0, 0, m, k)
    torch.cuda.synchronize()
    e.check()
    return out, (time.perf_counter() - t) / reps * 1e3
cases = [(32768, 1024, 10 ** 9, 1), (65536, 1024, 10 ** 9, 1), (262144, 1024, 10 ** 9, 1), (16384, 512, 10 ** 9, 1),
         (65536, 1024, 262144 - 2048, 4), (36864, 1024, 145408, 4)]
variants = sys.argv[1:] or ["0"]
for n, k, s0, m in cases:
    rows = 2048
    g = torch.Generator(device="cuda").manual_seed(n + k)
    sc = torch.randn(1, rows, n, device="cuda", generator=g) * 0.005
    os.environ["CSAIDX_STREAM_SELECT"] = "0"
    ref, t0 = run(sc, rows, n, k, s0, m, 10)
    line = f"n={n} k={k} m={m}: per-row {t0:.3f}"
    os.environ["CSAIDX_STREAM_SELECT"] = "1"
    for v in variants:
        os.environ["CSAIDX_L2_VARIANT"] = v
        out, t1 = run(sc, rows, n, k, s0, m, 10)
        same = torch.equal(ref[1], out[1]) and torch.equal(ref[0].view(torch.int32), out[0].view(torch.int32))
        line += f" | v{v} {t1:.3f}{'' if same else ' MISMATCH'}"
    print(line + f" | fallbacks {ks.select_fallbacks(reset=True)}", flush=True)
