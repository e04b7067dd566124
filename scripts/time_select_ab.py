"""Select timing on synthetic rows (dev tool): per case the wall time per
launch and a digest of the output; run once per CSAIDX_* setting and compare."""
import hashlib, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_02568_b200.api import KernelStats
from paper_2605_02568_b200.engine import Engine
e = Engine(0)
ks = KernelStats(e.handle)
cases = [(32768, 1024, 10 ** 9, 1), (65536, 1024, 10 ** 9, 1), (262144, 1024, 10 ** 9, 1), (16384, 512, 10 ** 9, 1),
         (65536, 1024, 262144 - 2048, 4), (36864, 1024, 145408, 4), (32768, 2048, 10 ** 9, 1), (32768, 256, 10 ** 9, 1),
         (40000, 4096, 10 ** 9, 1), (32771, 1024, 10 ** 9, 1)]
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for n, k, s0, m in cases:
    rows = 2048
    g = torch.Generator(device="cuda").manual_seed(n + k)
    sc = torch.randn(1, rows, (n + 3) // 4 * 4, device="cuda", generator=g) * 0.005
    for _ in range(2):
        out = e.select(sc, 1, rows, n, s0, 0, m, k)
    torch.cuda.synchronize()
    t = time.perf_counter()
    reps = 10
    for _ in range(reps):
        out = e.select(sc, 1, rows, n, s0, 0, m, k)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) / reps * 1e3
    e.check()
    h = hashlib.sha1(out[0].cpu().numpy().tobytes() + out[1].cpu().numpy().tobytes()).hexdigest()[:12]
    print(f"{tag} n={n} k={k} m={m}: {ms:.4f} ms  digest {h}  fallbacks {ks.select_fallbacks(reset=True)}", flush=True)
