"""One synthetic select launch shape, repeated (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_02568_b200.engine import Engine
e = Engine(0)
n, k, s0, m, rows, reps = (int(x) for x in (sys.argv[1:] + ["32768", "1024", "1000000000", "1", "2048", "3"])[:6])
g = torch.Generator(device="cuda").manual_seed(n + k)
sc = torch.randn(1, rows, n, device="cuda", generator=g) * 0.005
for _ in range(reps):
    e.select(sc, 1, rows, n, s0, 0, m, k)
e.check()
torch.cuda.synchronize()
