import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_02568_b200.engine import Engine
e = Engine(0)
n, k, rows = int(os.environ.get("N", 32768)), 1024, 2048
sc = torch.randn(1, rows, n, device="cuda") * 0.005
for it in range(3):
    v, i = e.select(sc, 1, rows, n, 10 ** 9, 0, 1, k)
e.check()
