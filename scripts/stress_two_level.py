"""Repeat the driver's two-level vs one-level comparison (race hunting)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2605_02568_b200 import api  # noqa: E402
from paper_2605_02568_b200.engine import Engine  # noqa: E402

e = Engine(0)
S, m, k = 65536, 4, 64
T = S // m
q = e.gen_normal_bf16(S * 64 * 128, 128 ** -0.5, 9, 1)
kc = e.gen_normal_bf16(T * 128, 128 ** -0.5, 9, 2)
w = e.gen_normal_f32(S * 64, (64 * 128) ** -0.5, 9, 3)
dims = api.ProblemDims.create(1, S, m, 64, 128, k)
cfg = api.DriverConfig(tile=api.TileConfig(2048, T))
starts = [S - 2048, 40960, 8192]
os.environ["CSAIDX_TWO_LEVEL"] = "0"
i0, v0, _ = api.run_chunked_device(q, kc, w, dims, cfg, starts)
drv = api.KernelStats(api.driver_engine(0))
os.environ["CSAIDX_TWO_LEVEL"] = "1"
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    drv.candidate_hits(reset=True)
    i1, v1, _ = api.run_chunked_device(q, kc, w, dims, cfg, starts)
    hits = drv.candidate_hits(reset=True)
    a, b = i0.cpu().numpy().reshape(-1, k), i1.cpu().numpy().reshape(-1, k)
    va, vb = v0.cpu().numpy().reshape(-1, k), v1.cpu().numpy().reshape(-1, k)
    bad = np.argwhere((a != b).any(axis=1)).ravel()
    print("rep", rep, "hits", hits, "bad rows", len(bad), bad[:6].tolist(), flush=True)
    for r in bad[:3]:
        d = np.argwhere(a[r] != b[r]).ravel()
        print("  row", r, "pos", d[:6].tolist(), "i0", a[r, d[:4]].tolist(), "i1", b[r, d[:4]].tolist(),
              "v0", va[r, d[:4]].tolist(), "v1", vb[r, d[:4]].tolist())
