"""Repeat the per-row vs persistent multi-row select comparison and report
which side (if any) diverges from the sort-based reference (race hunting)."""
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from test_gpu_kernels import ref_select  # noqa: E402
from paper_2605_02568_b200.engine import Engine  # noqa: E402

e = Engine(0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
bad = {"per_row": 0, "persistent": 0}
for cols, k in [(40000, 1024), (3000, 512), (9000, 100)]:
    rng = np.random.default_rng(cols)
    B, rows = 2, 37
    x = rng.normal(0, 1, (B, rows, cols)).astype(np.float32)
    x[1] = np.round(x[1] * 8) / 8
    ld = (cols + 3) // 4 * 4
    pad = np.zeros((B, rows, ld), np.float32)
    pad[:, :, :cols] = x
    dev = torch.from_numpy(pad).cuda()
    wv, wi = ref_select(x, cols + 5000, 0, 1, k)
    for r in range(reps):
        v0, i0 = e.select(dev, B, rows, cols, cols + 5000, 0, 1, k)
        e.check()
        e.set_partition(100, 7)
        v1, i1 = e.select(dev, B, rows, cols, cols + 5000, 0, 1, k)
        e.check()
        e.set_partition(0, 0)
        for name, ii in (("per_row", i0), ("persistent", i1)):
            got = ii.cpu().numpy()
            if not np.array_equal(got, wi):
                bad[name] += 1
                diff = np.argwhere((got != wi).any(axis=-1))
                print(cols, k, "rep", r, name, "bad rows", diff[:8].tolist(), "n", len(diff), flush=True)
print("summary", bad)
