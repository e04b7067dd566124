"""Which group maxima / score entries does score_gmax leave unwritten?"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
from paper_2605_02568_b200.engine import Engine  # noqa: E402
from test_gpu_kernels import _v4_dims  # noqa: E402

e = Engine(0)
S, m, k = 65536, 4, 64
T = S // m
q = e.gen_normal_bf16(S * 64 * 128, 128 ** -0.5, 9, 1)
kc = e.gen_normal_bf16(T * 128, 128 ** -0.5, 9, 2)
w = e.gen_normal_f32(S * 64, (64 * 128) ** -0.5, 9, 3)
d = _v4_dims(S, k)
for s0 in (S - 2048, 40960):
    rows = 2048
    tile, gmax = e.score_gmax(q, kc, w, d, s0, rows, 0, T, fill=float("nan"))
    e.check()
    t = tile[0].cpu().numpy()
    g = gmax[0].cpu().numpy()
    legal = np.minimum((s0 + np.arange(rows) + 1) // m, T)
    bad_t, bad_g = [], []
    for r in range(rows):
        n = legal[r]
        if np.isnan(t[r, :n]).any():
            bad_t.append((r, int(np.argwhere(np.isnan(t[r, :n]))[0][0])))
        ng = (n + 31) // 32
        x = np.pad(np.where(np.isnan(t[r, :n]), -np.inf, t[r, :n]), (0, ng * 32 - n), constant_values=-np.inf)
        ref = x.reshape(-1, 32).max(axis=1)
        mis = np.argwhere(~(g[r, :ng] == ref)).ravel()
        if len(mis):
            bad_g.append((r, mis[:4].tolist(), g[r, mis[:2]].tolist(), ref[mis[:2]].tolist()))
    print(s0, "unwritten score rows", len(bad_t), bad_t[:4], "gmax mismatching rows", len(bad_g), bad_g[:4])
