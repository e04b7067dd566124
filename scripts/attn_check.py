"""(dev, GPU box) Sparse attention vs the float64 restatement on small cases."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle.sparse_attention import sparse_attention
from paper_2605_02568_b200.engine import Engine

e = Engine(0)
torch.manual_seed(0)
for (B, S, T, k) in [(1, 4, 64, 16), (1, 8, 256, 64), (2, 6, 300, 100), (1, 16, 2048, 1024)]:
    H, D = 128, 576
    q = torch.randn(B, S, H, D, device="cuda").to(torch.bfloat16)
    kv = torch.randn(B, T, D, device="cuda").to(torch.bfloat16)
    idx = torch.stack([torch.stack([torch.randperm(T, device="cuda")[:k] for _ in range(S)]) for _ in range(B)]).int()
    idx[:, 0, k // 2:] = -1           # padding
    if S > 2:
        idx[:, 1, :] = -1             # an empty row
    if S > 3:
        idx[:, 2, 0] = T + 5          # out of range -> skipped
    sc = 1.0 / D ** 0.5
    out, lse = e.sparse_attention(q, kv, idx, sc)
    torch.cuda.synchronize()
    ro, rl = sparse_attention(q.float().cpu().numpy(), kv.float().cpu().numpy(), idx.cpu().numpy(), sc)
    go = out.float().cpu().numpy()
    gl = lse.cpu().numpy()
    err = np.abs(go - ro)
    scale = np.abs(ro).max(axis=-1, keepdims=True) + 1e-30
    rel = (err / scale).max()
    lerr = np.nanmax(np.abs(np.where(np.isinf(rl), 0, gl - rl)))
    inf_ok = np.array_equal(np.isinf(rl), np.isinf(gl))
    print(f"B={B} S={S} T={T} k={k}: max err/rowmax {rel:.3e}, mean abs err {err.mean():.3e}, lse err {lerr:.3e}, "
          f"empty rows ok {inf_ok}, nan {np.isnan(go).any()}", flush=True)
