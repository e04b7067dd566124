"""Score kernel wait-cycle breakdown per role (dev tool): where the MMA issuer idles."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_02568_b200.engine import Engine, dims_struct
from paper_2605_02568_b200._capi import check

e = Engine(0)
B, S, H, D, m, k = 1, 262144, 64, 128, 4, 1024
T = S // m
q = e.gen_normal_bf16(B * S * H * D, D ** -0.5, 3, 1)
kc = e.gen_normal_bf16(B * T * D, D ** -0.5, 3, 2)
w = e.gen_normal_f32(B * S * H, (D * H) ** -0.5, 3, 3)
dims = dims_struct(B, S, H, D, m, k)
out = torch.empty((1, 2048, T), dtype=torch.float32, device="cuda")
nsm = e.num_sms
for s0 in (int(os.environ.get("S0", 200704)), 40960):
    rows, cols = 2048, T
    legal = np.clip((s0 + np.arange(rows) + 1) // m, 0, cols)
    pairs = int(legal.sum())
    for _ in range(3):
        e.score(q, kc, w, dims, s0, rows, 0, cols, apply_mask=True, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        e.score(q, kc, w, dims, s0, rows, 0, cols, apply_mask=True, out=out)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    probe = torch.zeros(nsm * 8, dtype=torch.int64, device="cuda")
    check(e.lib.csaidx_engine_set_score_probe(e.handle, ctypes.c_void_p(probe.data_ptr())))
    e.score(q, kc, w, dims, s0, rows, 0, cols, apply_mask=True, out=out)
    e.check()
    check(e.lib.csaidx_engine_set_score_probe(e.handle, None))
    c = probe.view(nsm, 8).cpu().numpy().astype(np.float64)
    span = c[:, 3].mean()
    names = ["mma wait k_full", "mma wait acc_empty", "mma wait q_full", "mma span", "epi wait acc_full",
             "epi span", "prod wait k_empty", "prod wait q_empty"]
    print(f"s0={s0}: {ms:.3f} ms  {pairs * 16384 / ms / 1e9:.0f} TFLOP/s", flush=True)
    for i, n in enumerate(names):
        print(f"   {n:20s} {c[:, i].mean():12.0f} cycles  ({c[:, i].mean() / span * 100:5.1f}% of MMA span)  "
              f"min {c[:, i].min():.0f} max {c[:, i].max():.0f}", flush=True)
