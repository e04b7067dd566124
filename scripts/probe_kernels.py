"""Quick device-time probe of the three kernels at a C3-sized chunk (dev tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_02568_b200.engine import Engine, dims_struct

S, H, D, m, k = 262144, 64, 128, 4, 1024
T = S // m
e = Engine(0)
q = e.gen_normal_bf16(S * H * D, D ** -0.5, 1, 1)
kc = e.gen_normal_bf16(T * D, D ** -0.5, 1, 2)
w = e.gen_normal_f32(S * H, (D * H) ** -0.5, 1, 3)
dims = dims_struct(1, S, H, D, m, k)
for rows, s0 in [(2048, S - 2048), (2048, S // 2)]:
    cols = T
    ld = cols
    sb = torch.empty((1, rows, ld), dtype=torch.float32, device="cuda")
    legal_pairs = sum(min(cols, (s0 + i + 1) // m) for i in range(rows))
    for it in range(3):
        e.score(q, kc, w, dims, s0, rows, 0, cols, apply_mask=True, out=sb)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    ev0.record()
    for it in range(n):
        e.score(q, kc, w, dims, s0, rows, 0, cols, apply_mask=True, out=sb)
    ev1.record(); torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / n
    e.check()
    print(f"score_tc rows={rows} s0={s0}: {ms:.3f} ms, legal pairs {legal_pairs:.3e}, "
          f"{legal_pairs*16384/ms/1e9:.1f} TFLOP/s", flush=True)
    ev0.record()
    for it in range(n):
        v, i = e.select(sb, 1, rows, cols, s0, 0, m, k)
    ev1.record(); torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / n
    print(f"select rows={rows}: {ms:.3f} ms, {legal_pairs*4/ms/1e6:.1f} GB/s (1 pass equiv)", flush=True)
    rv = v.clone(); ri = i.clone()
    ev0.record()
    for it in range(n):
        e.merge(rv, ri, v, i)
    ev1.record(); torch.cuda.synchronize()
    print(f"merge rows={rows}: {ev0.elapsed_time(ev1)/n:.3f} ms", flush=True)
e.check()
