"""(dev, GPU box) A3 ablation speed: the score kernel on one late C3 chunk in
fp32 mode (production tcgen05), fp16_emulated on the tensor cores
(CSAIDX_KERNEL_TENSOR) and fp16_emulated on the bit-exact CUDA-core kernel
(on a 64-row slice: it is ~2-3 orders of magnitude slower)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_02568_b200.engine import Engine, dims_struct

e = Engine(0)
S, m, H, D, k = 262144, 4, 64, 128, 1024
T = S // m
dims = dims_struct(1, S, H, D, m, k)
q = e.gen_normal_bf16(S * H * D, D ** -0.5, 1, 1).view(1, S, H, D)
kc = e.gen_normal_bf16(T * D, D ** -0.5, 1, 2).view(1, T, D)
w = e.gen_normal_f32(S * H, (D * H) ** -0.5, 1, 3).view(1, S, H)


def timed(rows, s0, mode, kernel, reps):
    out = e.score(q, kc, w, dims, s0, rows, 0, T, mode=mode, kernel=kernel, apply_mask=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        e.score(q, kc, w, dims, s0, rows, 0, T, mode=mode, kernel=kernel, apply_mask=True, out=out)
    b.record()
    b.synchronize()
    e.check()
    return a.elapsed_time(b) / reps


rows, s0 = 2048, S - 2048
pairs = sum((s0 + i + 1) // m for i in range(rows))
res = {}
for name, mode, kernel, r, reps in [("fp32_tcgen05", 0, 0, rows, 20), ("fp16_emulated_tcgen05", 1, 2, rows, 20),
                                    ("fp16_emulated_exact_cuda_cores", 1, 1, 64, 2)]:
    ms = timed(r, S - r, mode, kernel, reps)
    p = sum((S - r + i + 1) // m for i in range(r))
    res[name] = {"rows": r, "ms": ms, "legal_pairs_per_s": p / ms * 1e3, "tflops": p * 16384 / ms / 1e9}
    print(name, json.dumps(res[name]), flush=True)
