"""Small GPU workloads for compute-sanitizer (tests/test_sanitizers_gpu.py):
each case drives one family of the hand-written kernels through the C-ABI at
a size the sanitizer finishes in seconds to a minute.

  smoke      V4 indexer step (tcgen05 score + select_final) and an exact-kernel
             run with a key tiling (select + merge + finalize)
  select     the per-row select: sampled threshold + bucket finish, heavy
             ties (radix path), mispredicted samples (exact global fallback),
             and the large-take path (k > 4096)
  persistent the persistent multi-row select (SM partition)
  two_level  the group-maxima score epilogue + two-level select, incl. a
             row whose last 32-key group is partial at the end of the buffer
  attention_pair  the same through the opt-in CTA-pair kernel (cluster of 2, DSMEM exchange)
  attention  the sparse attention over top-k indices (persistent tcgen05
             kernel: cp.async gathers, TMEM Q / S / P / O, lazy rescale),
             with padding, an empty row, out-of-range indices, large logits
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_02568_b200 import api
from paper_2605_02568_b200.engine import Engine, dims_struct


def rows(B, R, n, seed, quant=False):
    x = np.random.default_rng(seed).normal(0, 1, (B, R, n)).astype(np.float32)
    if quant:
        x = np.round(x * 4) / 4
    ld = (n + 3) // 4 * 4
    pad = np.zeros((B, R, ld), np.float32)
    pad[:, :, :n] = x
    return torch.from_numpy(pad).cuda()


def case_smoke(e):
    B, S, m, H, D, k = 1, 1024, 4, 64, 128, 64
    q = e.gen_normal_bf16(B * S * H * D, D ** -0.5, 1, 1)
    kc = e.gen_normal_bf16(B * (S // m) * D, D ** -0.5, 1, 2)
    w = e.gen_normal_f32(B * S * H, (D * H) ** -0.5, 1, 3)
    dims = api.ProblemDims.create(B, S, m, H, D, k)
    api.run_chunked_device(q, kc, w, dims, api.DriverConfig(tile=api.TileConfig(256, S // m)))
    api.run_chunked_device(q, kc, w, dims, api.DriverConfig(tile=api.TileConfig(256, 128)))
    qx = torch.randn(2 * 64 * 3 * 5, device="cuda")
    kx = torch.randn(2 * 16 * 5, device="cuda")
    wx = torch.randn(2 * 64 * 3, device="cuda")
    dx = api.ProblemDims.create(2, 64, 4, 3, 5, 6)
    api.run_chunked_device(qx, kx, wx, dx, api.DriverConfig(tile=api.TileConfig(9, 5),
                                                              kernel=api.ScoreKernel.scalar))


def case_select(e):
    e.select(rows(1, 4, 20000, 1), 1, 4, 20000, 10 ** 6, 0, 1, 1024)            # sampled + bucket finish
    e.select(rows(1, 3, 12000, 2, quant=True), 1, 3, 12000, 10 ** 6, 0, 1, 1024)  # heavy ties
    x = rows(1, 2, 65536, 3)
    x[..., ((torch.arange(65536, device="cuda") // 8) % 16) == 0] = -10.0     # the sample mispredicts
    e.select(x, 1, 2, 65536, 10 ** 7, 0, 1, 1024)                              # exact global fallback
    e.select(rows(1, 2, 9000, 4), 1, 2, 9000, 10 ** 6, 0, 1, 5000)             # large take
    e.select(rows(1, 3, 3000, 5), 1, 3, 3000, 10 ** 6, 0, 1, 512)              # short rows: direct path


def case_persistent(e):
    x = rows(2, 9, 20000, 6)
    e.set_partition(100, 7)
    try:
        e.select(x, 2, 9, 20000, 25000, 0, 1, 1024)
    finally:
        e.set_partition(0, 0)


def case_two_level(e):
    S, m, k = 8192, 4, 64
    T = S // m
    q = e.gen_normal_bf16(S * 64 * 128, 128 ** -0.5, 7, 1)
    kc = e.gen_normal_bf16(T * 128, 128 ** -0.5, 7, 2)
    w = e.gen_normal_f32(S * 64, (64 * 128) ** -0.5, 7, 3)
    d = dims_struct(1, S, 64, 128, m, k)
    s0, R = S - 64, 64
    tile, gmax = e.score_gmax(q, kc, w, d, s0, R, 0, T)
    oi = torch.zeros((1, R, k), dtype=torch.int64, device="cuda")
    ov = torch.zeros((1, R, k), dtype=torch.float32, device="cuda")
    e.select_final(tile, 1, R, T, s0, 0, m, k, oi, ov, 0, gmax=gmax)
    # T = 2050: the last row's last group (keys 2048..2079) ends past the
    # buffer's last row (ld = 2052); only its legal float4s may be read
    S2, k2 = 8200, 32
    T2 = S2 // m
    q2 = e.gen_normal_bf16(S2 * 64 * 128, 128 ** -0.5, 8, 1)
    kc2 = e.gen_normal_bf16(T2 * 128, 128 ** -0.5, 8, 2)
    w2 = e.gen_normal_f32(S2 * 64, (64 * 128) ** -0.5, 8, 3)
    d2 = dims_struct(1, S2, 64, 128, m, k2)
    tile2, gmax2 = e.score_gmax(q2, kc2, w2, d2, S2 - 64, 64, 0, T2)
    oi2 = torch.zeros((1, 64, k2), dtype=torch.int64, device="cuda")
    ov2 = torch.zeros((1, 64, k2), dtype=torch.float32, device="cuda")
    e.select_final(tile2, 1, 64, T2, S2 - 64, 0, m, k2, oi2, ov2, 0, gmax=gmax2)


def case_attention(e):
    H, D = 128, 576
    g = torch.Generator(device="cuda").manual_seed(3)
    for (B, S, T, k, scale) in [(1, 6, 300, 100, 1.0), (2, 3, 2048, 512, 4.0)]:
        q = (torch.randn(B, S, H, D, device="cuda", generator=g) * scale).to(torch.bfloat16)
        kv = torch.randn(B, T, D, device="cuda", generator=g).to(torch.bfloat16)
        idx = torch.argsort(torch.rand(B * S, T, device="cuda", generator=g), dim=1)[:, :k].reshape(B, S, k).int()
        idx[:, 0, k // 2:] = -1
        idx[:, 1, :] = -1
        idx[:, 2, 0] = T + 3
        e.sparse_attention(q, kv, idx.contiguous(), D ** -0.5)


def case_attention_pair(e):
    # the opt-in CTA-pair form (read per call by csaidx_cuda_sparse_attention)
    os.environ["CSAIDX_ATTN_PAIR"] = "1"
    try:
        case_attention(e)
    finally:
        del os.environ["CSAIDX_ATTN_PAIR"]


if __name__ == "__main__":
    e = Engine(0)
    for name in sys.argv[1:]:
        globals()[f"case_{name}"](e)
        e.check()
    torch.cuda.synchronize()
    print("cases ok:", " ".join(sys.argv[1:]))
