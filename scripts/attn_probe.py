"""(dev, GPU box) per-block clock64 stamps of the CTA-pair attention kernel
built with -DCSAIDX_ATTN_PROBE=1 (CTA 0: softmax warp 0 and the MMA issuer).
usage: python scripts/attn_probe.py [S] [k]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2605_02568_b200.engine import Engine

S, k = (int(x) for x in (sys.argv[1:] + ["2048", "1024"])[:2])
T, H, Dqk, Dv = 65536, 128, 576, 512
e = Engine(0)
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn(1, S, H, Dqk, device="cuda", generator=g).to(torch.bfloat16)
kv = torch.randn(1, T, Dqk, device="cuda", generator=g).to(torch.bfloat16)
idx = torch.argsort(torch.rand(S, T, device="cuda", generator=g), dim=1)[:, :k].int().unsqueeze(0).contiguous()
out = torch.empty(1, S, H, Dv, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    e.sparse_attention(q, kv, idx, 1.0 / Dqk ** 0.5, out=out)
torch.cuda.synchronize()
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2605_02568_b200", "lib", "libcsaidx_cuda.so"))
n = 2048 * 8
buf = (ctypes.c_longlong * n)()
assert lib.csaidx_dev_attn_probe(buf, n) == 0
a = np.frombuffer(buf, dtype=np.int64).reshape(2048, 8).astype(np.float64)
nb = (k + 31) // 32
blocks = a[64:1024]  # steady state
d = lambda i, j: np.median(blocks[:, j] - blocks[:, i])
per_block = np.median(np.diff(blocks[:, 0]))
print(f"per block (softmax iteration start to start): {per_block:.0f} cycles")
print(f"  send(g+1) [wait S(g+1), ld, st.async]: {d(0, 1):.0f}")
print(f"  kv_full + valid word + wait peer partial: {d(1, 2):.0f}")
print(f"  add + max + exp + P store + arrive: {d(2, 3):.0f}")
print(f"  MMA: kv_full(g) seen -> p_full(g) seen: {d(4, 5):.0f}; QK(g) issue vs softmax start of g: {np.median(blocks[:, 4] - blocks[:, 0]):.0f}")
print(f"  p_full(g) seen at MMA - P arrive by warp 0: {np.median(blocks[:, 5] - blocks[:, 3]):.0f}")
print(f"  MMA kv_full waits start to start: {np.median(np.diff(blocks[:, 4])):.0f}")
