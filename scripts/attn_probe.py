"""(dev, GPU box) per-block clock64 stamps of the CTA-pair attention kernel
built with -DCSAIDX_ATTN_PROBE=1 (CTA 0). Slots per block g: 0 softmax start,
1 own partial sent, 2 peer partial landed, 3 P stored (the team handling g);
4 MMA saw kv_full(g), 5 MMA saw p_full(g); 6 producer saw the stage free,
7 producer issued the copies.
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
n = 2048 * 16
buf = (ctypes.c_longlong * n)()
assert lib.csaidx_dev_attn_probe(buf, n) == 0
a = np.frombuffer(buf, dtype=np.int64).reshape(2048, 16).astype(np.float64)
nb = (k + 31) // 32
rows = [g for g in range(64, 1000) if 2 <= g % nb <= nb - 3]  # steady state, away from item boundaries
B = a[rows]
med = lambda v: float(np.median(v))
print(f"steady block period (MMA kv_full seen): {med(np.diff(a[64:1000, 4])[[r - 64 for r in rows[:-1]]]):.0f} cycles")
print(f"softmax (team of block g): start->sent {med(B[:,1]-B[:,0]):.0f}, sent->peer landed {med(B[:,2]-B[:,1]):.0f}, ->P stored {med(B[:,3]-B[:,2]):.0f}, total {med(B[:,3]-B[:,0]):.0f}")
print(f"  inside ->P stored: peer landed -> m(g-1) known {med(B[:,8]-B[:,2]):.0f}, -> exps done {med(B[:,9]-B[:,8]):.0f}, -> P stored+arrive {med(B[:,3]-B[:,9]):.0f}")
print(f"softmax start(g) - QK(g) kv_full seen: {med(B[:,0]-B[:,4]):.0f}; P stored(g) -> MMA sees p_full(g): {med(B[:,5]-B[:,3]):.0f}")
print(f"producer: stage free(g) -> copies issued {med(B[:,7]-B[:,6]):.0f}; copies issued(g) -> MMA sees kv_full(g) {med(B[:,4]-B[:,7]):.0f}")
print(f"stage free(g) - PV issue(g-7) [p_full seen]: {med(a[rows,6]-a[[r-7 for r in rows],5]):.0f}")
bidx = [gg for gg in range(64, 999) if (gg + 1) % nb == 0]
print(f"item boundary: MMA kv_full gap {med([a[gg+1,4]-a[gg,4] for gg in bidx]):.0f}, p_full gap {med([a[gg+1,5]-a[gg,5] for gg in bidx]):.0f}")
