"""Sparse attention over the indexer's top-k (f4) on one B200: throughput of
csaidx_cuda_sparse_attention at a V4-like decode-free shape (every query
attends k = 1024 gathered latent rows of a T-row cache), CUDA events over
the timed launches, NVML clocks during them. Prints one JSON line.

usage: python scripts/bench_attention.py [S] [T] [k] [steps]"""
import json, os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pynvml
from paper_2605_02568_b200.engine import Engine

S, T, k, steps = (int(x) for x in (sys.argv[1:] + ["8192", "65536", "1024", "20"])[:4])
H, Dqk, Dv = 128, 576, 512
e = Engine(0)
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn(1, S, H, Dqk, device="cuda", generator=g).to(torch.bfloat16)
kv = torch.randn(1, T, Dqk, device="cuda", generator=g).to(torch.bfloat16)
# distinct random indices per query (the indexer's output has no repeats)
idx = torch.argsort(torch.rand(S, T, device="cuda", generator=g), dim=1)[:, :k].int().unsqueeze(0).contiguous()
sc = 1.0 / Dqk ** 0.5
out = torch.empty(1, S, H, Dv, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    e.sparse_attention(q, kv, idx, sc, out=out)
torch.cuda.synchronize()
pynvml.nvmlInit()
hdl = pynvml.nvmlDeviceGetHandleByIndex(0)
clocks, power, stop = [], [], threading.Event()


def poll():
    while not stop.is_set():
        clocks.append(pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM))
        power.append(pynvml.nvmlDeviceGetPowerUsage(hdl) / 1000)
        time.sleep(0.02)


th = threading.Thread(target=poll)
th.start()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(steps):
    e.sparse_attention(q, kv, idx, sc, out=out)
b.record()
b.synchronize()
stop.set()
th.join()
ms = a.elapsed_time(b) / steps
e.check()
useful = 2.0 * H * k * (Dqk + Dv) * S          # QK^T + PV, FLOP per launch
issued = 2.0 * H * k * (2 * Dqk + Dv) * S      # QK^T is computed by both CTAs of a query
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
peak = peaks["bf16_tflops_sustained"]
med = lambda xs: sorted(xs)[len(xs) // 2] if xs else None
print(json.dumps({
    "kernel": "sparse_mla_kernel (tcgen05: S=QK^T M=128 N=32 K=576 with Q[:384] in TMEM, O+=PV M=128 N=256 K=32 with P in TMEM; cp.async gather)",
    "config": {"B": 1, "S": S, "T": T, "k": k, "heads": H, "dqk": Dqk, "dv": Dv, "indices": "random distinct per query"},
    "ms_per_launch": ms, "queries_per_s": S / ms * 1e3,
    "useful_tflops": useful / ms / 1e9, "issued_tflops": issued / ms / 1e9,
    "roofline": {"bound": "tensor", "achieved": useful / ms / 1e9, "peak": peak, "unit": "TFLOP/s",
                 "frac": useful / ms / 1e9 / peak, "issued_frac": issued / ms / 1e9 / peak,
                 "algorithmic": "2*H*k*(dqk+dv) FLOP per query"},
    "gather_bytes_per_query": 2 * k * Dqk * 2,
    "clocks": {"sm_mhz": med(clocks), "power_w": med(power), "samples": len(clocks)},
}))
