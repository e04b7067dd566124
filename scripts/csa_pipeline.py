"""The CSA layer step on one B200: the lightning indexer
(this library's chunked driver, device-resident) -> TopK(t) as int32 rows
written straight into the attention's index buffer (the index sink, no
int64 / fp32 outputs) -> sparse MLA attention over those rows
(csaidx_cuda_sparse_attention). The paper composes its indexer with
TileLang's attention the same way (Table "composition").
Synthetic inputs; CUDA events; prints one JSON line.

usage: python scripts/csa_pipeline.py [S] [k] [steps]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_02568_b200 import api
from paper_2605_02568_b200.engine import Engine

S, k, steps = (int(x) for x in (sys.argv[1:] + ["65536", "512", "3"])[:3])
B, m, Hi, D = 1, 4, 64, 128
H, Dqk, Dv = 128, 576, 512
T = S // m
e = Engine(0)
torch.cuda.reset_peak_memory_stats()
# indexer operands (V4-Flash indexer shape) and the attention's q / latent cache
q_i = e.gen_normal_bf16(B * S * Hi * D, D ** -0.5, 1, 1)
kc_i = e.gen_normal_bf16(B * T * D, D ** -0.5, 1, 2)
w_i = e.gen_normal_f32(B * S * Hi, (D * Hi) ** -0.5, 1, 3)
g = torch.Generator(device="cuda").manual_seed(7)
q_a = torch.randn(B, S, H, Dqk, device="cuda", generator=g, dtype=torch.bfloat16)
kv_a = torch.randn(B, T, Dqk, device="cuda", generator=g, dtype=torch.bfloat16)
idx = torch.empty(B, S, k, dtype=torch.int32, device="cuda")
out = torch.empty(B, S, H, Dv, dtype=torch.bfloat16, device="cuda")
dims = api.ProblemDims.create(B, S, m, Hi, D, k)
cfg = api.DriverConfig(tile=api.TileConfig(2048, T))
eng = api.driver_engine(0)
api.set_index_sink(eng, idx.data_ptr(), B, S, k)  # the indexer's rows land as int32 in idx
sc = Dqk ** -0.5


def indexer():
    api.run_chunked_device(q_i, kc_i, w_i, dims, cfg, outputs=False)


def attention():
    e.sparse_attention(q_a, kv_a, idx, sc, out=out, lse=False)


def timed(fn, n):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n


indexer()
attention()
torch.cuda.synchronize()
t_idx = timed(indexer, steps)
t_att = timed(attention, steps)
t_all = timed(lambda: (indexer(), attention()), steps)
api.set_index_sink(eng, None)
e.check()
legal = sum((t + 1) // m for t in range(S))
valid = int((idx >= 0).sum().item())
print(json.dumps({
    "pipeline": "indexer (chunked, c_S=2048, index sink int32) -> sparse MLA attention",
    "config": {"B": B, "S": S, "T": T, "k": k, "indexer": {"H_I": Hi, "d_h": D, "m": m},
               "attention": {"heads": H, "dqk": Dqk, "dv": Dv}},
    "indexer_ms": t_idx, "attention_ms": t_att, "pipeline_ms": t_all,
    "indexer_legal_pairs_per_s": legal / t_idx * 1e3,
    "attention_useful_tflops": 2.0 * H * valid * (Dqk + Dv) / t_att / 1e9,
    "valid_indices": valid,
    "peak_hbm_gb_torch": torch.cuda.max_memory_allocated() / 1e9,
    "note": "peak includes the attention's q [S,128,576] and out [S,128,512] bf16 tensors",
}))
