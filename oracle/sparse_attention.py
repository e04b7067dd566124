"""CPU restatement of the sparse attention that consumes the indexer's top-k
(SURVEY 8(f) f4). TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke()
and the benchmark's checker may import it; the product path never does.

The reference has no attention code (SPEC.md:8 puts "the attention step
itself" out of its scope; PAPER.md:97 defines the step as "a sparse
attention kernel reads only TopK(t) ... for each query"
composes the chunked indexer with TileLang's sparse MLA kernel). This
restates that sparse-MLA operator in float64:

    out[b,t,h,:dv] = sum_j softmax_j(sm_scale * q[b,t,h,:] . kv[b,i_j,:]) * kv[b,i_j,:dv]
    lse[b,t,h]     = log sum_j exp(sm_scale * q[b,t,h,:] . kv[b,i_j,:])

over the entries i_j of indices[b,t,:] with 0 <= i_j < T (the -1 padding and
out-of-range entries are skipped; a row with none yields out = 0, lse =
-inf). Parity is floating point (bf16 operands, fp32 accumulation, bf16 P
and output on the GPU): parity unpinned by any reference fixture — the
tolerance is stated in tests/test_sparse_attention_gpu.py.
"""
from __future__ import annotations

import numpy as np


def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    """uint16 bf16 bit patterns -> float32."""
    return (u16.astype(np.uint32) << 16).view(np.float32)


def sparse_attention(q: np.ndarray, kv: np.ndarray, indices: np.ndarray, sm_scale: float, dv: int = 512):
    """q [B,S,H,D], kv [B,T,D] (float arrays holding the bf16 values),
    indices [B,S,k] int -> (out [B,S,H,dv] float64, lse [B,S,H] float64)."""
    B, S, H, D = q.shape
    T = kv.shape[1]
    out = np.zeros((B, S, H, dv), dtype=np.float64)
    lse = np.full((B, S, H), -np.inf, dtype=np.float64)
    for b in range(B):
        kvb = kv[b].astype(np.float64)
        for t in range(S):
            idx = indices[b, t]
            sel = idx[(idx >= 0) & (idx < T)]
            if sel.size == 0:
                continue
            K = kvb[sel]                                   # [n, D]
            s = (q[b, t].astype(np.float64) @ K.T) * sm_scale  # [H, n]
            m = s.max(axis=1, keepdims=True)
            p = np.exp(s - m)
            l = p.sum(axis=1)
            out[b, t] = (p @ K[:, :dv]) / l[:, None]
            lse[b, t] = m[:, 0] + np.log(l)
    return out, lse
