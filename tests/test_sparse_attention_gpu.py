"""Sparse attention over the indexer's top-k through the
C-ABI (csaidx_cuda_sparse_attention), against the float64 restatement in
oracle/sparse_attention.py.

Tolerance (floating point: bf16 q / kv, fp32 accumulation, P rounded to bf16
for the PV product, bf16 output): per (query, head) row,
max |out - ref| <= 1e-2 * max |ref row|, mean |out - ref| <= 2^-8 (one bf16 ulp) * mean |ref|,
and |lse - ref| <= 1e-4 absolute; rows with no valid index give out = 0 and
lse = -inf exactly.
"""
import numpy as np
import pytest
import torch

from oracle.sparse_attention import sparse_attention as ref_attention

pytestmark = pytest.mark.gpu

H, DQK, DV = 128, 576, 512


@pytest.fixture(autouse=True, params=["pair", "single"])
def kernel_form(request, monkeypatch):
    """Every case on both kernels: the single-CTA form (default) and the
    CTA-pair form (CSAIDX_ATTN_PAIR=1: Dqk split across a cluster of 2)."""
    monkeypatch.setenv("CSAIDX_ATTN_PAIR", "1" if request.param == "pair" else "0")
    return request.param


@pytest.fixture(scope="module")
def eng():
    from paper_2605_02568_b200.engine import Engine
    return Engine(0)


def _check(out, lse, q, kv, idx, sc):
    ro, rl = ref_attention(q.float().cpu().numpy(), kv.float().cpu().numpy(), idx.cpu().numpy(), sc)
    go = out.float().cpu().numpy()
    gl = lse.cpu().numpy()
    empty = np.isinf(rl)
    assert np.array_equal(np.isinf(gl) & (gl < 0), empty)
    assert np.all(go[empty] == 0)
    err = np.abs(go - ro)
    rowmax = np.abs(ro).max(axis=-1, keepdims=True)
    live = ~empty
    assert np.all(err[live] <= 1e-2 * rowmax[live] + 1e-6), float((err[live] / (rowmax[live] + 1e-30)).max())
    assert err[live].mean() <= 2 ** -8 * np.abs(ro[live]).mean()
    assert np.abs(gl[live] - rl[live]).max() <= 1e-4
    return float((err[live] / (rowmax[live] + 1e-30)).max())


def _inputs(B, S, T, k, seed, scale=1.0, heads=H):
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = (torch.randn(B, S, heads, DQK, device="cuda", generator=g) * scale).to(torch.bfloat16)
    kv = torch.randn(B, T, DQK, device="cuda", generator=g).to(torch.bfloat16)
    idx = torch.argsort(torch.rand(B * S, T, device="cuda", generator=g), dim=1)[:, :k]
    return q, kv, idx.reshape(B, S, k).int().contiguous()


@pytest.mark.parametrize("B,S,T,k", [(1, 4, 64, 16), (1, 8, 256, 64), (2, 5, 300, 100), (1, 12, 4096, 1024),
                                     (1, 3, 8192, 2048), (2, 3, 5000, 4096), (1, 1, 10, 1), (3, 2, 40, 33),
                                     (1, 400, 2048, 96)])
def test_sparse_attention_matches_oracle(eng, B, S, T, k):
    q, kv, idx = _inputs(B, S, T, k, seed=B * 1000 + S * 10 + k)
    if k > 1:
        idx[:, 0, k // 2:] = -1      # padding tail
    if S > 2:
        idx[:, 1, :] = -1            # a query with no valid index
        idx[:, 2, 0] = T + 7         # out of range: skipped
    sc = DQK ** -0.5
    out, lse = eng.sparse_attention(q, kv, idx, sc)
    _check(out, lse, q, kv, idx, sc)


@pytest.mark.parametrize("heads", [256, 384])
def test_sparse_attention_head_groups(eng, heads):
    """H a multiple of 128: one work item per group of 128 heads."""
    B, S, T, k = 2, 5, 1000, 200
    q, kv, idx = _inputs(B, S, T, k, seed=heads, heads=heads)
    idx[:, 1, :] = -1
    idx[:, 0, 150:] = -1
    sc = DQK ** -0.5
    out, lse = eng.sparse_attention(q, kv, idx, sc)
    _check(out, lse, q, kv, idx, sc)


def test_sparse_attention_large_logits_rescale(eng):
    """Scores spread over ~100 in log2 units: the lazy O rescale (max grows
    by > 2^8 between blocks) runs on most rows; ordering the keys by
    increasing score forces a new maximum in nearly every block."""
    B, S, T, k = 1, 6, 2048, 512
    q, kv, idx = _inputs(B, S, T, k, seed=5, scale=4.0)
    s = torch.einsum("bshd,btd->bsht", q.float(), kv.float())[:, :, 0]  # head 0 scores
    order = torch.argsort(s.gather(2, idx.long()), dim=2)
    idx = idx.gather(2, order).int().contiguous()
    sc = DQK ** -0.5
    out, lse = eng.sparse_attention(q, kv, idx, sc)
    _check(out, lse, q, kv, idx, sc)


def test_sparse_attention_on_indexer_output(eng):
    """Composition: the indices come from this library's
    own chunked indexer on a V4-shaped problem (int64 TopKResult, -1 tail for
    the first queries) and feed the attention unchanged."""
    from paper_2605_02568_b200 import api
    from oracle.oracle import Oracle
    orc = Oracle()
    Bq, S, m, Hi, D, k = 1, 512, 4, 64, 128, 64
    qi, kci, wi = orc.generate_inputs(Bq, S, m, Hi, D, 3, bf16=True)
    dims = api.ProblemDims.create(Bq, S, m, Hi, D, k)
    res, _ = api.run_chunked(api.IndexerInputs.validated(qi, kci, wi, dims), dims,
                             api.DriverConfig(tile=api.TileConfig(128, 128)))
    idx = torch.from_numpy(res.indices.astype(np.int32)).cuda().contiguous()
    T = S // m
    g = torch.Generator(device="cuda").manual_seed(9)
    q = torch.randn(Bq, S, H, DQK, device="cuda", generator=g).to(torch.bfloat16)
    kv = torch.randn(Bq, T, DQK, device="cuda", generator=g).to(torch.bfloat16)
    sc = DQK ** -0.5
    out, lse = eng.sparse_attention(q, kv, idx, sc)
    _check(out, lse, q, kv, idx, sc)
    assert torch.isinf(lse[0, :3]).all()  # queries 0..2 have no legal compressed key (m = 4)


def test_sparse_attention_rejects_other_shapes(eng):
    from paper_2605_02568_b200._capi import InvalidArgument
    q = torch.zeros(1, 2, 64, DQK, dtype=torch.bfloat16, device="cuda")
    kv = torch.zeros(1, 8, DQK, dtype=torch.bfloat16, device="cuda")
    idx = torch.zeros(1, 2, 4, dtype=torch.int32, device="cuda")
    with pytest.raises(InvalidArgument):
        eng.sparse_attention(q, kv, idx, 1.0)
    q = torch.zeros(1, 2, H, DQK, dtype=torch.bfloat16, device="cuda")
    idx = torch.zeros(1, 2, 5000, dtype=torch.int32, device="cuda")
    with pytest.raises(InvalidArgument):
        eng.sparse_attention(q, kv, idx, 1.0)
