"""CPU checks of the sparse attention restatement (oracle/sparse_attention.py):
against a dense masked softmax over all T keys, padding / empty rows, and
invariance to the order of the index list."""
import numpy as np

from oracle.sparse_attention import sparse_attention


def _dense(q, kv, indices, sc, dv):
    B, S, H, D = q.shape
    T = kv.shape[1]
    out = np.zeros((B, S, H, dv))
    lse = np.full((B, S, H), -np.inf)
    for b in range(B):
        for t in range(S):
            mask = np.zeros(T, bool)
            idx = indices[b, t]
            mask[idx[(idx >= 0) & (idx < T)]] = True
            if not mask.any():
                continue
            s = (q[b, t].astype(np.float64) @ kv[b].astype(np.float64).T) * sc
            s[:, ~mask] = -np.inf
            mx = s.max(axis=1, keepdims=True)
            p = np.exp(s - mx)
            out[b, t] = p @ kv[b, :, :dv].astype(np.float64) / p.sum(axis=1, keepdims=True)
            lse[b, t] = mx[:, 0] + np.log(p.sum(axis=1))
    return out, lse


def test_matches_dense_masked_softmax():
    rng = np.random.default_rng(0)
    B, S, H, D, T, k, dv = 2, 5, 4, 24, 40, 7, 16
    q = rng.normal(size=(B, S, H, D)).astype(np.float32)
    kv = rng.normal(size=(B, T, D)).astype(np.float32)
    idx = np.stack([np.stack([rng.permutation(T)[:k] for _ in range(S)]) for _ in range(B)])
    idx[0, 1, 3:] = -1
    idx[1, 2, :] = -1
    idx[1, 3, 0] = T + 1
    o1, l1 = sparse_attention(q, kv, idx, 0.3, dv)
    o2, l2 = _dense(q, kv, idx, 0.3, dv)
    assert np.allclose(o1, o2, rtol=1e-12, atol=1e-12)
    assert np.array_equal(np.isinf(l1), np.isinf(l2))
    fin = np.isfinite(l2)
    assert np.allclose(l1[fin], l2[fin], rtol=1e-12)
    assert np.all(o1[1, 2] == 0) and np.all(np.isneginf(l1[1, 2]))


def test_index_order_does_not_matter():
    rng = np.random.default_rng(1)
    q = rng.normal(size=(1, 2, 3, 8))
    kv = rng.normal(size=(1, 20, 8))
    idx = np.stack([rng.permutation(20)[:9] for _ in range(2)])[None]
    o1, l1 = sparse_attention(q, kv, idx, 0.5, 6)
    o2, l2 = sparse_attention(q, kv, idx[:, :, ::-1].copy(), 0.5, 6)
    assert np.allclose(o1, o2) and np.allclose(l1, l2)
