"""Full-size checks on the B200 (BASELINE.json configs C2 and C3), where the
CPU oracle cannot score every row: size-independent properties on every row,
plus the exact tolerance rule (tests/parity.py) on sampled rows scored by the
oracle from the very bf16 operands the GPU consumed.

C3: B=1, S=262,144 (T=65,536), H_I=64, d_h=128, m=4, k=1024, c_S=2048.
C2: B=1, S=65,536 (T=16,384), k=512 — where the materialized path needs a
    256 GiB per-head intermediate on the reference; the GPU materialize path
    (head-reduced [S,T] matrix, 4 GiB) is checked bit-for-bit against chunked.
"""
import numpy as np
import pytest
import torch

from oracle.oracle import Oracle
from paper_2605_02568_b200 import api
from paper_2605_02568_b200.engine import Engine

from .parity import check_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def make_operands(B, S, H, D, m, seed=3):
    e = Engine(0)
    T = S // m
    q = e.gen_normal_bf16(B * S * H * D, D ** -0.5, seed, 1)
    kc = e.gen_normal_bf16(B * T * D, D ** -0.5, seed, 2)
    w = e.gen_normal_f32(B * S * H, (D * H) ** -0.5, seed, 3)
    torch.cuda.synchronize()
    return e, q, kc, w


def row_properties(idx, val, s0, m, k):
    """Every row: sorted under succ, exactly k_eff real entries, legal and
    unique indices, (-1, -inf) tail."""
    rows = idx.shape[0]
    t = s0 + np.arange(rows)
    keff = np.minimum((t + 1) // m, k)
    pos = np.arange(k)[None, :]
    real = pos < keff[:, None]
    assert np.all((idx >= 0) == real), "valid count != k_eff"
    assert np.all(np.isneginf(val[~real])) and np.all(idx[~real] == -1)
    legal = ((t + 1) // m)[:, None]
    assert np.all(idx[real] < np.broadcast_to(legal, idx.shape)[real])
    v = val.astype(np.float64)
    with np.errstate(invalid="ignore"):  # -inf - -inf in the sentinel tail
        dv = v[:, 1:] - v[:, :-1]
    both = real[:, 1:]
    assert not np.any((dv > 0) & both), "not descending"
    tie = (dv == 0) & both
    assert not np.any(tie & (idx[:, 1:] < idx[:, :-1])), "ties not by index"
    srt = np.sort(np.where(real, idx, -1 - pos), axis=1)
    assert not np.any((srt[:, 1:] == srt[:, :-1]) & (srt[:, 1:] >= 0)), "duplicate index"


def oracle_rows(orc, q, kc, w, rows_t, k, m, H, D):
    """Oracle scores (reference op order) of full causal rows, from the GPU's bf16 operands."""
    kcf = kc.float().view(-1, D).cpu().numpy()
    out = []
    for t in rows_t:
        L = (t + 1) // m
        qrow = q[t * H * D:(t + 1) * H * D].float().view(H, D).cpu().numpy()
        wrow = w[t * H:(t + 1) * H].cpu().numpy()
        sc = orc.score_tile(qrow[None, None], kcf[None, :L], wrow[None, None], 0, 0, 1, L)[0, 0]
        out.append(sc)
    return out


def test_c3_full_size_properties_and_sampled_oracle_rows():
    B, S, H, D, m, k = 1, 262144, 64, 128, 4, 1024
    e, q, kc, w = make_operands(B, S, H, D, m)
    dims = api.ProblemDims.create(B, S, m, H, D, k)
    cfg = api.DriverConfig(tile=api.TileConfig(2048, S // m))
    idx, val, st = api.run_chunked_device(q, kc, w, dims, cfg)
    idx2, val2, _ = api.run_chunked_device(q, kc, w, dims, cfg)
    assert torch.equal(idx, idx2) and torch.equal(val, val2), "not deterministic"
    hi = idx[0].cpu().numpy()
    hv = val[0].cpu().numpy()
    for s0 in range(0, S, 16384):  # every row, in slabs
        row_properties(hi[s0:s0 + 16384], hv[s0:s0 + 16384], s0, m, k)
    # sampled rows (incl. the heaviest) against the oracle, tolerance rule
    rows_t = [4103, 70001, 131071, 200003, S - 1]
    orc = Oracle()
    scores = oracle_rows(orc, q, kc, w, rows_t, k, m, H, D)
    rep = check_rows(hi[rows_t], hv[rows_t], scores, [(t + 1) // m for t in rows_t], k)
    assert rep["rows"] == len(rows_t)
    # key-tiling invariance at scale: c_T = 8192 (merge path) gives the same bytes
    starts = [0, 126976, 260096]
    cfg2 = api.DriverConfig(tile=api.TileConfig(2048, 8192))
    i3, v3, st3 = api.run_chunked_device(q, kc, w, dims, cfg2, starts)
    exp = np.concatenate([hi[s:s + 2048] for s in starts])
    assert np.array_equal(i3[0].cpu().numpy(), exp)
    assert st3.dispatch_count == sum(-(-((s + 2048) // m) // 8192) for s in starts)


def test_c3_prefilter_switch_is_bit_identical(monkeypatch):
    """The fused select pre-filter (CSAIDX_SELECT_PREFILTER=1) and the plain
    streaming select (default) give the same bytes at full C3 key length;
    most rows finish from the candidate bitmap."""
    B, S, H, D, m, k = 1, 262144, 64, 128, 4, 1024
    e, q, kc, w = make_operands(B, S, H, D, m, seed=9)
    dims = api.ProblemDims.create(B, S, m, H, D, k)
    cfg = api.DriverConfig(tile=api.TileConfig(2048, S // m))
    starts = [40960, 129024, 260096]
    drv = api.KernelStats(api.driver_engine(0))
    drv.candidate_hits(reset=True)
    monkeypatch.setenv("CSAIDX_SELECT_PREFILTER", "1")
    i1, v1, _ = api.run_chunked_device(q, kc, w, dims, cfg, starts)
    hits = drv.candidate_hits(reset=True)
    monkeypatch.setenv("CSAIDX_SELECT_PREFILTER", "0")
    i0, v0, _ = api.run_chunked_device(q, kc, w, dims, cfg, starts)
    assert drv.candidate_hits(reset=True) == 0
    assert torch.equal(i1, i0) and torch.equal(v1.view(torch.int32), v0.view(torch.int32))
    assert hits >= 0.95 * 3 * 2048, hits


def test_c2_chunked_equals_gpu_materialize_bitwise():
    B, S, H, D, m, k = 1, 65536, 64, 128, 4, 512
    e, q, kc, w = make_operands(B, S, H, D, m, seed=5)
    dims = api.ProblemDims.create(B, S, m, H, D, k)
    idx, val, _ = api.run_chunked_device(q, kc, w, dims, api.DriverConfig(tile=api.TileConfig(2048, 8192)))
    # materialized reference path on device: one [S, T] masked tile + per-row select
    qh = q.float().cpu().numpy()
    kch = kc.float().cpu().numpy()
    wh = w.cpu().numpy()
    inputs = api.IndexerInputs(qh, kch, wh)
    ref, _ = api.run_materialize(inputs, dims)
    assert np.array_equal(idx.cpu().numpy(), ref.indices)
    assert np.array_equal(val.cpu().numpy().view(np.uint32), ref.values.view(np.uint32))
    row_properties(ref.indices[0], ref.values[0], 0, m, k)


def test_c4_rank_shard_properties_and_sampled_oracle_rows():
    """C4 (S=1,048,576, T=262,144, k=1024) as rank 0 of an 8-GPU run: the
    rank's LPT chunks with rank-local q / w (generated per chunk from the
    same counter-based streams as a full draw). Every row: the structural
    properties; sampled rows incl. the longest (t = S-1, 262,144 legal keys):
    the north-star rule against the oracle on the consumed bf16 operands."""
    from paper_2605_02568_b200.shard import plan_shards

    B, S, H, D, m, k, cs = 1, 1048576, 64, 128, 4, 1024, 1024
    T = S // m
    shards, _ = plan_shards(S, m, cs, 8)
    mine = shards[0]
    e = Engine(0)
    q = torch.cat([e.gen_normal_bf16(cs * H * D, D ** -0.5, 3, 1, s0 * H * D) for s0 in mine])
    w = torch.cat([e.gen_normal_f32(cs * H, (D * H) ** -0.5, 3, 3, s0 * H) for s0 in mine])
    kc = e.gen_normal_bf16(B * T * D, D ** -0.5, 3, 2)
    dims = api.ProblemDims.create(B, S, m, H, D, k)
    cfg = api.DriverConfig(tile=api.TileConfig(cs, T))
    idx, val, st = api.run_chunked_device(q, kc, w, dims, cfg, mine, local_rows=True)
    hi, hv = idx[0].cpu().numpy(), val[0].cpu().numpy()
    for c, s0 in enumerate(mine):
        row_properties(hi[c * cs:(c + 1) * cs], hv[c * cs:(c + 1) * cs], s0, m, k)
    assert S - cs in mine  # LPT hands rank 0 the heaviest chunk
    picks = [(mine.index(S - cs), cs - 1), (mine.index(S - cs), 17), (len(mine) // 2, 511), (len(mine) - 1, 0)]
    rows_t = [mine[c] + r for c, r in picks]
    local = [c * cs + r for c, r in picks]
    orc = Oracle()
    kcf = kc.float().view(-1, D).cpu().numpy()
    scores = []
    for t, lr in zip(rows_t, local):
        L = (t + 1) // m
        qrow = q[lr * H * D:(lr + 1) * H * D].float().view(H, D).cpu().numpy()
        wrow = w[lr * H:(lr + 1) * H].cpu().numpy()
        scores.append(orc.score_tile(qrow[None, None], kcf[None, :L], wrow[None, None], 0, 0, 1, L)[0, 0])
    rep = check_rows(hi[local], hv[local], scores, [(t + 1) // m for t in rows_t], k)
    assert rep["rows"] == len(rows_t)
