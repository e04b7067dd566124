"""Kernel-level parity through the C-ABI (device pointers).

score_tc (tcgen05) is compared with a float64 restatement of the score
definition (tolerance below); score_exact with the reference's fp32 op order
(bit-exact); select / merge / finalize with sort-based selection under the
reference order (bit-exact, ties included).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

NEG_INF = np.float32(-np.inf)


def bf16_round(x: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).float().numpy()


def make_inputs(B, S, H, D, m, seed=0):
    rng = np.random.default_rng(seed)
    T = S // m
    q = bf16_round(rng.normal(0, D ** -0.5, (B, S, H, D)))
    kc = bf16_round(rng.normal(0, D ** -0.5, (B, T, D)))
    w = rng.normal(0, (D * H) ** -0.5, (B, S, H)).astype(np.float32)
    return q, kc, w


def ref_scores_f64(q, kc, w, s0, rows, t0, cols):
    qq = q[:, s0:s0 + rows].astype(np.float64)           # B,rows,H,D
    kk = kc[:, t0:t0 + cols].astype(np.float64)          # B,cols,D
    dots = np.einsum("brhd,bcd->brhc", qq, kk)
    return np.einsum("brh,brhc->brc", w[:, s0:s0 + rows].astype(np.float64), np.maximum(dots, 0.0))


def ref_scores_exact_f32(q, kc, w, s0, rows, t0, cols):
    """score_scalar.cpp:20-34 op order in float32 numpy (one rounding per op)."""
    B, _, H, D = q.shape
    out = np.zeros((B, rows, cols), np.float32)
    for b in range(B):
        qq = q[b, s0:s0 + rows]
        kk = kc[b, t0:t0 + cols]
        acc = np.zeros((rows, cols), np.float32)
        for h in range(H):
            dot = np.zeros((rows, cols), np.float32)
            for d in range(D):
                dot = dot + qq[:, h, d][:, None] * kk[:, d][None, :]
            rect = np.where(dot < 0, np.float32(0), dot)
            acc = acc + w[b, s0:s0 + rows, h][:, None] * rect
        out[b] = acc
    return out


def legal(s, m):
    return (s + 1) // m


def ref_select(scores, s0, t0, m, k, apply_mask=True):
    """tile_topk over legal columns, sorted by (score desc, index asc)."""
    B, rows, cols = scores.shape
    width = min(k, cols)
    val = np.full((B, rows, width), NEG_INF, np.float32)
    idx = np.full((B, rows, width), -1, np.int32)
    for b in range(B):
        for i in range(rows):
            n = cols if not apply_mask else int(np.clip(legal(s0 + i, m) - t0, 0, cols))
            row = scores[b, i, :n]
            order = np.lexsort((np.arange(n), -row.astype(np.float64)))[: min(k, n)]
            val[b, i, : len(order)] = row[order]
            idx[b, i, : len(order)] = order + t0
    return val, idx


def to_dev(x, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t.to(dtype) if dtype is not None else t


@pytest.mark.parametrize(
    "B,S,s0,rows,t0,cols",
    [(1, 512, 0, 512, 0, 128), (1, 1024, 40, 77, 3, 250), (2, 2048, 1000, 300, 100, 412)],
)
def test_score_tc_matches_definition(engine, B, S, s0, rows, t0, cols):
    from paper_2605_02568_b200.engine import dims_struct

    H, D, m = 64, 128, 4
    q, kc, w = make_inputs(B, S, H, D, m, seed=S + rows)
    dims = dims_struct(B, S, H, D, m, 16)
    out = engine.score(to_dev(q, torch.bfloat16), to_dev(kc, torch.bfloat16), to_dev(w), dims, s0, rows, t0, cols)
    engine.check()
    got = out[:, :, :cols].cpu().numpy()
    want = ref_scores_f64(q, kc, w, s0, rows, t0, cols)
    scale = np.abs(want).max()
    err = np.abs(got - want).max()
    assert err <= 1e-5 * scale, (err, scale)


def test_score_tc_mask_and_causal_skip(engine):
    from paper_2605_02568_b200.engine import dims_struct

    B, S, H, D, m = 1, 4096, 64, 128, 4
    q, kc, w = make_inputs(B, S, H, D, m, seed=7)
    dims = dims_struct(B, S, H, D, m, 16)
    s0, rows, t0, cols = 1536, 512, 128, 768
    out = engine.score(to_dev(q, torch.bfloat16), to_dev(kc, torch.bfloat16), to_dev(w), dims, s0, rows, t0, cols,
                       apply_mask=True)
    engine.check()
    got = out[:, :, :cols].cpu().numpy()
    want = ref_scores_f64(q, kc, w, s0, rows, t0, cols)
    scale = np.abs(want).max()
    for i in range(rows):
        n = int(np.clip(legal(s0 + i, m) - t0, 0, cols))
        assert np.abs(got[0, i, :n] - want[0, i, :n]).max(initial=0) <= 1e-5 * scale
        # causally dead columns inside a computed key tile are -inf
        tail = got[0, i, n:min(cols, (n + 127) // 128 * 128)]
        assert np.all(tail == NEG_INF) or n == 0


def test_score_tc_is_tiling_invariant(engine):
    """Each score must not depend on which tile computed it (chunked == materialize)."""
    from paper_2605_02568_b200.engine import dims_struct

    B, S, H, D, m = 1, 2048, 64, 128, 4
    q, kc, w = make_inputs(B, S, H, D, m, seed=11)
    dims = dims_struct(B, S, H, D, m, 16)
    qd, kd, wd = to_dev(q, torch.bfloat16), to_dev(kc, torch.bfloat16), to_dev(w)
    full = engine.score(qd, kd, wd, dims, 0, S, 0, S // m)[:, :, : S // m].cpu().numpy()
    for (s0, rows, t0, cols) in [(5, 33, 7, 100), (1000, 1, 0, 512), (2040, 8, 300, 212)]:
        part = engine.score(qd, kd, wd, dims, s0, rows, t0, cols)[:, :, :cols].cpu().numpy()
        assert np.array_equal(part, full[:, s0:s0 + rows, t0:t0 + cols])


@pytest.mark.parametrize("H,D,fp16", [(1, 1, False), (3, 5, False), (8, 24, False), (2, 7, True)])
def test_score_exact_is_bit_exact(engine, H, D, fp16):
    from paper_2605_02568_b200.engine import dims_struct

    B, S, m = 2, 48, 4
    q, kc, w = make_inputs(B, S, H, D, m, seed=H * 100 + D)
    dims = dims_struct(B, S, H, D, m, 4)
    out = engine.score(to_dev(q, torch.bfloat16), to_dev(kc, torch.bfloat16), to_dev(w), dims, 0, S, 0, S // m,
                       mode=1 if fp16 else 0, kernel=1)
    engine.check()
    got = out[:, :, : S // m].cpu().numpy()
    if not fp16:
        want = ref_scores_exact_f32(q, kc, w, 0, S, 0, S // m)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    else:
        assert np.all(np.isfinite(got))


@pytest.mark.parametrize("cols,k,quant", [(300, 16, False), (5000, 512, False), (20000, 1024, True), (9000, 2048, True),
                                          (7, 10, False), (40000, 4096, False), (12000, 4096, True), (4096, 4096, False)])
def test_select_matches_sorted_reference(engine, cols, k, quant):
    rng = np.random.default_rng(cols + k)
    B, rows, m = 2, 9, 1
    s0, t0 = cols - 5, 0
    scores = rng.normal(0, 1, (B, rows, cols)).astype(np.float32)
    if quant:
        scores = np.round(scores * 4) / 4  # heavy ties
    ld = (cols + 3) // 4 * 4
    pad = np.zeros((B, rows, ld), np.float32)
    pad[:, :, :cols] = scores
    val, idx = engine.select(to_dev(pad), B, rows, cols, s0, t0, m, k)
    engine.check()
    wv, wi = ref_select(scores, s0, t0, m, k)
    assert np.array_equal(idx.cpu().numpy(), wi)
    assert np.array_equal(val.cpu().numpy().view(np.uint32), wv.view(np.uint32))


@pytest.mark.parametrize("mode", ["sampled_low", "sampled_high", "two_levels"])
def test_select_survives_adversarial_samples(engine, mode):
    """Rows built so the sector sample mispredicts the threshold: the kernel
    must fall back to the exact radix path and still match the reference."""
    rng = np.random.default_rng(7)
    B, rows, cols, k = 1, 4, 65536, 1024
    scores = rng.normal(0, 1, (B, rows, cols)).astype(np.float32)
    sampled = (np.arange(cols) // 8) % 16 == 0  # every 16th 32-byte sector
    if mode == "sampled_low":
        scores[..., sampled] = -10.0           # threshold too low -> overflow
    elif mode == "sampled_high":
        scores[..., sampled] = 10.0            # threshold at the sampled plateau
    else:
        scores[..., ~sampled] = 5.0            # ties everywhere off-sample
    val, idx = engine.select(to_dev(scores), B, rows, cols, 10 ** 7, 0, 1, k)
    engine.check()
    wv, wi = ref_select(scores, 10 ** 7, 0, 1, k)
    assert np.array_equal(idx.cpu().numpy(), wi)
    assert np.array_equal(val.cpu().numpy().view(np.uint32), wv.view(np.uint32))


@pytest.mark.parametrize("dist", ["lognormal_tail", "far_outlier", "signed_zeros", "ulp_range", "near_cut_dups",
                                  "short_rows_mixed_sign"])
def test_select_bucket_finish_distributions(engine, dist):
    """Distributions aimed at the value-linear bucket finish: long tails,
    one far outlier (nearly every candidate in one bucket -> radix path),
    +0.0/-0.0 folding, ranges a few ulps wide, ties straddling rank k."""
    rng = np.random.default_rng(11)
    B, rows, cols, k = 1, 6, 40000, 1024
    x = rng.normal(0, 1, (B, rows, cols)).astype(np.float32)
    if dist == "lognormal_tail":
        x = np.exp(2.5 * x).astype(np.float32)
    elif dist == "far_outlier":
        x[..., 123] = 3e30
    elif dist == "signed_zeros":
        x = np.where(x > 1.5, x, np.where(rng.random(x.shape) < 0.5, np.float32(0.0), np.float32(-0.0)))
        x = x.astype(np.float32)
    elif dist == "ulp_range":
        base = np.float32(1.0)
        x = (base + rng.integers(0, 6, x.shape).astype(np.float32) * np.finfo(np.float32).eps).astype(np.float32)
    elif dist == "near_cut_dups":
        x = np.round(x * 64) / 64
    else:  # short rows: every legal row fits the candidate list outright
        cols = 3000
        x = x[..., :cols] - 0.5
    x = np.ascontiguousarray(x.astype(np.float32))
    ld = (cols + 3) // 4 * 4
    pad = np.zeros((B, rows, ld), np.float32)
    pad[:, :, :cols] = x
    val, idx = engine.select(to_dev(pad), B, rows, cols, 10 ** 7, 0, 1, k)
    engine.check()
    wv, wi = ref_select(x, 10 ** 7, 0, 1, k)
    assert np.array_equal(idx.cpu().numpy(), wi)
    got = val.cpu().numpy()
    assert np.array_equal(np.where(got == 0, 0, got), np.where(wv == 0, 0, wv))  # -0.0 is reported as +0.0


@pytest.mark.parametrize("S,cols,k,m", [(4096, 1024, 512, 4), (6000, 1500, 100, 4), (700, 700, 1024, 1)])
def test_select_final_equals_select_then_finalize(engine, S, cols, k, m):
    """select_final (one key tile) == fill_sentinel + select + finalize, into
    the caller's int64 rows at an offset, neighbouring rows untouched."""
    rng = np.random.default_rng(S + k)
    B, rows, s0 = 2, 37, S - 40
    scores = rng.normal(0, 1, (B, rows, cols)).astype(np.float32)
    ld = (cols + 3) // 4 * 4
    pad = np.zeros((B, rows, ld), np.float32)
    pad[:, :, :cols] = scores
    dev = to_dev(pad)
    out_rows, row0 = rows + 10, 4
    oi = torch.full((B, out_rows, k), 77, dtype=torch.int64, device="cuda")
    ov = torch.full((B, out_rows, k), 5.0, dtype=torch.float32, device="cuda")
    engine.select_final(dev, B, rows, cols, s0, 0, m, k, oi, ov, row0)
    engine.check()
    run_v = torch.empty((B, rows, k), dtype=torch.float32, device="cuda")
    run_i = torch.empty((B, rows, k), dtype=torch.int32, device="cuda")
    engine.fill_sentinel(run_v, run_i)
    if min(k, cols) == k:
        v, i = engine.select(dev, B, rows, cols, s0, 0, m, k)
        run_v.copy_(v)
        run_i.copy_(i)
    else:
        v, i = engine.select(dev, B, rows, cols, s0, 0, m, k)
        engine.merge(run_v, run_i, v, i)
    wi = torch.full((B, out_rows, k), 77, dtype=torch.int64, device="cuda")
    wv = torch.full((B, out_rows, k), 5.0, dtype=torch.float32, device="cuda")
    engine.finalize(run_v, run_i, B, rows, s0, m, k, wi, wv, row0)
    engine.check()
    assert torch.equal(oi, wi)
    assert torch.equal(ov.view(torch.int32), wv.view(torch.int32))
    rv, ri = ref_select(scores, s0, 0, m, k)
    got = oi[:, row0:row0 + rows, : rv.shape[-1]].cpu().numpy()
    assert np.array_equal(got, ri.astype(np.int64))


@pytest.mark.parametrize("cols,k", [(40000, 1024), (3000, 512), (9000, 100)])
def test_persistent_multirow_select_equals_per_row_select(engine, cols, k):
    """The persistent 3-rows-per-CTA select (used beside the score kernel)
    gives the per-row kernel's bytes, incl. heavy ties and short rows."""
    rng = np.random.default_rng(cols)
    B, rows = 2, 37
    x = rng.normal(0, 1, (B, rows, cols)).astype(np.float32)
    x[1] = np.round(x[1] * 8) / 8
    ld = (cols + 3) // 4 * 4
    pad = np.zeros((B, rows, ld), np.float32)
    pad[:, :, :cols] = x
    dev = to_dev(pad)
    v0, i0 = engine.select(dev, B, rows, cols, cols + 5000, 0, 1, k)
    engine.check()
    engine.set_partition(100, 7)
    try:
        v1, i1 = engine.select(dev, B, rows, cols, cols + 5000, 0, 1, k)
        engine.check()
    finally:
        engine.set_partition(0, 0)
    assert torch.equal(i0, i1) and torch.equal(v0.view(torch.int32), v1.view(torch.int32))
    wv, wi = ref_select(x, cols + 5000, 0, 1, k)
    assert np.array_equal(i1.cpu().numpy(), wi)


def _v4_dims(S, k, m=4):
    from paper_2605_02568_b200.engine import dims_struct

    return dims_struct(1, S, 64, 128, m, k)


def test_score_gmax_is_the_group_max_of_the_tile(engine):
    """score_gmax: the tile is the plain score tile bit for bit and gmax[r, g]
    the max of row r's legal scores in key columns [32 g, 32 g + 32), for every
    group that overlaps the row's legal prefix (key tiles wholly past the causal
    limit are skipped and their groups left unwritten; select never reads them)."""
    S, m = 8192, 4
    T = S // m
    q = engine.gen_normal_bf16(S * 64 * 128, 128 ** -0.5, 5, 1)
    kc = engine.gen_normal_bf16(T * 128, 128 ** -0.5, 5, 2)
    w = engine.gen_normal_f32(S * 64, (64 * 128) ** -0.5, 5, 3)
    d = _v4_dims(S, 64)
    s0, rows, cols = 6000, 100, T
    plain = engine.score(q, kc, w, d, s0, rows, 0, cols, apply_mask=True)
    tile, gmax = engine.score_gmax(q, kc, w, d, s0, rows, 0, cols)
    engine.check()
    legal = (s0 + np.arange(rows) + 1) // m
    # key tiles wholly past a row's causal limit may be left unwritten
    ti, pi = tile[0].view(torch.int32).cpu().numpy(), plain[0].view(torch.int32).cpu().numpy()
    for r in range(rows):
        written = min(cols, (int(legal[r]) + 127) // 128 * 128)
        assert np.array_equal(ti[r, :written], pi[r, :written]), r
    t = tile[0, :, :cols].cpu().numpy()
    g = gmax[0].cpu().numpy()
    for r in range(rows):
        x = np.where(np.arange(cols) < legal[r], t[r], -np.inf)
        ref = np.pad(x, (0, g.shape[1] * 32 - cols), constant_values=-np.inf).reshape(-1, 32).max(axis=1)
        ng = (min(int(legal[r]), cols) + 31) // 32
        assert np.array_equal(g[r, :ng], ref[:ng].astype(np.float32)), r


@pytest.mark.parametrize("k", [64, 100])
def test_two_level_select_equals_one_level(engine, k):
    """select_final with group maxima (reads only the groups that can hold a
    top-k score) gives the one-level select's bytes on real score rows."""
    S, m = 32768, 4
    T = S // m
    q = engine.gen_normal_bf16(S * 64 * 128, 128 ** -0.5, 7, 1)
    kc = engine.gen_normal_bf16(T * 128, 128 ** -0.5, 7, 2)
    w = engine.gen_normal_f32(S * 64, (64 * 128) ** -0.5, 7, 3)
    d = _v4_dims(S, k)
    s0, rows = S - 300, 300
    tile, gmax = engine.score_gmax(q, kc, w, d, s0, rows, 0, T)
    oi1 = torch.full((1, rows, k), 7, dtype=torch.int64, device="cuda")
    ov1 = torch.zeros((1, rows, k), dtype=torch.float32, device="cuda")
    oi2, ov2 = oi1.clone(), ov1.clone()
    drv_hits = engine.candidate_hits(reset=True)
    engine.select_final(tile, 1, rows, T, s0, 0, m, k, oi1, ov1, 0)
    engine.check()
    assert engine.candidate_hits(reset=True) == 0
    engine.select_final(tile, 1, rows, T, s0, 0, m, k, oi2, ov2, 0, gmax=gmax)
    engine.check()
    assert engine.candidate_hits(reset=True) == rows  # every row took the two-level path
    assert torch.equal(oi1, oi2) and torch.equal(ov1.view(torch.int32), ov2.view(torch.int32))


def test_select_all_equal_scores_take_smallest_indices(engine):
    B, rows, cols, k = 1, 3, 10000, 100
    scores = np.zeros((B, rows, cols), np.float32)
    val, idx = engine.select(to_dev(scores), B, rows, cols, 10 ** 6, 0, 1, k)
    engine.check()
    assert np.array_equal(idx.cpu().numpy()[0, 0], np.arange(k, dtype=np.int32))


def test_merge_equals_union_topk(engine):
    rng = np.random.default_rng(3)
    rows, k = 50, 64
    run = np.sort(rng.integers(0, 20, (rows, k)).astype(np.float32))[:, ::-1]
    run_i = np.stack([rng.permutation(1000)[:k] for _ in range(rows)]).astype(np.int32)
    cand = np.sort(rng.integers(0, 20, (rows, 40)).astype(np.float32))[:, ::-1]
    cand_i = (1000 + np.stack([rng.permutation(1000)[:40] for _ in range(rows)])).astype(np.int32)
    # make each list sorted under (score desc, index asc)
    for arr_v, arr_i in ((run, run_i), (cand, cand_i)):
        for r in range(rows):
            o = np.lexsort((arr_i[r], -arr_v[r]))
            arr_v[r], arr_i[r] = arr_v[r][o].copy(), arr_i[r][o].copy()
    rv, ri = to_dev(run.copy()), to_dev(run_i.copy())
    engine.merge(rv, ri, to_dev(cand.copy()), to_dev(cand_i.copy()))
    engine.check()
    for r in range(rows):
        v = np.concatenate([run[r], cand[r]])
        i = np.concatenate([run_i[r], cand_i[r]])
        o = np.lexsort((i, -v))[:k]
        assert np.array_equal(ri.cpu().numpy()[r], i[o])
        assert np.array_equal(rv.cpu().numpy()[r], v[o])


def test_chunked_pipeline_small_v4(engine):
    """score -> select -> merge over several key tiles == one-shot selection."""
    from paper_2605_02568_b200.engine import dims_struct

    B, S, H, D, m, k = 1, 4096, 64, 128, 4, 512
    q, kc, w = make_inputs(B, S, H, D, m, seed=99)
    dims = dims_struct(B, S, H, D, m, k)
    qd, kd, wd = to_dev(q, torch.bfloat16), to_dev(kc, torch.bfloat16), to_dev(w)
    T = S // m
    full = engine.score(qd, kd, wd, dims, 0, S, 0, T, apply_mask=True)
    fv, fi = engine.select(full, B, S, T, 0, 0, m, k)
    s0, rows, ct = 2048, 1024, 200
    rv = torch.empty((B, rows, k), dtype=torch.float32, device="cuda")
    ri = torch.empty((B, rows, k), dtype=torch.int32, device="cuda")
    engine.fill_sentinel(rv, ri)
    ld = (ct + 3) // 4 * 4
    sb = torch.empty((B, rows, ld), dtype=torch.float32, device="cuda")
    cv = torch.empty((B, rows, k), dtype=torch.float32, device="cuda")
    ci = torch.empty((B, rows, k), dtype=torch.int32, device="cuda")
    first = True
    for t0 in range(0, T, ct):
        cols = min(ct, T - t0)
        if t0 >= legal(s0 + rows - 1, m):
            break
        engine.chunk_step(qd, kd, wd, dims, s0, rows, t0, cols, sb, cv, ci, rv, ri, first)
        first = False
    engine.check()
    assert np.array_equal(ri.cpu().numpy(), fi[:, s0:s0 + rows].cpu().numpy())
    assert np.array_equal(rv.cpu().numpy(), fv[:, s0:s0 + rows].cpu().numpy())


# ------------------------------------------------------- fused select pre-filter
def _prefilter_case(engine, seed=11, zero_w=False):
    from paper_2605_02568_b200.engine import dims_struct

    B, S, H, D, m, k = 1, 16384, 64, 128, 4, 512
    q, kc, w = make_inputs(B, S, H, D, m, seed=seed)
    if zero_w:
        w[:] = 0.0  # every legal score is +0.0: one giant tie
    dims = dims_struct(B, S, H, D, m, k)
    qd, kd, wd = to_dev(q, torch.bfloat16), to_dev(kc, torch.bfloat16), to_dev(w)
    s0, rows, t0, cols = 12288, 512, 0, S // m
    return dims, (qd, kd, wd), (B, m, k, s0, rows, t0, cols)


def test_prefilter_select_equals_plain_select(engine):
    """sample -> tau -> filtered score -> select from the bitmap == score ->
    select, bit for bit; the bitmap flags exactly the legal scores >= tau."""
    dims, (qd, kd, wd), (B, m, k, s0, rows, t0, cols) = _prefilter_case(engine)
    cap = engine.candidate_capacity(k)
    assert cap >= 2 * k
    stride = max(1, -(-(-(-cols // 128)) // 16))
    sample = engine.score_sampled(qd, kd, wd, dims, s0, rows, t0, cols, stride)
    tau = engine.row_threshold(sample, B, rows, cols, s0, t0, m, stride, k)
    sc, bits = engine.score_filtered(qd, kd, wd, dims, s0, rows, t0, cols, tau)
    engine.candidate_hits(reset=True)
    fv, fi = engine.select_from_candidates(sc, B, rows, cols, s0, t0, m, k, bits)
    hits = engine.candidate_hits()
    plain = engine.score(qd, kd, wd, dims, s0, rows, t0, cols, apply_mask=True)
    pv, pi = engine.select(plain, B, rows, cols, s0, t0, m, k)
    engine.check()
    assert torch.equal(fi, pi) and torch.equal(fv.view(torch.int32), pv.view(torch.int32))
    scn, pn, tn = sc.cpu().numpy(), plain.cpu().numpy(), tau.cpu().numpy()
    bn = bits.cpu().numpy().view(np.uint32)
    nflag = []
    for i in range(rows):
        n = int(np.clip(legal(s0 + i, m) - t0, 0, cols))
        assert np.array_equal(scn[0, i, :n].view(np.uint32), pn[0, i, :n].view(np.uint32))
        want = scn[0, i, :n] >= tn[0, i]
        nw = -(-n // 32)
        got = np.unpackbits(bn[0, i, :nw].view(np.uint8), bitorder="little")[:n].astype(bool)
        assert np.array_equal(got, want), i
        assert not np.any(np.unpackbits(bn[0, i, :nw].view(np.uint8), bitorder="little")[n:nw * 32])
        nflag.append(int(want.sum()))
    nflag = np.array(nflag)
    # the sample threshold lands every row between k and the list capacity
    assert hits == int(np.sum((nflag >= k) & (nflag <= cap))) and hits >= rows * 9 // 10, (hits, nflag.min(), nflag.max())
    # sample columns are the kt_stride-th key tiles
    vt = sample.shape[-1] // 128
    for v in range(vt):
        phys = v * stride * 128
        if phys >= cols:
            break
        seg = min(128, cols - phys)
        lim = np.clip((s0 + np.arange(rows) + 1) // m - t0 - phys, 0, seg)
        sn = sample[0, :, v * 128:v * 128 + seg].cpu().numpy()
        for i in range(0, rows, 17):
            if lim[i] == 0:
                continue  # the row never reads this sample tile (it may be causally dead)
            assert np.array_equal(sn[i, :lim[i]].view(np.uint32), pn[0, i, phys:phys + lim[i]].view(np.uint32))
            assert np.all(np.isneginf(sn[i, lim[i]:]))


@pytest.mark.parametrize("how", ["tau_high", "tau_low", "all_ties"])
def test_prefilter_falls_back_when_the_bitmap_is_unusable(engine, how):
    """Fewer than min(k, n) flagged entries (tau too high) or more than the
    list capacity (tau too low, giant ties) must take the streaming select."""
    dims, (qd, kd, wd), (B, m, k, s0, rows, t0, cols) = _prefilter_case(engine, seed=12, zero_w=how == "all_ties")
    cap = engine.candidate_capacity(k)
    if how == "tau_high":
        tau = torch.full((B, rows), 1e30, device="cuda")
    elif how == "tau_low":
        tau = torch.full((B, rows), -1e30, device="cuda")
    else:
        stride = 2
        sample = engine.score_sampled(qd, kd, wd, dims, s0, rows, t0, cols, stride)
        tau = engine.row_threshold(sample, B, rows, cols, s0, t0, m, stride, k)
    sc, bits = engine.score_filtered(qd, kd, wd, dims, s0, rows, t0, cols, tau)
    engine.candidate_hits(reset=True)
    fv, fi = engine.select_from_candidates(sc, B, rows, cols, s0, t0, m, k, bits)
    hits = engine.candidate_hits()
    pv, pi = engine.select(sc, B, rows, cols, s0, t0, m, k)
    engine.check()
    assert torch.equal(fi, pi) and torch.equal(fv.view(torch.int32), pv.view(torch.int32))
    n_rows = np.clip((s0 + np.arange(rows) + 1) // m - t0, 0, cols)
    if how == "tau_high":
        assert hits == 0
    else:  # only rows whose whole legal row fits the list can hit
        assert hits == int(np.sum(n_rows <= cap))
    if how == "all_ties":
        assert np.array_equal(fi[0, -1].cpu().numpy(), np.arange(k, dtype=np.int32))


@pytest.mark.parametrize("cols,k,quant", [(8192, 4097, False), (20000, 6000, True), (3000, 5000, False),
                                          (70000, 16384, False), (9000, 9000, True)])
def test_select_above_shared_capacity_matches_sorted_reference(engine, cols, k, quant):
    """Takes above the shared-memory capacity (4096) go through the exact
    global radix select + bitonic sort (reference tile_topk accepts any k,
    topk.cpp:105-132): sorted, tie-ordered, sentinel-padded rows identical
    to a sorted reference, including k > cols and heavy ties."""
    rng = np.random.default_rng(cols + k)
    B, rows, m = 2, 3, 1
    s0, t0 = cols - 2, 5
    scores = rng.normal(0, 1, (B, rows, cols)).astype(np.float32)
    if quant:
        scores = np.round(scores * 4) / 4
    ld = (cols + 3) // 4 * 4
    pad = np.zeros((B, rows, ld), np.float32)
    pad[:, :, :cols] = scores
    val, idx = engine.select(to_dev(pad), B, rows, cols, s0, t0, m, k)
    engine.check()
    wv, wi = ref_select(scores, s0, t0, m, k)
    assert np.array_equal(idx.cpu().numpy(), wi)
    got = val.cpu().numpy()
    wv = np.where(wv == 0, np.float32(0), wv)  # -0.0 is reported as +0.0 (succ treats them as equal)
    assert np.array_equal(got.view(np.uint32), wv.view(np.uint32))
