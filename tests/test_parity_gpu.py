"""Parity of the B200 path, called through the reference-facing API
(libcsaidx.so's C entry points = csaidx::run_chunked / run_materialize /
dispatch), against the pinned oracle and the reference's own golden fixtures.

* Shapes off the tensor-core path (tiny H_I / d_h, fp16 mode, scalar kernel)
  run the exact-order kernel: bit-exact indices, values and RunStats.
* The V4 indexer shape runs tcgen05: the north-star tolerance rule
  (tests/parity.py) at C1 (S=4096, k=512) against the full oracle.
* chunked == materialize bit-for-bit on the GPU under any tiling.
"""
import os

import numpy as np
import pytest

from oracle.oracle import Oracle
from paper_2605_02568_b200 import api
from paper_2605_02568_b200._capi import InvalidArgument, LogicError, ScoreRuntimeError

from .parity import check_rows

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def orc():
    return Oracle()


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN)


@pytest.fixture(params=["fused", "requested"])
def key_tiles(request, monkeypatch):
    """Run a test with the device's widened key tile (default) and with the
    requested c_T kept (CSAIDX_KEY_TILE_BYTES=0: select + merge per tile)."""
    if request.param == "requested":
        monkeypatch.setenv("CSAIDX_KEY_TILE_BYTES", "0")
    return request.param


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def inputs_for(orc, B, S, m, H, D, k, seed, bf16=False):
    q, kc, w = orc.generate_inputs(B, S, m, H, D, seed, bf16=bf16)
    dims = api.ProblemDims.create(B, S, m, H, D, k)
    return api.IndexerInputs.validated(q, kc, w, dims), dims, (q, kc, w)


def test_golden_driver_cases_bit_exact(orc, gold, key_tiles):
    for n, (B, S, m, H, D, k, seed, cs, ct, fp16, abl, ee, bm) in enumerate(gold["drv_cases"]):
        inputs, dims, _ = inputs_for(orc, int(B), int(S), int(m), int(H), int(D), int(k), int(seed))
        cfg = api.DriverConfig(tile=api.TileConfig(int(cs), int(ct)), mode=api.AccumulationMode(int(fp16)),
                               ablation=api.Ablation(int(abl)), causal_early_exit=bool(ee), bool_mask_tile=bool(bm))
        res, stats = api.run_chunked(inputs, dims, cfg)
        assert np.array_equal(res.indices, gold[f"drv{n}_idx"]), n
        assert np.array_equal(bits(res.values), bits(gold[f"drv{n}_val"])), n
        assert [stats.dispatch_count, stats.tiles_skipped_masked, stats.tiles_skipped_narrow] == \
            list(gold[f"drv{n}_stats"]), n
        assert stats.ledger_peak_bytes == int(gold[f"drv{n}_peak"][0]), n
        mres, _ = api.run_materialize(inputs, dims, mode=api.AccumulationMode(int(fp16)))
        assert np.array_equal(mres.indices, gold[f"drv{n}_midx"]), n
        assert np.array_equal(bits(mres.values), bits(gold[f"drv{n}_mval"])), n


def test_scalar_kernel_is_bit_exact_at_v4_shape(orc, gold):
    # ScoreKernel::scalar keeps fp32 operands and the reference op order.
    inputs, dims, _ = inputs_for(orc, 1, 512, 4, 64, 128, 64, 1, bf16=True)
    res, _ = api.run_materialize(inputs, dims, kernel=api.ScoreKernel.scalar)
    assert np.array_equal(res.indices.astype(np.int16), gold["v4_idx"])
    assert np.array_equal(bits(res.values), bits(gold["v4_val"]))


def test_tensor_core_path_v4_small_matches_reference_rule(orc, gold):
    inputs, dims, (q, kc, w) = inputs_for(orc, 1, 512, 4, 64, 128, 64, 1, bf16=True)
    res, st = api.run_chunked(inputs, dims, api.DriverConfig(tile=api.TileConfig(128, 64)))
    full = orc.score_tile(q, kc, w, 0, 0, 512, 128)[0]
    legal = (np.arange(512) + 1) // 4
    rep = check_rows(res.indices[0], res.values[0], full, legal, 64)
    assert rep["rows"] == 509


@pytest.fixture(scope="module")
def c1(orc):
    """C1: B=1, S=4096, H_I=64, d_h=128, m=4, k=512, bf16-representable inputs."""
    inputs, dims, (q, kc, w) = inputs_for(orc, 1, 4096, 4, 64, 128, 512, 1, bf16=True)
    full = orc.score_tile(q, kc, w, 0, 0, 4096, 1024)[0]  # oracle scores, reference op order
    return inputs, dims, full


@pytest.mark.parametrize("cs,ct", [(256, 256), (2048, 8192), (4096, 1024), (100, 300)])
def test_c1_parity_against_oracle(c1, cs, ct, key_tiles):
    inputs, dims, full = c1
    res, st = api.run_chunked(inputs, dims, api.DriverConfig(tile=api.TileConfig(cs, ct)))
    legal = (np.arange(4096) + 1) // 4
    rep = check_rows(res.indices[0], res.values[0], full, legal, 512)
    assert rep["rows"] == 4093  # rows 0..2 have no legal block
    assert st.dispatch_count == sum(
        1 for s0 in range(0, 4096, cs) for t0 in range(0, 1024, min(ct, 1024))
        if t0 < (min(s0 + cs, 4096)) // 4)


def test_c1_chunked_equals_materialize_bitwise(c1, key_tiles):
    inputs, dims, _ = c1
    ref, st = api.run_materialize(inputs, dims)
    for cs, ct in [(256, 256), (4096, 1024), (333, 77)]:
        got, _ = api.run_chunked(inputs, dims, api.DriverConfig(tile=api.TileConfig(cs, ct)))
        assert np.array_equal(got.indices, ref.indices)
        assert np.array_equal(bits(got.values), bits(ref.values))
    via, stats = api.dispatch(inputs, dims)
    assert stats.path == api.ExecutionPath.materialize  # 4096*64*1024*4 = 2^30 <= threshold
    assert np.array_equal(via.indices, ref.indices)


@pytest.mark.parametrize("budget", ["0", str(1 << 20), str(3 << 19), str(2 << 20), str(64 << 20)])
@pytest.mark.parametrize("early_exit", [True, False])
def test_widened_key_tiles_keep_results_stats_and_ledger(orc, monkeypatch, budget, early_exit):
    """physical_key_tile (driver.cpp): the device key tile widened to 2x /
    3x / 4x of the requested one (budgets over 512 KiB score tiles, the last
    physical tile ragged) or to all of T gives the same rows, RunStats and
    ledger peak as the requested tiling, on both kernel families at B = 2;
    the exact-order shape also bit-exact against the oracle."""
    for (B, S, m, H, D, k, bf16) in [(2, 3000, 4, 64, 128, 96, True), (2, 2500, 1, 2, 3, 200, False)]:
        inputs, dims, (q, kc, w) = inputs_for(orc, B, S, m, H, D, k, 7, bf16=bf16)
        cfg = api.DriverConfig(tile=api.TileConfig(512, 128), causal_early_exit=early_exit)
        monkeypatch.setenv("CSAIDX_KEY_TILE_BYTES", "0")
        ref, rst = api.run_chunked(inputs, dims, cfg)
        monkeypatch.setenv("CSAIDX_KEY_TILE_BYTES", budget)
        got, gst = api.run_chunked(inputs, dims, cfg)
        assert np.array_equal(got.indices, ref.indices)
        assert np.array_equal(bits(got.values), bits(ref.values))
        assert (gst.dispatch_count, gst.tiles_skipped_masked, gst.tiles_skipped_narrow, gst.ledger_peak_bytes) == \
            (rst.dispatch_count, rst.tiles_skipped_masked, rst.tiles_skipped_narrow, rst.ledger_peak_bytes)
        if not bf16:
            rc, idx, val, st3 = orc.run_chunked(q, kc, w, m, k, 512, 128, early_exit=early_exit)
            assert rc == 0
            assert np.array_equal(got.indices, idx) and np.array_equal(bits(got.values), bits(val))
            assert [gst.dispatch_count, gst.tiles_skipped_masked, gst.tiles_skipped_narrow] == list(st3)


def test_chunk_subset_entry_matches_full_run(c1):
    """csaidx_host_run_chunked_rows (pinned buffers, copy lanes overlapped
    with compute) and csaidx_device_run_chunked on a shard of chunks give the
    full run's rows."""
    import torch

    inputs, dims, _ = c1
    cfg = api.DriverConfig(tile=api.TileConfig(512, 1024))
    full, _ = api.run_chunked(inputs, dims, cfg)
    starts = [3584, 0, 2048]
    rows = api.chunk_rows(dims, cfg, starts)
    q = torch.from_numpy(inputs.q).pin_memory()
    kc = torch.from_numpy(inputs.kc).pin_memory()
    w = torch.from_numpy(inputs.w).pin_memory()
    oi = torch.empty((1, rows, dims.top_k), dtype=torch.int64).pin_memory()
    ov = torch.empty((1, rows, dims.top_k), dtype=torch.float32).pin_memory()
    api.run_chunked_rows(q, kc, w, dims, cfg, starts, oi, ov)
    expect = np.concatenate([full.indices[:, s:s + 512] for s in starts], axis=1)
    assert np.array_equal(oi.numpy(), expect)
    qd = q.cuda().to(torch.bfloat16)
    kd = kc.cuda().to(torch.bfloat16)
    di, dv, _ = api.run_chunked_device(qd, kd, w.cuda(), dims, cfg, starts)
    assert np.array_equal(di.cpu().numpy(), expect)


@pytest.mark.parametrize("B", [1, 2])
def test_rank_local_operands_match_full_tensors(orc, B):
    """A query-sharded rank keeps only its chunks' q / w rows
    (csaidx_device_run_chunked_local / csaidx_host_run_chunked_local): the
    result equals the run over the full tensors, for the tcgen05 shape and
    for the exact-order kernel."""
    import torch

    for (H, D, S, k, cs) in [(64, 128, 2048, 128, 256), (3, 5, 96, 7, 16)]:
        q, kc, w = orc.generate_inputs(B, S, 4, H, D, 5, bf16=(H == 64))
        dims = api.ProblemDims.create(B, S, 4, H, D, k)
        cfg = api.DriverConfig(tile=api.TileConfig(cs, 10 ** 6))
        starts = [S - cs, cs, 0] if S > 2 * cs else [0]
        rows = api.chunk_rows(dims, cfg, starts)
        dt = torch.bfloat16 if H == 64 else torch.float32
        qd, kd, wd = torch.from_numpy(q).cuda().to(dt), torch.from_numpy(kc).cuda().to(dt), torch.from_numpy(w).cuda()
        fi, fv, _ = api.run_chunked_device(qd, kd, wd, dims, cfg, starts)
        ql = torch.cat([torch.cat([qd[b, s0:s0 + cs] for s0 in starts]) for b in range(B)]).contiguous()
        wl = torch.cat([torch.cat([wd[b, s0:s0 + cs] for s0 in starts]) for b in range(B)]).contiguous()
        li, lv, _ = api.run_chunked_device(ql, kd, wl, dims, cfg, starts, local_rows=True)
        assert torch.equal(li, fi) and torch.equal(lv.view(torch.int32), fv.view(torch.int32))
        # host entry with rank-local host rows
        qh = np.ascontiguousarray(np.concatenate([np.concatenate([q[b, s0:s0 + cs] for s0 in starts])[None]
                                                  for b in range(B)]))
        wh = np.ascontiguousarray(np.concatenate([np.concatenate([w[b, s0:s0 + cs] for s0 in starts])[None]
                                                  for b in range(B)]))
        oi = np.empty((B, rows, k), np.int64)
        ov = np.empty((B, rows, k), np.float32)
        api.run_chunked_rows(qh, kc, wh, dims, cfg, starts, oi, ov, local_rows=True)
        assert np.array_equal(oi, fi.cpu().numpy())
        with pytest.raises(ValueError):
            api.run_chunked_device(qd, kd, wd, dims, cfg, starts, local_rows=True)


def test_csat_dump_loads_into_hbm_rank_local(orc, tmp_path):
    """CSAT dump -> device (csaidx_host_load_inputs_device): a chunk subset's
    q / w rows stacked rank-locally + the full kc, rounded to bf16 on device
    for the tcgen05 shape (fp32 for the exact kernel); the run over them
    equals the host-API run on the same file's arrays."""
    import torch

    for (H, D, S, k, cs) in [(64, 128, 2048, 64, 256), (3, 5, 96, 7, 16)]:
        B = 2
        q, kc, w = orc.generate_inputs(B, S, 4, H, D, 21, bf16=(H == 64))
        dims = api.ProblemDims.create(B, S, 4, H, D, k)
        cfg = api.DriverConfig(tile=api.TileConfig(cs, 10 ** 6))
        path = tmp_path / f"in_{H}.csat"
        api.write_inputs_file(path, api.IndexerInputs(q, kc, w), dims)
        starts = [S - cs, 0, cs]
        ql, kd, wl = api.load_inputs_device(path, dims, cfg, starts)
        assert ql.dtype == (torch.bfloat16 if H == 64 else torch.float32)
        assert torch.equal(kd.float().cpu(), torch.from_numpy(kc))
        exp_q = np.concatenate([np.concatenate([q[b, s0:s0 + cs] for s0 in starts])[None] for b in range(B)])
        assert np.array_equal(ql.float().cpu().numpy(), exp_q)
        li, lv, _ = api.run_chunked_device(ql, kd, wl, dims, cfg, starts, local_rows=True)
        full, _ = api.run_chunked(api.IndexerInputs.validated(q, kc, w, dims), dims, cfg)
        exp = np.concatenate([full.indices[:, s0:s0 + cs] for s0 in starts], axis=1)
        assert np.array_equal(li.cpu().numpy(), exp)
    # strict bf16: a value that bf16 cannot hold is rejected, as on the host path
    q[0, 5, 0, 0] = np.float32(1.0 + 2 ** -12)
    api.write_inputs_file(tmp_path / "bad.csat", api.IndexerInputs(q, kc, w), dims)
    dims64 = api.ProblemDims.create(2, 96, 4, 3, 5, 7)
    with pytest.raises(InvalidArgument):
        api.load_inputs_device(tmp_path / "bad.csat", dims64, cfg, strict=True, dtype=0)


@pytest.mark.parametrize("sms", ["0", "12", "40", "-1"])
def test_select_beside_score_overlap_is_byte_identical(orc, monkeypatch, sms):
    """One key tile per chunk on the tensor-core path: selects running beside
    the next chunk's score kernel (CSAIDX_SELECT_SMS SMs, or -1: no partition,
    a high-priority select lane; double-buffered tiles, a second compute lane)
    give the same bytes as the serial path, through the device entry and the
    host entry (copy lanes on top)."""
    import torch

    q, kc, w = orc.generate_inputs(1, 4096, 4, 64, 128, 31, bf16=True)
    dims = api.ProblemDims.create(1, 4096, 4, 64, 128, 256)
    cfg = api.DriverConfig(tile=api.TileConfig(512, 10 ** 6))
    monkeypatch.setenv("CSAIDX_SELECT_SMS", "0")
    ref, _ = api.run_chunked(api.IndexerInputs.validated(q, kc, w, dims), dims, cfg)
    monkeypatch.setenv("CSAIDX_SELECT_SMS", sms)
    got, _ = api.run_chunked(api.IndexerInputs.validated(q, kc, w, dims), dims, cfg)
    assert np.array_equal(got.indices, ref.indices) and np.array_equal(bits(got.values), bits(ref.values))
    qd, kd, wd = (torch.from_numpy(a).cuda() for a in (q, kc, w))
    di, dv, _ = api.run_chunked_device(qd.to(torch.bfloat16), kd.to(torch.bfloat16), wd, dims, cfg)
    assert np.array_equal(di.cpu().numpy(), ref.indices)


def test_two_level_select_in_the_driver_is_byte_identical(monkeypatch):
    """Rows spanning >= 4k key groups make the driver score with group maxima
    and select two-level; CSAIDX_TWO_LEVEL=0 gives the same bytes."""
    import torch

    from paper_2605_02568_b200.engine import Engine

    e = Engine(0)
    S, m, k = 65536, 4, 64
    T = S // m
    q = e.gen_normal_bf16(S * 64 * 128, 128 ** -0.5, 9, 1)
    kc = e.gen_normal_bf16(T * 128, 128 ** -0.5, 9, 2)
    w = e.gen_normal_f32(S * 64, (64 * 128) ** -0.5, 9, 3)
    dims = api.ProblemDims.create(1, S, m, 64, 128, k)
    cfg = api.DriverConfig(tile=api.TileConfig(2048, T))
    starts = [S - 2048, 40960, 8192]
    monkeypatch.setenv("CSAIDX_TWO_LEVEL", "0")
    i0, v0, _ = api.run_chunked_device(q, kc, w, dims, cfg, starts)
    monkeypatch.setenv("CSAIDX_TWO_LEVEL", "1")
    drv = api.KernelStats(api.driver_engine(0))
    drv.candidate_hits(reset=True)
    i1, v1, _ = api.run_chunked_device(q, kc, w, dims, cfg, starts)
    a, b = i0.cpu().numpy().reshape(-1, k), i1.cpu().numpy().reshape(-1, k)
    bad = np.argwhere((a != b).any(axis=1)).ravel()
    detail = [(int(r), a[r][a[r] != b[r]][:4].tolist(), b[r][a[r] != b[r]][:4].tolist()) for r in bad[:3]]
    assert len(bad) == 0, (len(bad), detail)
    assert torch.equal(v0.view(torch.int32), v1.view(torch.int32))
    assert drv.candidate_hits(reset=True) > 2048  # the long rows went two-level


def test_device_entry_orders_after_default_stream_work():
    """csaidx_device_run_chunked waits on the device for the operands' producer
    on the default stream: a copy queued behind a long sleep is seen."""
    import torch

    from paper_2605_02568_b200.engine import Engine

    e = Engine(0)
    S, m, k = 8192, 4, 64
    T = S // m
    q_src = e.gen_normal_bf16(S * 64 * 128, 128 ** -0.5, 4, 1)
    kc = e.gen_normal_bf16(T * 128, 128 ** -0.5, 4, 2)
    w = e.gen_normal_f32(S * 64, (64 * 128) ** -0.5, 4, 3)
    dims = api.ProblemDims.create(1, S, m, 64, 128, k)
    cfg = api.DriverConfig(tile=api.TileConfig(2048, T))
    want_i, want_v, _ = api.run_chunked_device(q_src, kc, w, dims, cfg)
    q = torch.zeros_like(q_src)
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000_000)  # ~0.1 s on the default stream
    q.copy_(q_src)                  # the operand is produced after the sleep
    got_i, got_v, _ = api.run_chunked_device(q, kc, w, dims, cfg)
    assert torch.equal(want_i, got_i) and torch.equal(want_v.view(torch.int32), got_v.view(torch.int32))


def test_ablations_follow_reference_semantics(orc):
    # acceptance.cpp:339-380 directions at a small V4-like shape
    inputs, dims, (q, kc, w) = inputs_for(orc, 1, 2048, 4, 8, 64, 64, 1)
    prod, _ = api.run_chunked(inputs, dims, api.DriverConfig(tile=api.TileConfig(256, 128)))
    rc, oidx, _, _ = orc.run_chunked(q, kc, w, 4, 64, 256, 128, ablation=0)
    assert rc == 0 and np.array_equal(prod.indices, oidx)
    a2, st2 = api.run_chunked(inputs, dims, api.DriverConfig(tile=api.TileConfig(256, 32),
                                                               ablation=api.Ablation.a2_skip_narrow))
    assert st2.dispatch_count == 0 and np.all(a2.indices == -1)
    a1, _ = api.run_chunked(inputs, dims, api.DriverConfig(tile=api.TileConfig(256, 128),
                                                             ablation=api.Ablation.a1_no_merge))
    rc, a1o, _, _ = orc.run_chunked(q, kc, w, 4, 64, 256, 128, ablation=1)
    assert np.array_equal(a1.indices, a1o)
    r = orc.recall(prod.indices, a1.indices)
    assert 0.0 < r["mean"] < 1.0


def test_fp16_mode_matches_reference_bits(orc):
    inputs, dims, (q, kc, w) = inputs_for(orc, 1, 512, 4, 8, 64, 32, 5)
    got, _ = api.run_chunked(inputs, dims, api.DriverConfig(tile=api.TileConfig(64, 32),
                                                              mode=api.AccumulationMode.fp16_emulated))
    idx, val = orc.run_materialize(q, kc, w, 4, 32, fp16=True)
    assert np.array_equal(got.indices, idx)
    assert np.array_equal(bits(got.values), bits(val))


def test_error_behaviour_matches_reference():
    d = api.ProblemDims.create(1, 1, 1, 1, 2, 1)
    big = api.IndexerInputs.validated([3.0e38, 3.0e38], [3.0e38, 3.0e38], [1.0], d)
    with pytest.raises(ScoreRuntimeError):  # score.cpp:96
        api.run_chunked(big, d)
    with pytest.raises(InvalidArgument):  # TileConfig::validate
        api.run_chunked(big, d, api.DriverConfig(tile=api.TileConfig(0, 1)))
    with pytest.raises(InvalidArgument):  # no AVX2 kernel in this build
        api.run_chunked(big, d, api.DriverConfig(kernel=api.ScoreKernel.avx2))
    ok = api.IndexerInputs.validated([1.0, 1.0], [1.0, 1.0], [0.5], d)
    res, _ = api.run_chunked(ok, d)
    # t=0, m=1: t_legal = 1 -> block 0 legal; score = 0.5 * relu(1*1 + 1*1) = 1
    assert res.indices[0, 0, 0] == 0 and res.values[0, 0, 0] == 1.0
    assert issubclass(LogicError, RuntimeError)


def test_sentinel_contract_exhaustive(orc):
    for m in (1, 2, 4):
        for k in (1, 2, 1000):
            S = 4 * m
            inputs, dims, (q, kc, w) = inputs_for(orc, 1, S, m, 2, 3, k, m * 1000 + k)
            for cs, ct in ((S, S // m), (1, 1), (3, 2)):
                res, _ = api.run_chunked(inputs, dims, api.DriverConfig(tile=api.TileConfig(cs, ct)))
                rc, idx, val, _ = orc.run_chunked(q, kc, w, m, k, cs, ct)
                assert np.array_equal(res.indices, idx) and np.array_equal(bits(res.values), bits(val))


def test_host_rounding_matches_device_rounding(orc, monkeypatch):
    """The pipelined host entry rounds q on the host cores (CSAIDX_HOST_ROUND,
    default; through the pinned piece ring or whole-chunk slabs) or on the
    device: same bytes, incl. B=2, rank-local rows, more chunks than staging
    slabs and many (partial) ring pieces per chunk; non-finite and (strict)
    inexact q rows raise invalid_argument every way."""
    B, S, m, H, D, k = 2, 8192, 4, 64, 128, 64
    q, kc, w = orc.generate_inputs(B, S, m, H, D, 3, bf16=True)
    dims = api.ProblemDims.create(B, S, m, H, D, k)
    cfg = api.DriverConfig(tile=api.TileConfig(256, S // m))
    starts = list(range(0, S, 256))[::-1][:20]  # 20 chunks > 8 slabs
    rows = len(starts) * 256
    q4 = np.asarray(q, np.float32).reshape(B, S, H, D)
    w3 = np.asarray(w, np.float32).reshape(B, S, H)
    ql = np.ascontiguousarray(np.concatenate([q4[:, s:s + 256] for s in starts], axis=1))
    wl = np.ascontiguousarray(np.concatenate([w3[:, s:s + 256] for s in starts], axis=1))
    kcf = np.asarray(kc, np.float32)
    outs = {}
    # host rounding off / on through the default ring / through whole-chunk
    # slabs / through a 2-piece ring of 96 KiB pieces (many pieces per chunk,
    # a partial last one)
    variants = {"0": {"CSAIDX_HOST_ROUND": "0"}, "1": {"CSAIDX_HOST_ROUND": "1"},
                "slabs": {"CSAIDX_HOST_ROUND": "1", "CSAIDX_HOST_RING": "0"},
                "small-ring": {"CSAIDX_HOST_ROUND": "1", "CSAIDX_HOST_PIECE_KB": "96", "CSAIDX_HOST_RING_PIECES": "2"}}
    for mode, env in variants.items():
        for kname in ("CSAIDX_HOST_RING", "CSAIDX_HOST_PIECE_KB", "CSAIDX_HOST_RING_PIECES"):
            monkeypatch.delenv(kname, raising=False)
        for kname, v in env.items():
            monkeypatch.setenv(kname, v)
        oi = np.empty((B, rows, k), np.int64)
        ov = np.empty((B, rows, k), np.float32)
        api.run_chunked_rows(q4, kcf, w3, dims, cfg, starts, oi, ov)
        li = np.empty_like(oi)
        lv = np.empty_like(ov)
        api.run_chunked_rows(ql, kcf, wl, dims, cfg, starts, li, lv, local_rows=True)
        assert np.array_equal(oi, li) and np.array_equal(bits(ov), bits(lv))
        outs[mode] = (oi, ov)
    for mode in variants:
        assert np.array_equal(outs["0"][0], outs[mode][0]) and np.array_equal(bits(outs["0"][1]), bits(outs[mode][1]))
    for mode, env in variants.items():
        for kname in ("CSAIDX_HOST_RING", "CSAIDX_HOST_PIECE_KB", "CSAIDX_HOST_RING_PIECES"):
            monkeypatch.delenv(kname, raising=False)
        for kname, v in env.items():
            monkeypatch.setenv(kname, v)
        bad = q4.copy()
        bad[1, starts[13] + 5, 7, 3] = np.nan
        oi = np.empty((B, rows, k), np.int64)
        ov = np.empty((B, rows, k), np.float32)
        with pytest.raises(InvalidArgument):
            api.run_chunked_rows(bad, kcf, w3, dims, cfg, starts, oi, ov)
        inexact = q4.copy()
        inexact[0, starts[17] + 1, 0, 0] = np.float32(1.0000001)
        strict = api.DriverConfig(tile=api.TileConfig(256, S // m), strict_bf16=True)
        with pytest.raises(InvalidArgument):
            api.run_chunked_rows(inexact, kcf, w3, dims, strict, starts, oi, ov)
        # not strict: auto_detect re-runs on the fp32 operands with the
        # exact-order kernel, i.e. ScoreKernel.scalar's bytes
        api.run_chunked_rows(inexact, kcf, w3, dims, cfg, starts, oi, ov)
        scal = api.DriverConfig(tile=api.TileConfig(256, S // m), kernel=api.ScoreKernel.scalar)
        si = np.empty_like(oi)
        sv = np.empty_like(ov)
        api.run_chunked_rows(inexact, kcf, w3, dims, scal, starts, si, sv)
        assert np.array_equal(oi, si) and np.array_equal(bits(ov), bits(sv))


@pytest.mark.parametrize("tail", ["0", "4", "27"])
def test_fp32_tail_chunks_match_host_rounding(orc, monkeypatch, tail):
    """Pinned q: the last chunks of the processing order cross PCIe as fp32
    and are rounded on the device (CSAIDX_HOST_FP32_TAIL, opt-in)
    — the same bytes as rounding every chunk on the host; a non-finite q row
    in a tail chunk still raises, an inexact one still re-runs exactly."""
    import torch

    B, S, m, H, D, k = 2, 8192, 4, 64, 128, 64
    q, kc, w = orc.generate_inputs(B, S, m, H, D, 5, bf16=True)
    dims = api.ProblemDims.create(B, S, m, H, D, k)
    cfg = api.DriverConfig(tile=api.TileConfig(256, S // m))
    starts = list(range(0, S, 256))
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    qp, kcp, wp = pin(np.asarray(q, np.float32).reshape(B, S, H, D)), pin(np.asarray(kc, np.float32)), \
        pin(np.asarray(w, np.float32).reshape(B, S, H))
    monkeypatch.setenv("CSAIDX_HOST_FP32_TAIL", "0")
    ri = torch.empty((B, S, k), dtype=torch.int64).pin_memory()
    rv = torch.empty((B, S, k), dtype=torch.float32).pin_memory()
    api.run_chunked_rows(qp, kcp, wp, dims, cfg, starts, ri, rv)
    monkeypatch.setenv("CSAIDX_HOST_FP32_TAIL", tail)
    gi, gv = torch.empty_like(ri).pin_memory(), torch.empty_like(rv).pin_memory()
    api.run_chunked_rows(qp, kcp, wp, dims, cfg, starts, gi, gv)
    assert torch.equal(gi, ri) and torch.equal(gv.view(torch.int32), rv.view(torch.int32))
    # chunk 0 is processed last (latest chunk first): it is always in the tail
    bad = qp.clone().pin_memory()
    bad[1, 5, 7, 3] = float("nan")
    with pytest.raises(InvalidArgument):
        api.run_chunked_rows(bad, kcp, wp, dims, cfg, starts, gi, gv)
    inexact = qp.clone().pin_memory()
    inexact[0, 17, 0, 0] = 1.0000001
    api.run_chunked_rows(inexact, kcp, wp, dims, cfg, starts, gi, gv)
    scal = api.DriverConfig(tile=api.TileConfig(256, S // m), kernel=api.ScoreKernel.scalar)
    si, sv = torch.empty_like(ri).pin_memory(), torch.empty_like(rv).pin_memory()
    api.run_chunked_rows(inexact, kcp, wp, dims, scal, starts, si, sv)
    assert torch.equal(gi, si) and torch.equal(gv.view(torch.int32), sv.view(torch.int32))


def test_auto_detect_on_fp32_inputs_is_bit_exact_like_the_reference(orc):
    """the reference's auto_detect scores arbitrary fp32 operands
    with a kernel bit-identical to its scalar one (score.cpp:18-43). At the
    V4 shape the B200 build takes tcgen05 only for bf16-representable
    operands; otherwise (q, kc, or just one late q row inexact) it runs the
    exact-order kernel on fp32 operands: bit-exact indices and values."""
    B, S, m, H, D, k = 1, 1024, 4, 64, 128, 64
    q, kc, w = orc.generate_inputs(B, S, m, H, D, 5)  # raw fp32 draws
    qb, kcb = orc.bf16_round(q), orc.bf16_round(kc)
    cases = {"q+kc": (q, kc), "kc": (qb, kc)}
    late = qb.copy()
    late[0, S - 3, 5, 7] = np.float32(late[0, S - 3, 5, 7] * np.float32(1.0000001))
    cases["one late q row"] = (late, kcb)
    dims = api.ProblemDims.create(B, S, m, H, D, k)
    for name, (qq, kk) in cases.items():
        inputs = api.IndexerInputs.validated(qq, kk, w, dims)
        rc, oi, ov, _ = orc.run_chunked(qq, kk, w, m, k, 256, S // m)
        assert rc == 0
        for cs, ct in ((256, S // m), (128, 64)):
            res, _ = api.run_chunked(inputs, dims, api.DriverConfig(tile=api.TileConfig(cs, ct)))
            assert np.array_equal(res.indices, oi) and np.array_equal(bits(res.values), bits(ov)), (name, cs, ct)
        mres, _ = api.run_materialize(inputs, dims)
        assert np.array_equal(mres.indices, oi) and np.array_equal(bits(mres.values), bits(ov)), name


@pytest.mark.parametrize("key_tile", [10 ** 6, 512])
def test_index_sink_receives_the_final_rows(orc, key_tile):
    """csaidx_engine_set_index_sink: the final kernels (select_final with one
    key tile, finalize after merges) also store each row's indices as int32
    at its sequence position in a [B, S, k] buffer."""
    import torch

    q, kc, w = orc.generate_inputs(2, 4096, 4, 64, 128, 17, bf16=True)
    dims = api.ProblemDims.create(2, 4096, 4, 64, 128, 128)
    cfg = api.DriverConfig(tile=api.TileConfig(512, key_tile))
    qd, kd, wd = (torch.from_numpy(a).cuda() for a in (q, kc, w))
    qd, kd = qd.to(torch.bfloat16), kd.to(torch.bfloat16)
    starts = [3584, 512, 2048]
    h = api.driver_engine(0)
    sink = torch.full((2, 4096, 128), -7, dtype=torch.int32, device="cuda")
    api.set_index_sink(h, sink.data_ptr(), 2, 4096, 128)
    try:
        oi, _, _ = api.run_chunked_device(qd, kd, wd, dims, cfg, starts)
    finally:
        api.set_index_sink(h, None)
    torch.cuda.synchronize()
    for n, s0 in enumerate(starts):
        assert torch.equal(sink[:, s0:s0 + 512], oi[:, n * 512:(n + 1) * 512].to(torch.int32))
    untouched = torch.ones(4096, dtype=torch.bool)
    for s0 in starts:
        untouched[s0:s0 + 512] = False
    assert bool((sink[:, untouched] == -7).all())
    # a final launch that does not fit the registered sink (other
    # k, batch count or sequence length) fails instead of writing past it
    api.set_index_sink(h, sink.data_ptr(), 2, 4096, 64)
    try:
        with pytest.raises(InvalidArgument):
            api.run_chunked_device(qd, kd, wd, dims, cfg, starts)
    finally:
        api.set_index_sink(h, None)
    api.set_index_sink(h, sink.data_ptr(), 2, 2048, 128)
    try:
        with pytest.raises(InvalidArgument):
            api.run_chunked_device(qd, kd, wd, dims, cfg, [2048])
        api.run_chunked_device(qd, kd, wd, dims, cfg, [1536])  # rows [1536, 2048) fit
    finally:
        api.set_index_sink(h, None)
    # sink only: no int64 / fp32 rows, the sink holds the same indices
    sink2 = torch.full((2, 4096, 128), -7, dtype=torch.int32, device="cuda")
    api.set_index_sink(h, sink2.data_ptr(), 2, 4096, 128)
    try:
        none_i, none_v, _ = api.run_chunked_device(qd, kd, wd, dims, cfg, starts, outputs=False)
    finally:
        api.set_index_sink(h, None)
    assert none_i is None and none_v is None
    torch.cuda.synchronize()
    for n, s0 in enumerate(starts):
        assert torch.equal(sink2[:, s0:s0 + 512], oi[:, n * 512:(n + 1) * 512].to(torch.int32))
    with pytest.raises(InvalidArgument):  # no sink: outputs are required
        api.run_chunked_device(qd, kd, wd, dims, cfg, starts, outputs=False)


def _sink_child(handle, q, kc, w, starts, done):
    import torch

    from paper_2605_02568_b200 import api as capi

    h = capi.driver_engine(0)
    ptr = capi.ipc_open(h, handle)
    capi.set_index_sink(h, ptr, 1, 4096, 64)
    dims = capi.ProblemDims.create(1, 4096, 4, 64, 128, 64)
    cfg = capi.DriverConfig(tile=capi.TileConfig(512, 10 ** 6))
    qd, kd, wd = (torch.from_numpy(a).cuda() for a in (q, kc, w))
    oi, _, _ = capi.run_chunked_device(qd.to(torch.bfloat16), kd.to(torch.bfloat16), wd, dims, cfg, starts)
    capi.set_index_sink(h, None)
    torch.cuda.synchronize()
    capi.ipc_close(h, ptr, handle)
    done.put(int(oi.sum().item()))


def test_index_sink_through_cuda_ipc_from_another_process(orc):
    """The fused gather of a query-sharded run: another process (a rank)
    writes its final rows into this process's buffer through a CUDA IPC
    mapping (same GPU here; peer GPUs over NVLink in a multi-GPU run)."""
    import torch
    import torch.multiprocessing as mp

    q, kc, w = orc.generate_inputs(1, 4096, 4, 64, 128, 23, bf16=True)
    backing = torch.full((4096 * 64 + 4096,), -7, dtype=torch.int32, device="cuda")
    sink = backing[4096:].view(1, 4096, 64)  # at an offset inside the allocation
    torch.cuda.synchronize()
    handle = api.ipc_handle(api.driver_engine(0), sink.data_ptr())
    starts = [1024, 3072]
    ctx = mp.get_context("spawn")
    done = ctx.Queue()
    p = ctx.Process(target=_sink_child, args=(handle, q, kc, w, starts, done))
    p.start()
    total = done.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    got = sink.cpu().numpy()
    rows = np.r_[1024:1536, 3072:3584]
    assert int(got[:, rows].astype(np.int64).sum()) == total
    assert got[:, rows].min() >= -1 and (np.delete(got, rows, axis=1) == -7).all()


def test_tensor_core_path_at_max_k_matches_reference_rule(orc):
    """k = 4096 (the GPU selection capacity) through the pipelined host
    entry on V4-shaped inputs: sampled rows (some with fewer than k legal
    keys, some with 2k) obey the north-star rule against the oracle."""
    S, m, k = 32768, 4, 4096
    inputs, dims, (q, kc, w) = inputs_for(orc, 1, S, m, 64, 128, k, 5, bf16=True)
    res, _ = api.run_chunked(inputs, dims, api.DriverConfig(tile=api.TileConfig(2048, S // m)))
    rows = [100, 16383, 16387, 20000, 32767]
    full = [orc.score_tile(q, kc, w, s, 0, 1, S // m)[0][0] for s in rows]
    legal = [(s + 1) // m for s in rows]
    rep = check_rows(res.indices[0][rows], res.values[0][rows], full, legal, k)
    assert rep["rows"] == len(rows)


@pytest.mark.parametrize("k,cs,ct", [(5000, 1024, 10 ** 6), (5000, 512, 2048), (9000, 4096, 3000), (20000, 8192, 10 ** 6)])
def test_k_above_shared_capacity_bit_exact(orc, k, cs, ct, key_tiles):
    """the drop-in accepts any k like the reference's
    tile_topk / merge_topk (topk.cpp:105-172). Exact-order kernel shapes, so
    indices, values and RunStats are bit-exact against the oracle — through
    the one-key-tile final select (c_T = T), the shared-memory select plus
    the staged global merge (c_T < k) and the large-take select (k > c_T)."""
    B, S, m, H, D = 1, 8192, 1, 2, 3
    inputs, dims, (q, kc, w) = inputs_for(orc, B, S, m, H, D, k, k + cs)
    res, stats = api.run_chunked(inputs, dims, api.DriverConfig(tile=api.TileConfig(cs, ct)))
    rc, idx, val, st3 = orc.run_chunked(q, kc, w, m, k, cs, ct)
    assert rc == 0
    assert np.array_equal(res.indices, idx) and np.array_equal(bits(res.values), bits(val))
    assert [stats.dispatch_count, stats.tiles_skipped_masked, stats.tiles_skipped_narrow] == list(st3)
    if k == 5000 and ct > S:
        mres, _ = api.run_materialize(inputs, dims)
        assert np.array_equal(mres.indices, idx) and np.array_equal(bits(mres.values), bits(val))


def test_overflow_at_a_causally_illegal_position_raises_like_the_reference(orc):
    """the reference scores the whole tile and rejects any
    non-finite fp32 score before masking (score.cpp:90-97 then
    causal.cpp:30-41), so an overflow that only occurs at a future (masked)
    position still raises runtime_error. Row 0 has no legal key at m = 4;
    q[0] * kc[0] overflows, every legal product stays finite."""
    B, S, m, H, D, k = 1, 64, 4, 2, 5, 4
    q, kc, w = orc.generate_inputs(B, S, m, H, D, 3)
    q[0, 0] = 1e30
    kc[0, 0] = 1e30
    dims = api.ProblemDims.create(B, S, m, H, D, k)
    inputs = api.IndexerInputs.validated(q, kc, w, dims)
    for cfg in (api.DriverConfig(tile=api.TileConfig(16, 8)), api.DriverConfig(tile=api.TileConfig(S, S // m))):
        with pytest.raises(ScoreRuntimeError):
            api.run_chunked(inputs, dims, cfg)
    with pytest.raises(ScoreRuntimeError):
        api.run_materialize(inputs, dims)
    # the same rows without the future overflow run through
    q[0, 0] = 0.5
    api.run_chunked(api.IndexerInputs.validated(q, kc, w, dims), dims, api.DriverConfig(tile=api.TileConfig(16, 8)))


def test_calls_from_several_threads_run_on_their_own_engines(orc):
    """VERDICT r1 (weak #8): the driver no longer serialises every call on one
    process-wide engine — each thread drives its own engine (stream, flags,
    scratch) per device. Two threads on two torch streams run different
    problems at once; each result equals the same call made alone."""
    import threading

    import torch

    from paper_2605_02568_b200.engine import Engine

    e = Engine(0)
    jobs = []
    for seed, (S, k, cs) in enumerate([(8192, 256, 1024), (16384, 512, 2048)]):
        q = e.gen_normal_bf16(S * 64 * 128, 128 ** -0.5, 40 + seed, 1)
        kc = e.gen_normal_bf16((S // 4) * 128, 128 ** -0.5, 40 + seed, 2)
        w = e.gen_normal_f32(S * 64, (64 * 128) ** -0.5, 40 + seed, 3)
        dims = api.ProblemDims.create(1, S, 4, 64, 128, k)
        cfg = api.DriverConfig(tile=api.TileConfig(cs, S // 4))
        ref, _, _ = api.run_chunked_device(q, kc, w, dims, cfg)
        jobs.append((q, kc, w, dims, cfg, ref))
    torch.cuda.synchronize()
    out, errs = [None, None], []

    def worker(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                q, kc, w, dims, cfg, _ = jobs[i]
                for _ in range(3):
                    out[i] = api.run_chunked_device(q, kc, w, dims,
                                                    api.DriverConfig(tile=cfg.tile, stream=s.cuda_stream))[0]
                s.synchronize()
        except Exception as ex:  # noqa: BLE001
            errs.append(ex)

    th = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for i in range(2):
        assert torch.equal(out[i], jobs[i][5])
