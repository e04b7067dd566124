"""AccumulationMode::fp16_emulated on the tensor cores (CSAIDX_KERNEL_TENSOR /
gpu::Options::fp16_tensor_cores): the reference's binary16 rounding points
(score_scalar.cpp:29-32, half.cpp:84-91 — dot rounded to binary16 with
saturation, ReLU, acc = half(acc + w * r) in ascending h) applied to the MMA's
dot products. Only the dot product's summation order differs from the
reference, so scores agree to binary16 rounding: the test requires >= 99% of
tile entries bit-equal to the reference's fp16 scores and every other entry
within 4 binary16 ulps of its row's largest |score| (a one-ulp flip of one
head's dot or of a partial sum is an absolute error at the scale of the
partial sums, which cancellation can leave larger than the final value's own
ulp); at the driver level the index
sets are held to a recall bound (binary16 scores tie often, so a one-ulp
difference moves entries across the k-th place). The default auto_detect
path stays on the bit-exact CUDA-core kernel (tests/test_parity_gpu.py)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

MODE_FP16, KERNEL_TENSOR = 1, 2


@pytest.fixture(scope="module")
def orc():
    from oracle.oracle import Oracle
    return Oracle()


def _ulp16(x):
    """binary16 spacing at |x| (subnormal spacing below 2^-14)."""
    a = np.maximum(np.abs(x), 2.0 ** -14)
    return 2.0 ** (np.floor(np.log2(a)) - 10)


def test_fp16_tile_matches_reference_rounding(orc):
    from paper_2605_02568_b200.engine import Engine, dims_struct
    e = Engine(0)
    B, S, m, H, D, k = 1, 1024, 4, 64, 128, 64
    q, kc, w = orc.generate_inputs(B, S, m, H, D, 21, bf16=True)
    T = S // m
    dims = dims_struct(B, S, H, D, m, k)
    qt = torch.from_numpy(q).cuda().to(torch.bfloat16)
    kt = torch.from_numpy(kc).cuda().to(torch.bfloat16)
    wt = torch.from_numpy(w).cuda()
    for s0, rows, t0, cols in [(0, 256, 0, T), (512, 512, 0, T), (101, 37, 16, 131)]:  # + a partial item
        out = e.score(qt, kt, wt, dims, s0, rows, t0, cols, mode=MODE_FP16, kernel=KERNEL_TENSOR)
        e.check()
        got = out[:, :, :cols].cpu().numpy()
        ref = orc.score_tile(q, kc, w, s0, t0, rows, cols, fp16=True)
        same = got.view(np.uint32) == ref.view(np.uint32)
        assert same.mean() >= 0.99, same.mean()
        scale = _ulp16(np.abs(ref).max(axis=-1, keepdims=True))
        assert np.all(np.abs(got - ref) <= 4 * scale), (np.abs(got - ref) / scale).max()


def test_fp16_driver_on_tensor_cores_recall(orc):
    from paper_2605_02568_b200 import api
    B, S, m, H, D, k = 1, 2048, 4, 64, 128, 128
    q, kc, w = orc.generate_inputs(B, S, m, H, D, 5, bf16=True)
    dims = api.ProblemDims.create(B, S, m, H, D, k)
    cfg = api.DriverConfig(tile=api.TileConfig(512, S // m), mode=api.AccumulationMode.fp16_emulated,
                           fp16_tensor_cores=True)
    res, stats = api.run_chunked(api.IndexerInputs.validated(q, kc, w, dims), dims, cfg)
    rc, ref_idx, ref_val, _ = orc.run_chunked(q, kc, w, m, k, 512, S // m, fp16=True)
    assert rc == 0
    legal = (np.arange(S) + 1) // m
    rec = []
    for t in range(m, S):
        n = min(k, legal[t])
        a = set(res.indices[0, t, :n].tolist())
        b = set(ref_idx[0, t, :n].tolist())
        rec.append(len(a & b) / n)
        # the sentinel tail and the k_eff contract are the reference's
        assert np.all(res.indices[0, t, n:] == -1)
    rec = np.array(rec)
    assert rec.mean() >= 0.99 and rec.min() >= 0.9, (rec.mean(), rec.min())
    # values: the selected scores are binary16 values within 4 ulps of the reference's
    sel = res.values[0, m:, :]
    fin = np.isfinite(sel)
    assert np.all(np.float32(np.float16(sel[fin])) == sel[fin])


def test_fp16_default_stays_exact(orc):
    """Without the option, fp16_emulated keeps the bit-exact kernel on the V4 shape."""
    from paper_2605_02568_b200 import api
    B, S, m, H, D, k = 1, 256, 4, 64, 128, 16
    q, kc, w = orc.generate_inputs(B, S, m, H, D, 9, bf16=True)
    dims = api.ProblemDims.create(B, S, m, H, D, k)
    res, _ = api.run_chunked(api.IndexerInputs.validated(q, kc, w, dims), dims,
                             api.DriverConfig(tile=api.TileConfig(64, 64), mode=api.AccumulationMode.fp16_emulated))
    rc, ref_idx, ref_val, _ = orc.run_chunked(q, kc, w, m, k, 64, 64, fp16=True)
    assert rc == 0 and np.array_equal(res.indices, ref_idx)
    assert np.array_equal(res.values.view(np.uint32), ref_val.view(np.uint32))
