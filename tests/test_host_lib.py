"""CPU-only checks of the boundary libraries: both .so files load and export
every symbol their C headers declare, and the host-side arithmetic of the
drop-in API (byte models, dispatch counts, path choice, legality) matches the
reference's values (types.cpp, driver.cpp; known answers from test_types.cpp,
test_driver.cpp, acceptance.cpp). No GPU compute is invoked here.
"""
import ctypes
import os
import re

import numpy as np

import pytest

from paper_2605_02568_b200 import _capi, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(csaidx_\w+)\s*\(", src)))


@pytest.mark.parametrize("header,lib", [("csaidx_cuda.h", _capi.CUDA_LIB), ("csaidx_host.h", _capi.HOST_LIB)])
def test_library_exports_every_declared_symbol(header, lib):
    names = declared(header)
    assert len(names) > 8
    so = ctypes.CDLL(lib)
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, missing


def test_python_binding_covers_the_headers():
    from paper_2605_02568_b200 import multi

    assert set(declared("csaidx_cuda.h")) == set(_capi.CUDA_SYMBOLS) | set(multi._SYMBOLS)
    assert set(declared("csaidx_host.h")) == set(api.HOST_SYMBOLS) | set(multi._HOST_SYMBOLS)
    multi._libs()  # every binding resolves


def test_problem_dims_create_and_rejections():
    d = api.ProblemDims.create(1, 4096, 4, 64, 128, 512)
    assert (d.key_blocks, d.q_elems) == (1024, 4096 * 64 * 128)
    with pytest.raises(ValueError):
        api.ProblemDims.create(1, 10, 4, 1, 1, 1)  # S % m != 0 (types.cpp:54-56)
    with pytest.raises(ValueError):
        api.ProblemDims.create(0, 8, 4, 1, 1, 1)


def test_byte_models_match_reference_values():
    deploy = lambda s: api.ProblemDims.create(1, s, 4, 64, 128, 512)
    # acceptance.cpp:207-212
    assert api.materialize_bytes(deploy(65536)) == 274877906944
    assert api.materialize_bytes(deploy(131072)) == 1099511627776
    assert api.materialize_bytes(deploy(262144)) == 4398046511104
    # test_driver.cpp:264-279 (2048 * 64 * 512 * 4)
    path, pred = api.choose_path(api.ProblemDims.create(1, 2048, 4, 64, 128, 512), 1 << 30)
    assert path == api.ExecutionPath.materialize and pred == 268435456
    assert api.choose_path(api.ProblemDims.create(1, 8192, 4, 64, 128, 512), 1 << 30)[0] == api.ExecutionPath.chunked
    # bound for {128, 32}, k = 64: tile + scratch + run buffer (acceptance.cpp:248-284)
    assert api.chunked_peak_model_bytes(1, api.TileConfig(128, 32), 64, False) == 128 * 32 * 4 + 128 * 32 * 12 + 128 * 64 * 12
    assert api.chunked_peak_model_bytes(1, api.TileConfig(128, 32), 64, True) == 163840 + 128 * 32


def test_byte_model_overflow_is_overflow_error():
    huge = api.ProblemDims(batch=1 << 40, seq_len=1 << 40, key_blocks=1 << 30, heads=64, head_dim=1, ratio=1, top_k=1)
    with pytest.raises(OverflowError):
        api.materialize_bytes(huge)


def test_dispatch_count_model_values():
    # test_driver.cpp:130-142
    d = api.ProblemDims.create(1, 16384, 4, 2, 4, 512)
    assert [api.dispatch_count_model(d, api.TileConfig(2048, ct)) for ct in (1024, 1536, 2048, 4096)] == [32, 24, 16, 8]
    assert api.dispatch_count_model(d, api.TileConfig(2048, 40960)) == 8
    assert api.dispatch_count_model(d, api.TileConfig(163840, 40960)) == 1
    assert api.dispatch_count_model(api.ProblemDims.create(1, 10, 2, 1, 1, 1), api.TileConfig(4, 2)) == 9
    with pytest.raises(ValueError):
        api.dispatch_count_model(d, api.TileConfig(0, 1))


def test_legality_helpers():
    assert [api.t_legal(t, 4) for t in range(8)] == [0, 0, 0, 1, 1, 1, 1, 2]
    assert api.k_eff(4095, 4, 2000) == 1024
    with pytest.raises(ValueError):
        api.t_legal(-1, 4)


def test_no_gpu_means_loud_failure_not_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    d = api.ProblemDims.create(1, 8, 4, 1, 1, 1)
    inputs = api.IndexerInputs.validated([1.0] * 8, [1.0, 2.0], [1.0] * 8, d)
    with pytest.raises(_capi.CsaidxError):
        api.run_chunked(inputs, d)


@pytest.mark.parametrize("n", [37, 1_000_003])
def test_host_round_bf16_is_round_to_nearest_even(n):
    """csaidx_host_round_bf16 (the pipelined entry's host rounding) gives the
    bf16 bit patterns of torch's RNE conversion (== __float2bfloat16_rn on
    device) incl. ties, subnormals, signed zeros and overflow to inf."""
    import torch

    rng = np.random.default_rng(n)
    x = (rng.normal(0, 1, n) * np.exp2(rng.integers(-140, 120, n))).astype(np.float32)
    u = x.view(np.uint32)
    u[::7] = (u[::7] & 0xffff0000) | 0x8000          # exact ties, both lsb parities
    x[1::11] = np.float32(1.5e-41)                     # subnormal
    x[2::13] = np.float32(-0.0)
    x[3::17] = np.finfo(np.float32).max                # rounds up to inf
    got, nonfinite, inexact = api.round_bf16(x)
    want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, want)
    assert not nonfinite and inexact


def test_host_round_bf16_flags():
    exact = np.array([1.0, -2.5, 0.0, 3.0e38], np.float32)
    exact = (exact.view(np.uint32) & 0xffff0000).view(np.float32)
    _, nf, ix = api.round_bf16(exact)
    assert not nf and not ix
    bad = np.ones(100_000, np.float32)
    bad[77_777] = np.inf
    _, nf, _ = api.round_bf16(bad)
    assert nf
    bad[77_777] = np.nan
    _, nf, _ = api.round_bf16(bad)
    assert nf
