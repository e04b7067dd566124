"""North-star parity at the BASELINE sizes, in GPUTEST.

Every config is held to tests/parity.py's rule (index sets bit-exact except
inside the 1e-5-relative k/k+1 tie band; mean recall 1.0000, min >= 0.998)
against the CPU oracle (reference op order) scored from the very bf16
operands the GPU consumed:

* a FULL-oracle V4 run whose rows are longer than the select's candidate
  capacity (S = 16,384, k = 512: rows of up to 4,096 keys vs capacity 2,048),
  every one of its 16,381 scored rows, under the production tiling
  (c_T = T: sample -> threshold -> stream -> gather -> bucket finish) and
  under a merge tiling (c_T = 1024);
* C2 (S = 65,536, k = 512), C3 (S = 262,144, k = 1024), C4 rank 0 of 8
  (S = 1,048,576, k = 1024, rank-local operands) and C5 (B = 2,
  S = 131,072) at every k of the sweep on a reduced (c_S, c_T) grid, on
  >= 256 stratified rows each (tests/scale_oracle.py), per batch;
* k = 4096 (the select's largest take) on V4 rows longer than its
  candidate capacity.

Recall statistics are printed per config and, with CSAIDX_PARITY_LOG set,
appended to that file as JSON lines.
"""
import numpy as np
import pytest
import torch

from oracle.oracle import Oracle
from paper_2605_02568_b200 import _capi, api
from paper_2605_02568_b200.engine import Engine

from .parity import check_rows
from .scale_oracle import check_sampled, record, stratified_rows

pytestmark = pytest.mark.gpu

H, D, M = 64, 128, 4


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def orc():
    return Oracle()


def cand_cap(k):
    return int(_capi.cuda_lib().csaidx_cuda_candidate_capacity(k))


def device_operands(B, S, seed):
    """Counter-based bf16 q / kc and fp32 w on the device (same distributions
    as the reference generator, synth.cpp:66-81)."""
    e = Engine(0)
    T = S // M
    q = e.gen_normal_bf16(B * S * H * D, D ** -0.5, seed, 1)
    kc = e.gen_normal_bf16(B * T * D, D ** -0.5, seed, 2)
    w = e.gen_normal_f32(B * S * H, (D * H) ** -0.5, seed, 3)
    torch.cuda.synchronize()
    return q, kc, w


@pytest.mark.parametrize("ct", [None, 1024])
def test_full_oracle_v4_rows_beyond_candidate_capacity(orc, ct):
    """Every row of a V4 instance whose long rows take the production
    sampled-threshold select, through the reference-facing host API."""
    B, S, k = 1, 16384, 512
    T = S // M
    assert T > cand_cap(k)  # rows t >= 4 * cap take the sampled path
    q, kc, w = orc.generate_inputs(B, S, M, H, D, 21, bf16=True)
    dims = api.ProblemDims.create(B, S, M, H, D, k)
    cfg = api.DriverConfig(tile=api.TileConfig(2048, ct or T))
    res, st = api.run_chunked(api.IndexerInputs.validated(q, kc, w, dims), dims, cfg)
    t = np.arange(S)
    legal = (t + 1) // M
    scores = orc.score_rows(q[0], w[0], kc[0], np.zeros(S, np.int64), legal)
    rep = check_rows(res.indices[0], res.values[0], scores, legal, k)
    assert rep["rows"] == S - (M - 1)
    rep.update(batch=0, label=f"full-oracle S={S} k={k} c_T={ct or T}", longest=int(legal.max()))
    record([rep])


def test_c2_stratified_oracle_rows(orc):
    B, S, k, cs = 1, 65536, 512, 2048
    q, kc, w = device_operands(B, S, 5)
    dims = api.ProblemDims.create(B, S, M, H, D, k)
    idx, val, _ = api.run_chunked_device(q, kc, w, dims, api.DriverConfig(tile=api.TileConfig(cs, S // M)))
    rows = stratified_rows(S, M, k, cand_cap(k), range(0, S, cs), cs, n=256, seed=2)
    assert len(rows) >= 256
    check_sampled(orc, q, kc, w, idx, val, dims, rows, label="C2 S=65536 k=512")


def test_c3_stratified_oracle_rows(orc):
    B, S, k, cs = 1, 262144, 1024, 2048
    q, kc, w = device_operands(B, S, 3)
    dims = api.ProblemDims.create(B, S, M, H, D, k)
    idx, val, _ = api.run_chunked_device(q, kc, w, dims, api.DriverConfig(tile=api.TileConfig(cs, S // M)))
    rows = stratified_rows(S, M, k, cand_cap(k), range(0, S, cs), cs, n=256, seed=3)
    assert len(rows) >= 256
    check_sampled(orc, q, kc, w, idx, val, dims, rows, label="C3 S=262144 k=1024")


def test_c4_rank0_of_8_stratified_oracle_rows(orc):
    """C4 as rank 0 of an 8-GPU run: the rank's LPT chunks, rank-local q / w."""
    from paper_2605_02568_b200.shard import plan_shards

    B, S, k, cs = 1, 1048576, 1024, 1024
    T = S // M
    shards, _ = plan_shards(S, M, cs, 8)
    mine = shards[0]
    e = Engine(0)
    q = torch.cat([e.gen_normal_bf16(cs * H * D, D ** -0.5, 3, 1, s0 * H * D) for s0 in mine])
    w = torch.cat([e.gen_normal_f32(cs * H, (D * H) ** -0.5, 3, 3, s0 * H) for s0 in mine])
    kc = e.gen_normal_bf16(B * T * D, D ** -0.5, 3, 2)
    torch.cuda.synchronize()
    dims = api.ProblemDims.create(B, S, M, H, D, k)
    idx, val, _ = api.run_chunked_device(q, kc, w, dims, api.DriverConfig(tile=api.TileConfig(cs, T)), mine,
                                         local_rows=True)
    pos = {s0: c for c, s0 in enumerate(mine)}
    owned = set(mine)
    rows = stratified_rows(S, M, k, cand_cap(k), mine, cs, n=256, seed=4, allowed=lambda t: (t // cs) * cs in owned)
    assert len(rows) >= 256 and S - 1 in rows
    check_sampled(orc, q, kc, w, idx, val, dims, rows, local=lambda t: pos[(t // cs) * cs] * cs + t % cs,
                  label="C4 rank 0/8 S=1048576 k=1024")


# C5 (B = 2, S = 131,072, T = 32,768): every k of the sweep, each on one
# (c_S, c_T) cell of the reduced grid, rotating through the grid's corners
C5_CELLS = [(256, 512, 4096), (512, 2048, 32768), (1024, 8192, 8192), (2048, 1024, 16384)]


@pytest.fixture(scope="module")
def c5_operands():
    return device_operands(2, 131072, 7)


@pytest.mark.parametrize("k,cs,ct", C5_CELLS)
def test_c5_sweep_cells_stratified_oracle_rows(orc, c5_operands, k, cs, ct):
    B, S = 2, 131072
    q, kc, w = c5_operands
    dims = api.ProblemDims.create(B, S, M, H, D, k)
    idx, val, _ = api.run_chunked_device(q, kc, w, dims, api.DriverConfig(tile=api.TileConfig(cs, ct)))
    rows = stratified_rows(S, M, k, cand_cap(k), range(0, S, cs), cs, n=256, seed=k)
    assert len(rows) >= 256
    check_sampled(orc, q, kc, w, idx, val, dims, rows, label=f"C5 k={k} c_S={cs} c_T={ct}")
    # tiling invariance of the sweep: the (2048, T) cell gives the same bytes
    if (cs, ct) != (2048, S // M):
        i2, v2, _ = api.run_chunked_device(q, kc, w, dims, api.DriverConfig(tile=api.TileConfig(2048, S // M)))
        assert torch.equal(idx, i2) and torch.equal(val.view(torch.int32), v2.view(torch.int32))


def test_k4096_rows_beyond_candidate_capacity_stratified(orc):
    B, S, k, cs = 1, 65536, 4096, 2048
    assert S // M > cand_cap(k)
    q, kc, w = device_operands(B, S, 11)
    dims = api.ProblemDims.create(B, S, M, H, D, k)
    idx, val, _ = api.run_chunked_device(q, kc, w, dims, api.DriverConfig(tile=api.TileConfig(cs, S // M)))
    rows = stratified_rows(S, M, k, cand_cap(k), range(0, S, cs), cs, n=256, seed=5)
    check_sampled(orc, q, kc, w, idx, val, dims, rows, label="V4 S=65536 k=4096")


def test_k8192_v4_stratified_oracle_rows(orc):
    """k above the shared-memory select (4096) at the V4 shape on the tensor-core
    path: the large-take select, held to the north-star rule."""
    B, S, k, cs = 1, 65536, 8192, 2048
    q, kc, w = device_operands(B, S, 12)
    dims = api.ProblemDims.create(B, S, M, H, D, k)
    idx, val, _ = api.run_chunked_device(q, kc, w, dims, api.DriverConfig(tile=api.TileConfig(cs, S // M)))
    rows = stratified_rows(S, M, k, 2 * k, range(0, S, cs), cs, n=256, seed=6)
    check_sampled(orc, q, kc, w, idx, val, dims, rows, label="V4 S=65536 k=8192")
