"""The query-sharded multi-GPU driver (csaidx::gpu::MultiRank through
paper_2605_02568_b200/multi.py) running the real kernels, with two ranks that
share this box's one GPU (each its own process and CUDA context, a gloo
process group and the host-staged TorchCollectives transport), in both
gather modes:

* peer — the final select kernels of rank 1 store their int32 index rows into
  rank 0's [B, S, k] buffer through a CUDA IPC mapping (NVLink on a
  multi-GPU node);
* collective — the rows are gathered after the compute and scattered into
  sequence order on rank 0.

Rank 0's assembled [B, S, k] must equal, byte for byte, the single-GPU run of
the whole instance (and each rank's local rows its slice of it). The NCCL
transport is checked at world size 1 (the only size one GPU allows).
"""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu

B, S, H, D, M, K, CS = 2, 8192, 64, 128, 4, 512, 512


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _operands(e, chunks):
    """Rank-local stacks ([B, rows, ...] in chunks order) from the counter-based
    generator, so each rank's rows equal the same rows of a full draw."""
    q = torch.cat([e.gen_normal_bf16(min(CS, S - s0) * H * D, D ** -0.5, 13, 1, (b * S + s0) * H * D)
                   for b in range(B) for s0 in chunks])
    w = torch.cat([e.gen_normal_f32(min(CS, S - s0) * H, (D * H) ** -0.5, 13, 3, (b * S + s0) * H)
                   for b in range(B) for s0 in chunks])
    return q, w


def _worker(rank, world, port, gather, q_out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2605_02568_b200 import api, multi
    from paper_2605_02568_b200.engine import Engine

    ok = True
    try:
        e = Engine(0)
        dims = api.ProblemDims.create(B, S, M, H, D, K)
        cfg = api.DriverConfig(tile=api.TileConfig(CS, S // M))
        comm = multi.TorchCollectives()
        root = torch.full((B, S, K), -7, dtype=torch.int32, device="cuda") if rank == 0 else None
        mr = multi.MultiRank(comm, dims, cfg, gather, root)
        q, w = _operands(e, mr.chunks)
        kc = e.gen_normal_bf16(B * (S // M) * D, D ** -0.5, 13, 2) if rank == 0 else \
            torch.zeros(B * (S // M) * D, dtype=torch.bfloat16, device="cuda")
        li = torch.empty((B, mr.rows, K), dtype=torch.int64, device="cuda")
        lv = torch.empty((B, mr.rows, K), dtype=torch.float32, device="cuda")
        for _ in range(2):  # the mapping / buffers are reused across steps
            mr.run(q, kc, w, li, lv)
        torch.cuda.synchronize()
        # every rank: its local rows equal its slice of the single-GPU run
        qf = e.gen_normal_bf16(B * S * H * D, D ** -0.5, 13, 1)
        wf = e.gen_normal_f32(B * S * H, (D * H) ** -0.5, 13, 3)
        kf = e.gen_normal_bf16(B * (S // M) * D, D ** -0.5, 13, 2)
        ok &= bool(torch.equal(kc, kf))  # the key broadcast
        fi, fv, _ = api.run_chunked_device(qf, kf, wf, dims, cfg)
        r = 0
        for s0 in mr.chunks:
            n = min(CS, S - s0)
            ok &= bool(torch.equal(li[:, r:r + n], fi[:, s0:s0 + n]))
            ok &= bool(torch.equal(lv[:, r:r + n].view(torch.int32), fv[:, s0:s0 + n].view(torch.int32)))
            r += n
        if rank == 0:  # the assembled result: every rank's rows at their positions
            ok &= bool(torch.equal(root, fi.to(torch.int32)))
        if gather == 0:  # peer gather without local outputs: rank 0's rows are the only copy
            if rank == 0:
                root.fill_(-7)
            dist.barrier()
            mr.run(q, kc, w)
            torch.cuda.synchronize()
            if rank == 0:
                ok &= bool(torch.equal(root, fi.to(torch.int32)))
        mr.close()
    except Exception as ex:  # noqa: BLE001
        print(f"rank {rank}: {type(ex).__name__}: {ex}", flush=True)
        ok = False
    oks = [None] * world
    dist.all_gather_object(oks, bool(ok))
    if rank == 0:
        q_out.put(all(oks))
    dist.destroy_process_group()


@pytest.mark.parametrize("gather", [0, 1], ids=["peer", "collective"])
def test_two_ranks_on_one_gpu_assemble_the_single_gpu_result(gather):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, gather, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


@pytest.mark.parametrize("gather", [0, 1], ids=["peer", "collective"])
def test_nccl_transport_world_one(gather):
    from paper_2605_02568_b200 import api, multi
    from paper_2605_02568_b200.engine import Engine

    e = Engine(0)
    comm = multi.NcclCollectives(0, 1, multi.nccl_unique_id(), 0)
    try:
        dims = api.ProblemDims.create(B, S, M, H, D, K)
        cfg = api.DriverConfig(tile=api.TileConfig(CS, S // M))
        root = torch.full((B, S, K), -7, dtype=torch.int32, device="cuda")
        mr = multi.MultiRank(comm, dims, cfg, gather, root)
        assert mr.chunks == list(range(0, S, CS)) and mr.rows == S
        q, w = _operands(e, mr.chunks)
        kc = e.gen_normal_bf16(B * (S // M) * D, D ** -0.5, 13, 2)
        mr.run(q, kc, w)
        fi, _, _ = api.run_chunked_device(q, kc, w, dims, cfg)
        assert torch.equal(root, fi.to(torch.int32))
        mr.close()
    finally:
        comm.close()
