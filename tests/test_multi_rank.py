"""Host-side logic of the query-sharded multi-GPU path, on CPU with gloo
(world size 2): every chunk is owned by exactly one rank, LPT keeps the
causal work balanced, and the gathered per-rank rows reassemble into the
[S, k] output in sequence order. The same code (paper_2605_02568_b200/shard.py)
drives bench.py's NCCL run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_02568_b200.shard import assemble, chunk_starts, chunk_work, plan_shards, rows_of


def test_lpt_covers_and_balances():
    S, m, cs = 262144, 4, 2048
    for world in (1, 2, 4, 8):
        shards, loads = plan_shards(S, m, cs, world)
        flat = sorted(s for sh in shards for s in sh)
        assert flat == chunk_starts(S, cs)
        total = sum(chunk_work(S, m, cs, s) for s in flat)
        assert sum(loads) == total
        # within one chunk of perfect balance (contiguous blocks would give 1.875x at P=8)
        assert max(loads) - min(loads) <= max(chunk_work(S, m, cs, s) for s in flat)
        assert max(loads) / (total / world) < 1.02


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, S, cs, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shards, _ = plan_shards(S, 4, cs, world)
    mine = shards[rank]
    rows = rows_of(S, cs, mine)
    # stand-in for the device result: every packed row carries its global index
    part = np.zeros((1, rows, k), np.int64)
    r = 0
    for s0 in mine:
        n = min(cs, S - s0)
        part[0, r:r + n] = np.arange(s0, s0 + n)[:, None]
        r += n
    max_rows = torch.tensor([rows])
    dist.all_reduce(max_rows, op=dist.ReduceOp.MAX)
    send = torch.zeros((1, int(max_rows), k), dtype=torch.int64)
    send[:, :rows] = torch.from_numpy(part)
    kc = torch.arange(16, dtype=torch.float32) if rank == 0 else torch.zeros(16)
    dist.broadcast(kc, src=0)  # the key broadcast
    gathered = [torch.empty_like(send) for _ in range(world)] if rank == 0 else None
    dist.gather(send, gathered, dst=0)
    if rank == 0:
        full = assemble([g.numpy() for g in gathered], shards, S, cs)
        ok = bool(np.all(full[0, :, 0] == np.arange(S))) and bool(torch.equal(kc, torch.arange(16.0)))
        q.put(ok)
    dist.destroy_process_group()


def test_gloo_two_rank_gather_reassembles_sequence_order():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    S, cs, k = 8192, 512, 4
    procs = [ctx.Process(target=_worker, args=(r, 2, port, S, cs, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True
