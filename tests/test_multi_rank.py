"""Host side of the query-sharded multi-GPU driver, on CPU (no GPU needed):

* the library's LPT plan (csaidx::gpu::plan_shards, C++) covers every chunk
  once, balances causal work, and equals an independent Python statement of
  the same rule;
* the torch.distributed transport (multi.TorchCollectives) behind the C
  table the driver calls — bcast, allgather_host, gatherv, barrier — moves
  the right bytes between two gloo ranks when invoked through its C function
  pointers, exactly as libcsaidx.so invokes it.
The GPU run of the driver itself (two ranks sharing one GPU, real kernels)
is tests/test_multi_gpu.py.
"""
import ctypes
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_02568_b200.shard import chunk_starts, chunk_work, plan_shards


def lpt_reference(S, m, cs, world):
    """The plan rule stated independently: chunks by decreasing causal work
    (ties: later chunk first), each to the least-loaded rank (ties: lowest)."""
    starts = list(range(0, S, min(cs, S)))
    cost = sorted(((chunk_work(S, m, cs, s), s) for s in starts), reverse=True)
    loads = [0] * world
    owned = [[] for _ in range(world)]
    for c, s in cost:
        r = min(range(world), key=lambda i: (loads[i], i))
        loads[r] += c
        owned[r].append(s)
    return [sorted(o) for o in owned], loads


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


def test_library_plan_equals_python_statement():
    for S, m, cs, world in [(262144, 4, 2048, 8), (1048576, 4, 1024, 8), (65536, 4, 2048, 3), (4096, 1, 512, 5),
                            (100, 4, 7, 4), (8192, 2, 8192, 2)]:
        assert plan_shards(S, m, cs, world) == lpt_reference(S, m, cs, world), (S, m, cs, world)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _transport_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_02568_b200.multi import TorchCollectives

    c = TorchCollectives()
    s = c._struct  # the table libcsaidx.so receives; call through its function pointers
    ok = s.rank == rank and s.world == world and s.device_buffers == 0
    # bcast: root 1's bytes land everywhere, in place
    buf = (ctypes.c_uint8 * 40)(*([rank * 7 + 1] * 40))
    ok &= s.bcast(None, ctypes.addressof(buf), 40, 1, None) == 0
    ok &= bytes(buf) == bytes([8] * 40)
    # allgather_host: rank r contributes 72 bytes of r
    blob = (ctypes.c_uint8 * 72)(*([rank + 3] * 72))
    out = (ctypes.c_uint8 * (72 * world))()
    ok &= s.allgather_host(None, ctypes.addressof(blob), ctypes.addressof(out), 72) == 0
    ok &= bytes(out) == b"".join(bytes([r + 3] * 72) for r in range(world))
    # gatherv: rank r sends 100 * (r + 1) bytes of value r + 10 -> root 0 at recv_off[r]
    sizes = [100 * (r + 1) for r in range(world)]
    offs = [sum(sizes[:r]) for r in range(world)]
    send = (ctypes.c_uint8 * sizes[rank])(*([rank + 10] * sizes[rank]))
    recv = (ctypes.c_uint8 * sum(sizes))()
    rb = (ctypes.c_size_t * world)(*sizes)
    ro = (ctypes.c_size_t * world)(*offs)
    ok &= s.gatherv(None, ctypes.addressof(send), sizes[rank], ctypes.addressof(recv), rb, ro, 0, None) == 0
    if rank == 0:
        ok &= bytes(recv) == b"".join(bytes([r + 10] * sizes[r]) for r in range(world))
    ok &= s.barrier(None, None) == 0
    oks = [None] * world
    dist.all_gather_object(oks, bool(ok))
    if rank == 0:
        q.put(all(oks))
    dist.destroy_process_group()


def test_torch_transport_through_its_c_table_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_transport_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True
