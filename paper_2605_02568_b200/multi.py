"""Python binding of the query-sharded multi-GPU driver (include/csaidx_host.h
csaidx_multi_*, C++ csaidx::gpu::MultiRank) and its transports.

One process per GPU. The library owns the LPT plan, the key broadcast from
rank 0, the peer mapping of rank 0's [B, S, k] int32 result (the final select
kernels store every rank's rows there over NVLink) or the collective gather,
and the end-of-step barrier. A transport is a ``csaidx_collectives`` table:

* ``NcclCollectives`` — NCCL (libnccl resolved by the library at run time);
  the 128-byte unique id travels over any channel (``nccl_unique_id`` on one
  rank, e.g. ``torch.distributed.broadcast_object_list`` to the others).
* ``TorchCollectives`` — host-staged callbacks over an initialised
  ``torch.distributed`` process group (gloo): the logic path on one GPU or
  on CPU-only hosts.

The reference runs the same loop on ``DriverConfig::threads`` host workers
(driver.cpp:115-165); ranks are GPUs here.
"""
from __future__ import annotations

import ctypes
from ctypes import CFUNCTYPE, POINTER, Structure, c_int, c_int64, c_size_t, c_uint64, c_void_p

import numpy as np

from . import _capi, api

GATHER_PEER, GATHER_COLLECTIVE = 0, 1

_BCAST = CFUNCTYPE(c_int, c_void_p, c_void_p, c_size_t, c_int, c_void_p)
_ALLGATHER = CFUNCTYPE(c_int, c_void_p, c_void_p, c_void_p, c_size_t)
_BARRIER = CFUNCTYPE(c_int, c_void_p, c_void_p)
_GATHERV = CFUNCTYPE(c_int, c_void_p, c_void_p, c_size_t, c_void_p, POINTER(c_size_t), POINTER(c_size_t), c_int,
                     c_void_p)


class CollectivesC(Structure):
    """csaidx_collectives (include/csaidx_cuda.h)."""

    _fields_ = [
        ("ctx", c_void_p),
        ("rank", c_int),
        ("world", c_int),
        ("device_buffers", c_int),
        ("bcast", _BCAST),
        ("allgather_host", _ALLGATHER),
        ("barrier", _BARRIER),
        ("gatherv", _GATHERV),
    ]


_SYMBOLS = {
    "csaidx_nccl_unique_id": (c_int, [c_void_p]),
    "csaidx_nccl_collectives_create": (c_int, [c_int, c_int, c_void_p, c_int, POINTER(POINTER(CollectivesC))]),
    "csaidx_nccl_collectives_destroy": (c_int, [POINTER(CollectivesC)]),
}
_HOST_SYMBOLS = {
    "csaidx_host_plan_shards": (c_int, [POINTER(_capi.Dims), c_int64, c_int, c_int, c_void_p, c_int64,
                                        POINTER(c_int64), c_void_p]),
    "csaidx_multi_create": (c_int, [POINTER(CollectivesC), POINTER(_capi.Dims), POINTER(api.RunConfig), c_int,
                                    c_void_p, POINTER(c_void_p)]),
    "csaidx_multi_chunks": (c_int, [c_void_p, POINTER(POINTER(c_int64)), POINTER(c_int64), POINTER(c_int64)]),
    "csaidx_multi_run": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                                 POINTER(api.RunStatsC)]),
    "csaidx_multi_destroy": (c_int, [c_void_p]),
}
_bound = False


def _libs():
    global _bound
    cuda, host = _capi.cuda_lib(), api.host_lib()
    if not _bound:
        for lib, table in ((cuda, _SYMBOLS), (host, _HOST_SYMBOLS)):
            for name, (res, args) in table.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
        _bound = True
    return cuda, host


def plan_shards(dims: api.ProblemDims, query_tile: int, world: int):
    """csaidx::gpu::plan_shards -> (per-rank ascending chunk starts, per-rank causal pairs per batch)."""
    _, host = _libs()
    cd = dims.c()
    loads = np.zeros(world, np.uint64)
    shards = []
    for r in range(world):
        n = c_int64()
        api._check(host.csaidx_host_plan_shards(ctypes.byref(cd), query_tile, world, r, None, 0, ctypes.byref(n),
                                                None))
        starts = np.zeros(max(n.value, 1), np.int64)
        api._check(host.csaidx_host_plan_shards(ctypes.byref(cd), query_tile, world, r, starts.ctypes.data,
                                                starts.size, ctypes.byref(n), loads.ctypes.data))
        shards.append([int(s) for s in starts[:n.value]])
    return shards, [int(x) for x in loads]


# ----------------------------------------------------------------- transports
def nccl_unique_id() -> bytes:
    cuda, _ = _libs()
    buf = ctypes.create_string_buffer(128)
    _capi.check(cuda.csaidx_nccl_unique_id(buf))
    return buf.raw


class NcclCollectives:
    """NCCL communicator of this rank (ncclCommInitRank on `device`)."""

    def __init__(self, rank: int, world: int, uid: bytes, device: int = 0):
        cuda, _ = _libs()
        self._lib = cuda
        ptr = POINTER(CollectivesC)()
        _capi.check(cuda.csaidx_nccl_collectives_create(rank, world, ctypes.create_string_buffer(uid, 128), device,
                                                         ctypes.byref(ptr)))
        self._ptr = ptr
        self.rank, self.world = rank, world

    @property
    def c(self):
        return self._ptr

    def close(self):
        if self._ptr:
            self._lib.csaidx_nccl_collectives_destroy(self._ptr)
            self._ptr = None


class TorchCollectives:
    """Host-staged transport over a torch.distributed process group (gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self._fns = (_BCAST(self._bcast), _ALLGATHER(self._allgather), _BARRIER(self._barrier),
                     _GATHERV(self._gatherv))
        self._struct = CollectivesC(None, self.rank, self.world, 0, *self._fns)

    @property
    def c(self):
        return ctypes.pointer(self._struct)

    @staticmethod
    def _view(ptr, n):
        import torch

        return torch.frombuffer((ctypes.c_uint8 * n).from_address(ptr), dtype=torch.uint8)

    def _bcast(self, ctx, buf, nbytes, root, stream):
        try:
            if nbytes:
                self.dist.broadcast(self._view(buf, nbytes), src=root, group=self.group)
            return 0
        except Exception:  # noqa: BLE001 — reported as a status across the C boundary
            return _capi.RUNTIME_ERROR

    def _allgather(self, ctx, inp, out, nbytes):
        import torch

        try:
            parts = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(self.world)]
            self.dist.all_gather(parts, self._view(inp, nbytes).clone(), group=self.group)
            dst = self._view(out, nbytes * self.world)
            for r, p in enumerate(parts):
                dst[r * nbytes:(r + 1) * nbytes] = p
            return 0
        except Exception:  # noqa: BLE001
            return _capi.RUNTIME_ERROR

    def _barrier(self, ctx, stream):
        try:
            self.dist.barrier(group=self.group)
            return 0
        except Exception:  # noqa: BLE001
            return _capi.RUNTIME_ERROR

    def _gatherv(self, ctx, send, send_bytes, recv, recv_bytes, recv_off, root, stream):
        import torch

        try:
            sizes = [int(recv_bytes[r]) for r in range(self.world)]
            pad = max(max(sizes), 1)
            mine = torch.zeros(pad, dtype=torch.uint8)
            if send_bytes:
                mine[:send_bytes] = self._view(send, send_bytes)
            parts = [torch.empty(pad, dtype=torch.uint8) for _ in range(self.world)] if self.rank == root else None
            self.dist.gather(mine, parts, dst=root, group=self.group)
            if self.rank == root:
                for r in range(self.world):
                    if sizes[r]:
                        self._view(recv + int(recv_off[r]), sizes[r])[:] = parts[r][:sizes[r]]
            return 0
        except Exception:  # noqa: BLE001
            return _capi.RUNTIME_ERROR

    def close(self):
        pass


# ----------------------------------------------------------------- the driver
class MultiRank:
    """csaidx_multi: one rank of a query-sharded run (include/csaidx_host.h)."""

    def __init__(self, comm, dims: api.ProblemDims, config: api.DriverConfig, gather: int = GATHER_PEER,
                 root_out=None):
        _, host = _libs()
        self._host, self.comm, self.dims, self.config = host, comm, dims, config
        self._cd, self._cc = dims.c(), config.c()
        h = c_void_p()
        ptr = c_void_p(root_out.data_ptr()) if root_out is not None else None
        api._check(host.csaidx_multi_create(comm.c, ctypes.byref(self._cd), ctypes.byref(self._cc), gather, ptr,
                                            ctypes.byref(h)))
        self._h = h
        starts, n, rows = POINTER(c_int64)(), c_int64(), c_int64()
        api._check(host.csaidx_multi_chunks(h, ctypes.byref(starts), ctypes.byref(n), ctypes.byref(rows)))
        self.chunks = [int(starts[i]) for i in range(n.value)]
        self.rows = rows.value

    def run(self, q, kc, w, local_idx=None, local_val=None):
        """q / w: this rank's rows (torch CUDA, chunks order); kc: [B, T, d_h]
        (read on rank 0, overwritten by the broadcast elsewhere)."""
        import torch

        dtype = _capi.DTYPE_BF16 if q.dtype == torch.bfloat16 else _capi.DTYPE_F32
        cur = torch.cuda.current_stream(q.device)
        if cur.cuda_stream != 0:
            cur.synchronize()
        st = api.RunStatsC()

        def p(t):
            return c_void_p(t.data_ptr()) if t is not None else None

        api._check(self._host.csaidx_multi_run(self._h, p(q), p(kc), dtype, p(w), p(local_idx), p(local_val),
                                               ctypes.byref(st)))
        return api.RunStats(st.dispatch_count, st.tiles_skipped_masked, st.tiles_skipped_narrow,
                            st.ledger_peak_bytes, st.device_peak_bytes, api.ExecutionPath.chunked)

    def close(self):
        if self._h:
            self._host.csaidx_multi_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
