"""Python mirror of the reference driver API (proj/include/csaidx/driver.hpp,
types.hpp) over libcsaidx.so's C entry points (include/csaidx_host.h).

Same names, argument meaning and error behaviour as the C++ API:
``ProblemDims.create`` rejects bad extents with ``InvalidArgument``
(a ValueError), a non-finite fp32 score raises ``ScoreRuntimeError``, a
broken sentinel contract ``LogicError``. The compute runs on the B200; there
is no CPU path.
"""
from __future__ import annotations

import ctypes
import enum
import os
from ctypes import POINTER, Structure, c_char_p, c_int, c_int64, c_uint64, c_void_p
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import Dims, check as _check_cuda

SENTINEL_INDEX = -1
TOPK_ENTRY_BYTES = 12


class AccumulationMode(enum.IntEnum):
    fp32 = 0
    fp16_emulated = 1


class ScoreKernel(enum.IntEnum):
    auto_detect = 0
    scalar = 1
    avx2 = 2


class Ablation(enum.IntEnum):
    none = 0
    a1_no_merge = 1
    a2_skip_narrow = 2


class ExecutionPath(enum.IntEnum):
    materialize = 0
    chunked = 1


class RunConfig(Structure):
    """csaidx_run_config (include/csaidx_host.h)."""

    _fields_ = [
        ("query_tile", c_int64),
        ("key_tile", c_int64),
        ("mode", c_int),
        ("ablation", c_int),
        ("kernel", c_int),
        ("causal_early_exit", c_int),
        ("bool_mask_tile", c_int),
        ("threads", c_int),
        ("auto_threshold_bytes", c_uint64),
        ("device", c_int),
        ("strict_bf16", c_int),
        ("stream", c_void_p),
        ("fp16_tensor_cores", c_int),
    ]


class RunStatsC(Structure):
    _fields_ = [
        ("dispatch_count", c_int64),
        ("tiles_skipped_masked", c_int64),
        ("tiles_skipped_narrow", c_int64),
        ("ledger_peak_bytes", c_uint64),
        ("device_peak_bytes", c_uint64),
        ("path", c_int),
    ]


class SectionInfoC(Structure):
    _fields_ = [("tag", ctypes.c_uint8), ("rank", ctypes.c_uint8), ("dims", ctypes.c_uint32 * 4),
                ("elems", c_uint64), ("offset", c_uint64)]


_F = POINTER(ctypes.c_float)
HOST_SYMBOLS = {
    "csaidx_host_write_inputs_file": (c_int, [ctypes.c_char_p, c_void_p, c_void_p, c_void_p, POINTER(Dims),
                                              POINTER(c_uint64)]),
    "csaidx_host_scan_sections": (c_int, [ctypes.c_char_p, POINTER(SectionInfoC), c_int, POINTER(c_int)]),
    "csaidx_host_read_inputs": (c_int, [ctypes.c_char_p, POINTER(Dims), c_void_p, c_void_p, c_void_p]),
    "csaidx_host_load_inputs_device": (c_int, [ctypes.c_char_p, POINTER(Dims), c_int64, c_void_p, c_int64, c_int,
                                               c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "csaidx_host_last_error": (c_char_p, []),
    "csaidx_host_default_config": (None, [POINTER(RunConfig)]),
    "csaidx_host_engine": (c_int, [c_int, POINTER(c_void_p)]),
    "csaidx_host_run_chunked": (c_int, [c_void_p, c_void_p, c_void_p, POINTER(Dims), POINTER(RunConfig), c_void_p,
                                        c_void_p, POINTER(RunStatsC)]),
    "csaidx_host_run_materialize": (c_int, [c_void_p, c_void_p, c_void_p, POINTER(Dims), POINTER(RunConfig),
                                            c_void_p, c_void_p, POINTER(RunStatsC)]),
    "csaidx_host_dispatch": (c_int, [c_void_p, c_void_p, c_void_p, POINTER(Dims), POINTER(RunConfig), c_void_p,
                                     c_void_p, POINTER(RunStatsC)]),
    "csaidx_host_run_chunked_rows": (c_int, [c_void_p, c_void_p, c_void_p, POINTER(Dims), POINTER(RunConfig),
                                             c_void_p, c_int64, c_void_p, c_void_p, c_int64, POINTER(RunStatsC)]),
    "csaidx_host_run_chunked_local": (c_int, [c_void_p, c_void_p, c_void_p, POINTER(Dims), POINTER(RunConfig),
                                              c_void_p, c_int64, c_void_p, c_void_p, c_int64, POINTER(RunStatsC)]),
    "csaidx_device_run_chunked": (c_int, [c_void_p, c_void_p, c_int, c_void_p, POINTER(Dims), POINTER(RunConfig),
                                          c_void_p, c_int64, c_void_p, c_void_p, c_int64, POINTER(RunStatsC)]),
    "csaidx_device_run_chunked_local": (c_int, [c_void_p, c_void_p, c_int, c_void_p, POINTER(Dims),
                                                POINTER(RunConfig), c_void_p, c_int64, c_void_p, c_void_p, c_int64,
                                                POINTER(RunStatsC)]),
    "csaidx_host_problem_dims": (c_int, [c_int64] * 6 + [POINTER(Dims)]),
    "csaidx_host_dispatch_count_model": (c_int, [POINTER(Dims), c_int64, c_int64, POINTER(c_int64)]),
    "csaidx_host_chunked_peak_model_bytes": (c_int, [c_int64, c_int64, c_int64, c_int64, c_int, POINTER(c_uint64)]),
    "csaidx_host_materialize_bytes": (c_int, [POINTER(Dims), POINTER(c_uint64)]),
    "csaidx_host_choose_path": (c_int, [POINTER(Dims), c_uint64, POINTER(c_int), POINTER(c_uint64)]),
    "csaidx_host_t_legal": (c_int64, [c_int64, c_int64]),
    "csaidx_host_k_eff": (c_int64, [c_int64, c_int64, c_int64]),
    "csaidx_host_round_bf16": (c_int, [c_void_p, c_void_p, c_uint64, POINTER(c_int), POINTER(c_int)]),
    "csaidx_host_last_transfer": (c_int, [POINTER(c_uint64), POINTER(c_uint64), POINTER(c_int64), POINTER(c_int64)]),
}

_host = None


def host_lib():
    global _host
    if _host is None:
        _capi.cuda_lib()  # the driver library depends on it
        if not os.path.exists(_capi.HOST_LIB):
            raise ImportError(f"{_capi.HOST_LIB} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(_capi.HOST_LIB)
        for name, (res, args) in HOST_SYMBOLS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _host = lib
    return _host


def _check(rc: int) -> None:
    if rc != _capi.OK:
        msg = host_lib().csaidx_host_last_error().decode(errors="replace")
        raise _capi._ERRORS.get(rc, _capi.CsaidxError)(msg)


# ----------------------------------------------------------------- types


@dataclass
class ProblemDims:
    batch: int = 1
    seq_len: int = 1
    key_blocks: int = 1
    heads: int = 1
    head_dim: int = 1
    ratio: int = 1
    top_k: int = 1

    @staticmethod
    def create(batch, seq_len, ratio, heads, head_dim, top_k) -> "ProblemDims":
        d = Dims()
        _check(host_lib().csaidx_host_problem_dims(batch, seq_len, ratio, heads, head_dim, top_k, ctypes.byref(d)))
        return ProblemDims(d.batch, d.seq_len, d.key_blocks, d.heads, d.head_dim, d.ratio, d.top_k)

    def c(self) -> Dims:
        return Dims(self.batch, self.seq_len, self.key_blocks, self.heads, self.head_dim, self.ratio, self.top_k)

    @property
    def q_elems(self):
        return self.batch * self.seq_len * self.heads * self.head_dim

    @property
    def kc_elems(self):
        return self.batch * self.key_blocks * self.head_dim

    @property
    def w_elems(self):
        return self.batch * self.seq_len * self.heads


@dataclass
class TileConfig:
    query_tile: int = 2048
    key_tile: int = 8192


@dataclass
class DriverConfig:
    tile: TileConfig = field(default_factory=TileConfig)
    mode: AccumulationMode = AccumulationMode.fp32
    ablation: Ablation = Ablation.none
    kernel: ScoreKernel = ScoreKernel.auto_detect
    auto_threshold_bytes: int = 1 << 30
    causal_early_exit: bool = True
    bool_mask_tile: bool = False
    threads: int = 1
    # gpu::Options
    device: int = 0
    strict_bf16: bool = False
    stream: int = 0
    fp16_tensor_cores: bool = False

    def c(self) -> RunConfig:
        return RunConfig(self.tile.query_tile, self.tile.key_tile, int(self.mode), int(self.ablation),
                         int(self.kernel), int(self.causal_early_exit), int(self.bool_mask_tile), self.threads,
                         self.auto_threshold_bytes, self.device, int(self.strict_bf16), c_void_p(self.stream),
                         int(self.fp16_tensor_cores))


@dataclass
class RunStats:
    dispatch_count: int = 0
    tiles_skipped_masked: int = 0
    tiles_skipped_narrow: int = 0
    ledger_peak_bytes: int = 0
    device_peak_bytes: int = 0
    path: ExecutionPath = ExecutionPath.chunked


@dataclass
class IndexerInputs:
    q: np.ndarray   # [B, S, H, D] fp32
    kc: np.ndarray  # [B, T, D]
    w: np.ndarray   # [B, S, H]

    @staticmethod
    def validated(q, kc, w, dims: ProblemDims) -> "IndexerInputs":
        q = np.ascontiguousarray(q, dtype=np.float32).reshape(-1)
        kc = np.ascontiguousarray(kc, dtype=np.float32).reshape(-1)
        w = np.ascontiguousarray(w, dtype=np.float32).reshape(-1)
        for arr, n, name in ((q, dims.q_elems, "q"), (kc, dims.kc_elems, "kc"), (w, dims.w_elems, "w")):
            if arr.size != n:
                raise _capi.InvalidArgument(f"IndexerInputs: {name} extent mismatch")
        for arr, name in ((q, "q"), (kc, "kc"), (w, "w")):
            if not np.all(np.isfinite(arr)):
                raise _capi.InvalidArgument(f"IndexerInputs: non-finite entry in {name}")
        return IndexerInputs(q, kc, w)


@dataclass
class TopKResult:
    batch: int
    seq_len: int
    top_k: int
    indices: np.ndarray  # [B, S, k] int64
    values: np.ndarray   # [B, S, k] fp32

    @staticmethod
    def sized(dims: ProblemDims) -> "TopKResult":
        shape = (dims.batch, dims.seq_len, dims.top_k)
        return TopKResult(dims.batch, dims.seq_len, dims.top_k, np.full(shape, -1, np.int64),
                          np.full(shape, -np.inf, np.float32))

    def valid_count(self, b: int, t: int) -> int:
        row = self.indices[b, t]
        hits = np.flatnonzero(row == SENTINEL_INDEX)
        return int(hits[0]) if hits.size else self.top_k


def _ptr(a: np.ndarray):
    return c_void_p(a.ctypes.data)


def _host_call(fn, inputs: IndexerInputs, dims: ProblemDims, config: DriverConfig):
    for arr in (inputs.q, inputs.kc, inputs.w):
        if arr.dtype != np.float32 or not arr.flags["C_CONTIGUOUS"]:
            raise _capi.InvalidArgument("operands must be contiguous fp32 arrays")
    out = TopKResult.sized(dims)
    st = RunStatsC()
    cd, cc = dims.c(), config.c()
    _check(fn(_ptr(inputs.q), _ptr(inputs.kc), _ptr(inputs.w), ctypes.byref(cd), ctypes.byref(cc),
              _ptr(out.indices), _ptr(out.values), ctypes.byref(st)))
    stats = RunStats(st.dispatch_count, st.tiles_skipped_masked, st.tiles_skipped_narrow, st.ledger_peak_bytes,
                     st.device_peak_bytes, ExecutionPath(st.path))
    return out, stats


def run_chunked(inputs: IndexerInputs, dims: ProblemDims, config: DriverConfig | None = None):
    """driver.hpp:70-72 -> (TopKResult, RunStats)."""
    return _host_call(host_lib().csaidx_host_run_chunked, inputs, dims, config or DriverConfig())


def run_materialize(inputs: IndexerInputs, dims: ProblemDims, mode=AccumulationMode.fp32,
                    kernel=ScoreKernel.auto_detect, config: DriverConfig | None = None):
    """driver.hpp:77-79 -> (TopKResult, RunStats)."""
    cfg = config or DriverConfig()
    cfg = DriverConfig(**{**cfg.__dict__, "mode": mode, "kernel": kernel})
    return _host_call(host_lib().csaidx_host_run_materialize, inputs, dims, cfg)


def dispatch(inputs: IndexerInputs, dims: ProblemDims, config: DriverConfig | None = None):
    """driver.hpp:87-89 -> (TopKResult, RunStats with .path)."""
    return _host_call(host_lib().csaidx_host_dispatch, inputs, dims, config or DriverConfig())


def chunk_rows(dims: ProblemDims, config: DriverConfig, chunk_starts) -> int:
    cs = min(config.tile.query_tile, dims.seq_len)
    return int(sum(min(cs, dims.seq_len - int(s)) for s in chunk_starts))


def run_chunked_rows(q, kc, w, dims: ProblemDims, config: DriverConfig, chunk_starts, out_idx, out_val,
                     local_rows=False):
    """Host-buffer run over a chunk subset (csaidx_host_run_chunked_rows).

    q/kc/w/out_* are contiguous host arrays (numpy, or pinned torch CPU
    tensors); only the chunk rows of q/w are copied to the device.
    local_rows: q / w hold only those rows, stacked in chunk-list order
    (csaidx_host_run_chunked_local)."""
    starts = np.ascontiguousarray(chunk_starts, dtype=np.int64)
    st = RunStatsC()
    cd, cc = dims.c(), config.c()

    def ptr(a):
        return c_void_p(a.data_ptr()) if hasattr(a, "data_ptr") else _ptr(a)

    entry = host_lib().csaidx_host_run_chunked_local if local_rows else host_lib().csaidx_host_run_chunked_rows
    _check(entry(ptr(q), ptr(kc), ptr(w), ctypes.byref(cd), ctypes.byref(cc), _ptr(starts), starts.size,
                 ptr(out_idx), ptr(out_val), out_idx.shape[1], ctypes.byref(st)))
    return RunStats(st.dispatch_count, st.tiles_skipped_masked, st.tiles_skipped_narrow, st.ledger_peak_bytes,
                    st.device_peak_bytes, ExecutionPath.chunked)


# ---------------------------------------------------------------- CSAT input dump
def write_inputs_file(path, inputs: "IndexerInputs", dims: ProblemDims) -> int:
    """tensor_io.hpp write_inputs_file (csaidx_host_write_inputs_file); returns bytes written."""
    n = c_uint64(0)
    cd = dims.c()
    q, kc, w = (np.ascontiguousarray(a, np.float32) for a in (inputs.q, inputs.kc, inputs.w))
    _check(host_lib().csaidx_host_write_inputs_file(os.fsencode(path), _ptr(q), _ptr(kc), _ptr(w),
                                                    ctypes.byref(cd), ctypes.byref(n)))
    return n.value


def scan_sections(path):
    """Header scan with read_sections' checks: [(tag, rank, dims, elems, payload_offset)]."""
    buf = (SectionInfoC * 8)()
    n = c_int(0)
    _check(host_lib().csaidx_host_scan_sections(os.fsencode(path), buf, 8, ctypes.byref(n)))
    return [(s.tag, s.rank, tuple(s.dims[:s.rank]), s.elems, s.offset) for s in buf[:min(n.value, 8)]]


def read_inputs(path, dims: ProblemDims):
    """read_sections + shape check -> IndexerInputs-shaped host arrays (q, kc, w)."""
    q = np.empty((dims.batch, dims.seq_len, dims.heads, dims.head_dim), np.float32)
    kc = np.empty((dims.batch, dims.key_blocks, dims.head_dim), np.float32)
    w = np.empty((dims.batch, dims.seq_len, dims.heads), np.float32)
    cd = dims.c()
    _check(host_lib().csaidx_host_read_inputs(os.fsencode(path), ctypes.byref(cd), _ptr(q), _ptr(kc), _ptr(w)))
    return q, kc, w


def load_inputs_device(path, dims: ProblemDims, config: DriverConfig, chunk_starts=None, strict=False, device=0,
                       dtype=None):
    """CSAT dump -> torch CUDA tensors (csaidx_host_load_inputs_device): q / kc in the score
    kernel's operand type (bf16 for the tensor-core shape), w fp32; with chunk_starts only
    those query chunks' q / w rows, stacked for run_chunked_device(..., local_rows=True)."""
    import torch

    if dtype is None:
        cd0 = dims.c()
        kern = 0 if int(config.kernel) == 0 else 1  # ScoreKernel.auto_detect -> tcgen05 when the shape allows
        tc = _capi.cuda_lib().csaidx_cuda_score_uses_tensor_cores(ctypes.byref(cd0), _capi.DTYPE_BF16,
                                                                   int(config.mode), kern)
        dtype = _capi.DTYPE_BF16 if tc else _capi.DTYPE_F32
    rows = dims.seq_len
    starts = None
    n_chunks = 0
    if chunk_starts is not None:
        starts = np.ascontiguousarray(chunk_starts, dtype=np.int64)
        n_chunks = starts.size
        rows = chunk_rows(dims, config, chunk_starts)
    tdt = torch.bfloat16 if dtype == _capi.DTYPE_BF16 else torch.float32
    dev = torch.device("cuda", device)
    q = torch.empty((dims.batch, rows, dims.heads, dims.head_dim), dtype=tdt, device=dev)
    kc = torch.empty((dims.batch, dims.key_blocks, dims.head_dim), dtype=tdt, device=dev)
    w = torch.empty((dims.batch, rows, dims.heads), dtype=torch.float32, device=dev)
    torch.cuda.synchronize(dev)
    cd = dims.c()
    _check(host_lib().csaidx_host_load_inputs_device(
        os.fsencode(path), ctypes.byref(cd), config.tile.query_tile, None if starts is None else _ptr(starts),
        n_chunks, dtype, int(strict), device, c_void_p(q.data_ptr()), c_void_p(kc.data_ptr()),
        c_void_p(w.data_ptr())))
    return q, kc, w


def run_chunked_device(q, kc, w, dims: ProblemDims, config: DriverConfig, chunk_starts=None, out_idx=None,
                       out_val=None, local_rows=False, outputs=True):
    """Device-resident Algorithm 2 (csaidx_device_run_chunked): torch CUDA tensors in, torch tensors out.

    local_rows: q / w hold only the listed chunks' rows, stacked in list order
    (csaidx_device_run_chunked_local), as a query-sharded rank keeps them.
    outputs=False: no int64 / fp32 output rows (needs an index sink on the
    driver engine, set_index_sink, which then holds the only copy)."""
    import torch

    dtype = _capi.DTYPE_BF16 if q.dtype == torch.bfloat16 else _capi.DTYPE_F32
    # the entry orders itself after the legacy default stream; work on a
    # torch side stream has to be complete first
    cur = torch.cuda.current_stream(q.device)
    if cur.cuda_stream != 0:
        cur.synchronize()
    starts = None
    n_chunks = 0
    rows = dims.seq_len
    if chunk_starts is not None:
        starts = np.ascontiguousarray(chunk_starts, dtype=np.int64)
        n_chunks = starts.size
        cs = min(config.tile.query_tile, dims.seq_len)
        rows = int(sum(min(cs, dims.seq_len - int(s)) for s in starts))
    if out_idx is None and outputs:
        out_idx = torch.empty((dims.batch, rows, dims.top_k), dtype=torch.int64, device=q.device)
        out_val = torch.empty((dims.batch, rows, dims.top_k), dtype=torch.float32, device=q.device)
    st = RunStatsC()
    cd, cc = dims.c(), config.c()
    entry = host_lib().csaidx_device_run_chunked_local if local_rows else host_lib().csaidx_device_run_chunked
    if local_rows and (q.numel() != dims.batch * rows * dims.heads * dims.head_dim or
                       w.numel() != dims.batch * rows * dims.heads):
        raise ValueError("local_rows: q / w must hold exactly the listed chunks' rows")
    _check(entry(
        c_void_p(q.data_ptr()), c_void_p(kc.data_ptr()), dtype, c_void_p(w.data_ptr()), ctypes.byref(cd),
        ctypes.byref(cc), None if starts is None else _ptr(starts), n_chunks,
        c_void_p(out_idx.data_ptr()) if out_idx is not None else None,
        c_void_p(out_val.data_ptr()) if out_val is not None else None,
        out_idx.shape[1] if out_idx is not None else rows, ctypes.byref(st)))
    stats = RunStats(st.dispatch_count, st.tiles_skipped_masked, st.tiles_skipped_narrow, st.ledger_peak_bytes,
                     st.device_peak_bytes, ExecutionPath.chunked)
    return out_idx, out_val, stats


def driver_engine(device: int = 0):
    """Handle of the engine libcsaidx.so's driver uses on `device`."""
    h = c_void_p()
    _check(host_lib().csaidx_host_engine(device, ctypes.byref(h)))
    return h


def set_index_sink(engine, dst_ptr: int | None, batch: int = 0, seq_len: int = 0, k: int = 0):
    """csaidx_engine_set_index_sink: final rows are also stored as int32 into
    the [batch, seq_len, k] buffer at dst_ptr (possibly a peer GPU's, see
    ipc_open); None disables."""
    _check_cuda(_capi.cuda_lib().csaidx_engine_set_index_sink(engine, c_void_p(dst_ptr or 0), batch, seq_len, k))


def ipc_handle(engine, dev_ptr: int) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding dev_ptr, offset)."""
    buf = ctypes.create_string_buffer(64)
    off = c_uint64()
    _check_cuda(_capi.cuda_lib().csaidx_cuda_ipc_handle(engine, c_void_p(dev_ptr), buf, ctypes.byref(off)))
    return buf.raw, off.value


def ipc_open(engine, handle: tuple[bytes, int]) -> int:
    """Maps another process's allocation (peer access enabled lazily); the
    returned pointer addresses the same byte as the exporter's dev_ptr."""
    raw, off = handle
    ptr = c_void_p()
    _check_cuda(_capi.cuda_lib().csaidx_cuda_ipc_open(engine, ctypes.create_string_buffer(raw, 64), off,
                                                      ctypes.byref(ptr)))
    return ptr.value


def ipc_close(engine, dev_ptr: int, handle: tuple[bytes, int]):
    _check_cuda(_capi.cuda_lib().csaidx_cuda_ipc_close(engine, c_void_p(dev_ptr), handle[1]))


class KernelStats:
    """Launch counts / event-timed device ms per kernel class of an engine."""

    def __init__(self, handle):
        self.h = handle
        self.lib = _capi.cuda_lib()

    def profiling(self, on: bool):
        _check_cuda(self.lib.csaidx_engine_set_profiling(self.h, int(on)))

    def reset(self):
        _check_cuda(self.lib.csaidx_engine_reset_stats(self.h))

    def get(self, kind: int):
        n, ms = c_int64(), ctypes.c_double()
        _check_cuda(self.lib.csaidx_engine_kernel_stats(self.h, kind, ctypes.byref(n), ctypes.byref(ms)))
        return n.value, ms.value

    def select_fallbacks(self, reset: bool = False) -> int:
        n = c_int64()
        _check_cuda(self.lib.csaidx_engine_select_fallbacks(self.h, ctypes.byref(n), int(reset)))
        return n.value

    def candidate_hits(self, reset: bool = False) -> int:
        """Rows finished from the fused pre-filter's candidate lists."""
        n = c_int64()
        _check_cuda(self.lib.csaidx_engine_candidate_hits(self.h, ctypes.byref(n), int(reset)))
        return n.value

    def mem(self):
        live, peak = c_uint64(), c_uint64()
        _check_cuda(self.lib.csaidx_engine_mem_stats(self.h, ctypes.byref(live), ctypes.byref(peak)))
        return live.value, peak.value


# ------------------------------------------------------- host arithmetic


def t_legal(t: int, ratio: int) -> int:
    if t < 0 or ratio < 1:
        raise _capi.InvalidArgument("t_legal: t must be >= 0 and ratio >= 1")
    return int(host_lib().csaidx_host_t_legal(t, ratio))


def k_eff(t: int, ratio: int, top_k: int) -> int:
    if top_k < 0:
        raise _capi.InvalidArgument("k_eff: top_k must be >= 0")
    return int(host_lib().csaidx_host_k_eff(t, ratio, top_k))


def round_bf16(src: np.ndarray):
    """Host rounding of the pipelined entry (csaidx_host_round_bf16): fp32 ->
    bf16 bit patterns (uint16), plus the non-finite / inexact flags."""
    src = np.ascontiguousarray(src, dtype=np.float32)
    dst = np.empty(src.shape, dtype=np.uint16)
    nf, ix = ctypes.c_int(0), ctypes.c_int(0)
    _check(host_lib().csaidx_host_round_bf16(src.ctypes.data_as(c_void_p), dst.ctypes.data_as(c_void_p), src.size,
                                             ctypes.byref(nf), ctypes.byref(ix)))
    return dst, bool(nf.value), bool(ix.value)


def dispatch_count_model(dims: ProblemDims, tile: TileConfig) -> int:
    out = c_int64()
    cd = dims.c()
    _check(host_lib().csaidx_host_dispatch_count_model(ctypes.byref(cd), tile.query_tile, tile.key_tile,
                                                        ctypes.byref(out)))
    return out.value


def chunked_peak_model_bytes(batch: int, tile: TileConfig, top_k: int, bool_mask_tile: bool) -> int:
    out = c_uint64()
    _check(host_lib().csaidx_host_chunked_peak_model_bytes(batch, tile.query_tile, tile.key_tile, top_k,
                                                            int(bool_mask_tile), ctypes.byref(out)))
    return out.value


def materialize_bytes(dims: ProblemDims) -> int:
    out = c_uint64()
    cd = dims.c()
    _check(host_lib().csaidx_host_materialize_bytes(ctypes.byref(cd), ctypes.byref(out)))
    return out.value


def choose_path(dims: ProblemDims, threshold_bytes: int):
    path, pred = c_int(), c_uint64()
    cd = dims.c()
    _check(host_lib().csaidx_host_choose_path(ctypes.byref(cd), threshold_bytes, ctypes.byref(path),
                                              ctypes.byref(pred)))
    return ExecutionPath(path.value), pred.value


def last_transfer():
    """(h2d bytes, d2h bytes, chunks sent as fp32, chunks) of this thread's
    last host-buffer chunked call (csaidx_host_last_transfer)."""
    h, d, r, n = c_uint64(), c_uint64(), c_int64(), c_int64()
    _check(host_lib().csaidx_host_last_transfer(ctypes.byref(h), ctypes.byref(d), ctypes.byref(r), ctypes.byref(n)))
    return h.value, d.value, r.value, n.value
