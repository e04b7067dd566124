"""Device-level handle over the C-ABI: one engine per GPU.

Tensors are torch CUDA tensors (PyTorch is used for device memory and
streams only); every compute call goes through libcsaidx_cuda.so.
"""
from __future__ import annotations

import ctypes
from ctypes import byref, c_int, c_int64, c_uint64, c_void_p

import torch

from . import _capi
from ._capi import Dims, check

NEG_INF = float("-inf")


def dims_struct(batch, seq_len, heads, head_dim, ratio, top_k, key_blocks=None) -> Dims:
    if key_blocks is None:
        key_blocks = seq_len // ratio
    return Dims(batch, seq_len, key_blocks, heads, head_dim, ratio, top_k)


def _dtype(t):
    if t.dtype == torch.bfloat16:
        return _capi.DTYPE_BF16
    if t.dtype == torch.float32:
        return _capi.DTYPE_F32
    raise TypeError(f"q/kc must be bf16 or fp32, got {t.dtype}")


def _p(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


class Engine:
    """Wraps csaidx_engine (include/csaidx_cuda.h)."""

    def __init__(self, device: int = 0, use_torch_stream: bool = True):
        self.lib = _capi.cuda_lib()
        self.device = device
        h = c_void_p()
        check(self.lib.csaidx_engine_create(device, byref(h)))
        self.handle = h
        if use_torch_stream:
            self.use_stream(torch.cuda.current_stream(device))

    def close(self):
        if self.handle:
            self.lib.csaidx_engine_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass

    def use_stream(self, stream: torch.cuda.Stream | None):
        """Enqueue on a torch stream (None: the engine's own stream)."""
        if stream is None:
            check(self.lib.csaidx_engine_use_own_stream(self.handle))
        else:
            check(self.lib.csaidx_engine_set_stream(self.handle, c_void_p(stream.cuda_stream)))

    @property
    def num_sms(self) -> int:
        n = c_int()
        check(self.lib.csaidx_engine_num_sms(self.handle, byref(n)))
        return n.value

    def check(self):
        check(self.lib.csaidx_engine_check(self.handle))

    def mem_stats(self):
        live, peak = c_uint64(), c_uint64()
        check(self.lib.csaidx_engine_mem_stats(self.handle, byref(live), byref(peak)))
        return live.value, peak.value

    # ------------------------------------------------------------ operands
    def to_bf16(self, src: torch.Tensor, strict: bool = False) -> torch.Tensor:
        assert src.dtype == torch.float32 and src.is_cuda and src.is_contiguous()
        dst = torch.empty(src.shape, dtype=torch.bfloat16, device=src.device)
        check(self.lib.csaidx_cuda_to_bf16(self.handle, _p(src), _p(dst), src.numel(), int(strict)))
        return dst

    def gen_normal_bf16(self, n: int, stddev: float, seed: int, stream_id: int, offset: int = 0) -> torch.Tensor:
        out = torch.empty(n, dtype=torch.bfloat16, device=f"cuda:{self.device}")
        check(self.lib.csaidx_cuda_gen_normal_bf16(self.handle, _p(out), n, stddev, seed, stream_id, offset))
        self.check()  # the tensor may be handed to torch or another engine next
        return out

    def gen_normal_f32(self, n: int, stddev: float, seed: int, stream_id: int, offset: int = 0) -> torch.Tensor:
        out = torch.empty(n, dtype=torch.float32, device=f"cuda:{self.device}")
        check(self.lib.csaidx_cuda_gen_normal_f32(self.handle, _p(out), n, stddev, seed, stream_id, offset))
        self.check()
        return out

    # ------------------------------------------------------------ hot path
    def score(self, q, kc, w, dims: Dims, s0, rows, t0, cols, mode=0, kernel=0, apply_mask=False, out=None):
        ld = (cols + 3) // 4 * 4
        if out is None:
            out = torch.empty((dims.batch, rows, ld), dtype=torch.float32, device=q.device)
        else:
            ld = out.shape[-1]
        check(self.lib.csaidx_cuda_score(self.handle, _p(q), _p(kc), _dtype(q), _p(w), byref(dims), s0, rows, t0,
                                         cols, mode,
                                         kernel, int(apply_mask), _p(out), ld))
        return out

    def select(self, scores, batch, rows, cols, s0, t0, ratio, k, apply_mask=True):
        ld = scores.shape[-1]
        width = min(k, cols)
        val = torch.empty((batch, rows, width), dtype=torch.float32, device=scores.device)
        idx = torch.empty((batch, rows, width), dtype=torch.int32, device=scores.device)
        check(self.lib.csaidx_cuda_select(self.handle, _p(scores), batch, rows, ld, cols, s0, t0, ratio,
                                          int(apply_mask), k, _p(val), _p(idx), width))
        return val, idx

    # ------------------------------------------------ fused select pre-filter
    def candidate_capacity(self, k: int) -> int:
        return int(self.lib.csaidx_cuda_candidate_capacity(k))

    def score_sampled(self, q, kc, w, dims: Dims, s0, rows, t0, cols, kt_stride):
        vt = (-(-cols // 128) + kt_stride - 1) // kt_stride
        out = torch.empty((dims.batch, rows, vt * 128), dtype=torch.float32, device=q.device)
        check(self.lib.csaidx_cuda_score_sampled(self.handle, _p(q), _p(kc), _p(w), byref(dims), s0, rows, t0, cols,
                                                 kt_stride, _p(out), out.shape[-1]))
        return out

    def row_threshold(self, sample, batch, rows, cols, s0, t0, ratio, kt_stride, k):
        tau = torch.empty((batch, rows), dtype=torch.float32, device=sample.device)
        check(self.lib.csaidx_cuda_row_threshold(self.handle, _p(sample), sample.shape[-1], batch, rows, cols, s0, t0,
                                                 ratio, kt_stride, k, _p(tau)))
        return tau

    def candidate_words(self, cols: int) -> int:
        return int(self.lib.csaidx_cuda_candidate_words(cols))

    def score_filtered(self, q, kc, w, dims: Dims, s0, rows, t0, cols, tau):
        """Masked score tile + per-row candidate bitmap (legal scores >= tau)."""
        ld = (cols + 3) // 4 * 4
        out = torch.empty((dims.batch, rows, ld), dtype=torch.float32, device=q.device)
        bits = torch.zeros((dims.batch, rows, self.candidate_words(cols)), dtype=torch.int32, device=q.device)
        check(self.lib.csaidx_cuda_score_filtered(self.handle, _p(q), _p(kc), _p(w), byref(dims), s0, rows, t0, cols,
                                                  _p(out), ld, _p(tau), _p(bits), bits.shape[-1]))
        return out, bits

    def select_from_candidates(self, scores, batch, rows, cols, s0, t0, ratio, k, bits):
        ld = scores.shape[-1]
        width = min(k, cols)
        val = torch.empty((batch, rows, width), dtype=torch.float32, device=scores.device)
        idx = torch.empty((batch, rows, width), dtype=torch.int32, device=scores.device)
        check(self.lib.csaidx_cuda_select_from_candidates(self.handle, _p(scores), batch, rows, ld, cols, s0, t0,
                                                          ratio, k, _p(bits), bits.shape[-1], _p(val),
                                                          _p(idx), width))
        return val, idx

    def select_final(self, scores, batch, rows, cols, s0, t0, ratio, k, out_idx, out_val, out_row0, bits=None,
                     gmax=None):
        """tile_topk + sentinel pass straight into int64/fp32 output rows [b, out_row0 + i, :k]
        (gmax: group maxima of score_gmax -> two-level select on long rows)."""
        ld = scores.shape[-1]
        check(self.lib.csaidx_cuda_select_final(self.handle, _p(scores), batch, rows, ld, cols, s0, t0, ratio, k,
                                                _p(bits), bits.shape[-1] if bits is not None else 0,
                                                _p(gmax), gmax.shape[-1] if gmax is not None else 0,
                                                _p(out_idx), _p(out_val), out_idx.shape[1], out_row0))

    def score_gmax(self, q, kc, w, dims: Dims, s0, rows, t0, cols, fill=None):
        """Masked tcgen05 score tile + per-32-key group maxima of every row
        (fill: initial value of both outputs, to expose unwritten entries)."""
        ld = (cols + 3) // 4 * 4
        out = torch.empty((dims.batch, rows, ld), dtype=torch.float32, device=q.device)
        gmax = torch.empty((dims.batch, rows, (cols + 31) // 32), dtype=torch.float32, device=q.device)
        if fill is not None:
            out.fill_(fill)
            gmax.fill_(fill)
        check(self.lib.csaidx_cuda_score_gmax(self.handle, _p(q), _p(kc), _p(w), byref(dims), s0, rows, t0, cols,
                                              _p(out), ld, dims.seq_len, s0, _p(gmax), gmax.shape[-1]))
        return out, gmax

    # ------------------------------------------------ sparse attention (f4)
    def sparse_attention(self, q, kv, indices, sm_scale, out=None, lse=True):
        """Sparse MLA-style attention over indices [B, S, k] (int32, -1 = padding):
        q bf16 [B, S, H, 576] (H a multiple of 128), kv bf16 [B, T, 576] ->
        out bf16 [B, S, H, 512] (+ lse fp32 [B, S, H]); csaidx_cuda_sparse_attention."""
        B, S, H, Dqk = q.shape
        T = kv.shape[1]
        k = indices.shape[-1]
        dv = 512
        if out is None:
            out = torch.empty((B, S, H, dv), dtype=torch.bfloat16, device=q.device)
        lse_t = torch.empty((B, S, H), dtype=torch.float32, device=q.device) if lse else None
        check(self.lib.csaidx_cuda_sparse_attention(self.handle, _p(q), _p(kv), _p(indices), B, S, T, H, Dqk, dv, k,
                                                    indices.stride(1), float(sm_scale), _p(out), out.stride(2),
                                                    _p(lse_t) if lse_t is not None else None))
        return out, lse_t

    def set_partition(self, score_sms: int, select_sms: int):
        """csaidx_engine_set_partition: score launches on score_sms SMs, selects as
        select_sms persistent multi-row CTAs (0, 0 = the whole GPU)."""
        check(self.lib.csaidx_engine_set_partition(self.handle, score_sms, select_sms))

    def candidate_hits(self, reset: bool = True) -> int:
        n = c_int64(0)
        check(self.lib.csaidx_engine_candidate_hits(self.handle, byref(n), int(reset)))
        return n.value

    def merge(self, run_val, run_idx, cand_val, cand_idx, overwrite=False, check_overlap=False):
        k = run_val.shape[-1]
        nrows = run_val.numel() // k
        width = cand_val.shape[-1]
        check(self.lib.csaidx_cuda_merge(self.handle, _p(run_val), _p(run_idx), nrows, k, _p(cand_val),
                                         _p(cand_idx), width, width, int(overwrite), int(check_overlap)))

    def fill_sentinel(self, val, idx):
        check(self.lib.csaidx_cuda_fill_sentinel(self.handle, _p(val), _p(idx), val.numel()))

    def finalize(self, run_val, run_idx, batch, rows, s0, ratio, k, out_idx, out_val, out_row0, check_keff=True):
        out_rows = out_idx.shape[1]
        check(self.lib.csaidx_cuda_finalize(self.handle, _p(run_val), _p(run_idx), batch, rows, s0, ratio, k,
                                            int(check_keff), _p(out_idx), _p(out_val), out_rows, out_row0))

    def chunk_step(self, q, kc, w, dims, s0, rows, t0, cols, score_buf, cand_val, cand_idx, run_val, run_idx,
                   first_tile, mode=0, kernel=0, overwrite=False):
        check(self.lib.csaidx_cuda_chunk_step(self.handle, _p(q), _p(kc), _dtype(q), _p(w), byref(dims), s0, rows,
                                              t0, cols,
                                              mode, kernel, _p(score_buf), score_buf.shape[-1], _p(cand_val),
                                              _p(cand_idx), _p(run_val), _p(run_idx), int(first_tile),
                                              int(overwrite)))
