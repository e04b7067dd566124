"""ctypes binding of the C-ABI boundary (include/csaidx_cuda.h).

The shared library is built in-tree (``paper_2605_02568_b200/lib``) by
``__graft_entry__.build()``. There is no CPU path: when the library or a GPU
is missing, calls raise instead of falling back.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int64, c_size_t, c_uint64, c_void_p

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
CUDA_LIB = os.path.join(LIB_DIR, "libcsaidx_cuda.so")
HOST_LIB = os.path.join(LIB_DIR, "libcsaidx.so")

OK, INVALID_ARGUMENT, RUNTIME_ERROR, OVERFLOW_ERROR, LOGIC_ERROR, CUDA_ERROR = range(6)
KERNEL_AUTO, KERNEL_EXACT = 0, 1
DTYPE_BF16, DTYPE_F32 = 0, 1
MODE_FP32, MODE_FP16_EMULATED = 0, 1
KIND_SCORE, KIND_SELECT, KIND_MERGE, KIND_FINALIZE, KIND_PREP, KIND_ATTENTION = range(6)


class CsaidxError(RuntimeError):
    """Base class; subclasses mirror the reference's exception types."""


class InvalidArgument(CsaidxError, ValueError):
    """std::invalid_argument."""


class ScoreRuntimeError(CsaidxError):
    """std::runtime_error (e.g. non-finite fp32 score)."""


class ByteModelOverflow(CsaidxError, OverflowError):
    """std::overflow_error."""


class LogicError(CsaidxError):
    """std::logic_error (internal invariant)."""


class CudaError(CsaidxError):
    """CUDA failure (the C++ layer maps it to std::runtime_error)."""


_ERRORS = {
    INVALID_ARGUMENT: InvalidArgument,
    RUNTIME_ERROR: ScoreRuntimeError,
    OVERFLOW_ERROR: ByteModelOverflow,
    LOGIC_ERROR: LogicError,
    CUDA_ERROR: CudaError,
}


class Dims(ctypes.Structure):
    """csaidx_dims == ProblemDims (types.hpp:19-34)."""

    _fields_ = [
        ("batch", c_int64),
        ("seq_len", c_int64),
        ("key_blocks", c_int64),
        ("heads", c_int64),
        ("head_dim", c_int64),
        ("ratio", c_int64),
        ("top_k", c_int64),
    ]


# name -> (restype, argtypes); every symbol include/csaidx_cuda.h declares.
CUDA_SYMBOLS = {
    "csaidx_cuda_last_error": (c_char_p, []),
    "csaidx_cuda_abi_version": (c_int, []),
    "csaidx_cuda_device_count": (c_int, [POINTER(c_int)]),
    "csaidx_engine_create": (c_int, [c_int, POINTER(c_void_p)]),
    "csaidx_engine_destroy": (c_int, [c_void_p]),
    "csaidx_engine_set_stream": (c_int, [c_void_p, c_void_p]),
    "csaidx_engine_use_own_stream": (c_int, [c_void_p]),
    "csaidx_engine_get_stream": (c_int, [c_void_p, POINTER(c_void_p)]),
    "csaidx_engine_num_sms": (c_int, [c_void_p, POINTER(c_int)]),
    "csaidx_engine_check": (c_int, [c_void_p]),
    "csaidx_engine_take_inexact": (c_int, [c_void_p, POINTER(c_int)]),
    "csaidx_engine_sync": (c_int, [c_void_p]),
    "csaidx_cuda_narrow_indices": (c_int, [c_void_p, c_void_p, c_void_p, c_int64]),
    "csaidx_cuda_scatter_rows": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64]),
    "csaidx_engine_mem_stats": (c_int, [c_void_p, POINTER(c_uint64), POINTER(c_uint64)]),
    "csaidx_engine_reset_peak": (c_int, [c_void_p]),
    "csaidx_engine_set_profiling": (c_int, [c_void_p, c_int]),
    "csaidx_engine_kernel_stats": (c_int, [c_void_p, c_int, POINTER(c_int64), POINTER(ctypes.c_double)]),
    "csaidx_engine_reset_stats": (c_int, [c_void_p]),
    "csaidx_engine_select_fallbacks": (c_int, [c_void_p, POINTER(c_int64), c_int]),
    "csaidx_engine_candidate_hits": (c_int, [c_void_p, POINTER(c_int64), c_int]),
    "csaidx_engine_set_select_probe": (c_int, [c_void_p, c_void_p]),
    "csaidx_engine_set_score_probe": (c_int, [c_void_p, c_void_p]),
    "csaidx_engine_use_lane": (c_int, [c_void_p, c_int]),
    "csaidx_engine_signal": (c_int, [c_void_p, c_int]),
    "csaidx_engine_await": (c_int, [c_void_p, c_int]),
    "csaidx_engine_sync_slot": (c_int, [c_void_p, c_int]),
    "csaidx_engine_copy_on_lane": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_size_t]),
    "csaidx_engine_await_stream": (c_int, [c_void_p, c_void_p]),
    "csaidx_engine_set_index_sink": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64]),
    "csaidx_cuda_ipc_handle": (c_int, [c_void_p, c_void_p, c_void_p, POINTER(c_uint64)]),
    "csaidx_cuda_ipc_open": (c_int, [c_void_p, c_void_p, c_uint64, POINTER(c_void_p)]),
    "csaidx_cuda_ipc_close": (c_int, [c_void_p, c_void_p, c_uint64]),
    "csaidx_engine_set_partition": (c_int, [c_void_p, c_int, c_int]),
    "csaidx_cuda_select_overlap_capable": (c_int, [c_int64]),
    "csaidx_cuda_alloc": (c_int, [c_void_p, c_size_t, POINTER(c_void_p)]),
    "csaidx_cuda_free": (c_int, [c_void_p, c_void_p]),
    "csaidx_cuda_copy": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t]),
    "csaidx_cuda_memset": (c_int, [c_void_p, c_void_p, c_int, c_size_t]),
    "csaidx_cuda_host_alloc": (c_int, [c_void_p, c_size_t, POINTER(c_void_p)]),
    "csaidx_cuda_host_free": (c_int, [c_void_p, c_void_p]),
    "csaidx_cuda_host_is_pinned": (c_int, [c_void_p, POINTER(c_int)]),
    "csaidx_cuda_to_bf16": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int]),
    "csaidx_cuda_score": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int, c_void_p, POINTER(Dims), c_int64, c_int64, c_int64, c_int64,
         c_int, c_int, c_int, c_void_p, c_int64],
    ),
    "csaidx_cuda_score_rows": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int, c_void_p, POINTER(Dims), c_int64, c_int64, c_int64, c_int64,
         c_int, c_int, c_int, c_void_p, c_int64, c_int64, c_int64],
    ),
    "csaidx_cuda_score_uses_tensor_cores": (c_int, [POINTER(Dims), c_int, c_int, c_int]),
    "csaidx_cuda_bool_mask": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64]),
    "csaidx_cuda_apply_bool_mask": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64]),
    "csaidx_cuda_select": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int, c_int64,
         c_void_p, c_void_p, c_int64],
    ),
    "csaidx_cuda_select_capacity": (c_int, []),
    "csaidx_cuda_candidate_capacity": (c_int, [c_int64]),
    "csaidx_cuda_candidate_words": (c_int64, [c_int64]),
    "csaidx_cuda_score_sampled": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, POINTER(Dims), c_int64, c_int64, c_int64, c_int64, c_int,
         c_void_p, c_int64],
    ),
    "csaidx_cuda_row_threshold": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int, c_int64,
         c_void_p],
    ),
    "csaidx_cuda_score_filtered": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, POINTER(Dims), c_int64, c_int64, c_int64, c_int64,
         c_void_p, c_int64, c_void_p, c_void_p, c_int64],
    ),
    "csaidx_cuda_select_from_candidates": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64,
         c_void_p, c_int64, c_void_p, c_void_p, c_int64],
    ),
    "csaidx_cuda_select_final": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64,
         c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_int64],
    ),
    "csaidx_cuda_score_gmax": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, POINTER(Dims), c_int64, c_int64, c_int64, c_int64,
         c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64],
    ),
    "csaidx_cuda_merge": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_int64, c_int64, c_int, c_int],
    ),
    "csaidx_cuda_fill_sentinel": (c_int, [c_void_p, c_void_p, c_void_p, c_int64]),
    "csaidx_cuda_sparse_attention": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64,
         c_int64, c_float, c_void_p, c_int64, c_void_p],
    ),
    "csaidx_cuda_finalize": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_int, c_void_p, c_void_p,
         c_int64, c_int64],
    ),
    "csaidx_cuda_chunk_step": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_int, c_void_p, POINTER(Dims), c_int64, c_int64, c_int64, c_int64, c_int, c_int,
         c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int],
    ),
    "csaidx_cuda_gen_normal_bf16": (c_int, [c_void_p, c_void_p, c_int64, c_double, c_uint64, c_uint64, c_int64]),
    "csaidx_cuda_gen_normal_f32": (c_int, [c_void_p, c_void_p, c_int64, c_double, c_uint64, c_uint64, c_int64]),
}

_cuda = None


def cuda_lib():
    """Load libcsaidx_cuda.so (raises if it was not built)."""
    global _cuda
    if _cuda is None:
        if not os.path.exists(CUDA_LIB):
            raise ImportError(f"{CUDA_LIB} missing: run __graft_entry__.build() (no CPU fallback exists)")
        lib = ctypes.CDLL(CUDA_LIB)
        for name, (res, args) in CUDA_SYMBOLS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _cuda = lib
    return _cuda


def check(rc: int) -> None:
    if rc != OK:
        msg = cuda_lib().csaidx_cuda_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, CsaidxError)(msg)
