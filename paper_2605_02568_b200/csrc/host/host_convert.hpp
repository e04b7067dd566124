// Host-side fp32 -> bf16 rounding for the pipelined host entry: the
// reference API hands q over as fp32 (types.hpp:49-57), and PCIe is the
// bound of the end-to-end call, so q rows are rounded on the host cores into
// pinned bf16 staging slabs and cross the bus at half the bytes. Same
// rounding as the device path (csaidx_cuda_to_bf16 / __float2bfloat16_rn:
// round to nearest even), same checks (IndexerInputs::validated,
// types.cpp:73-92: non-finite entries; strict mode: non-representable ones).
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>

namespace csaidx::detail {

struct Bf16Flags {
    bool nonfinite = false;
    bool inexact = false;
};

// Rounds src[0, n) into dst[0, n) on the host worker pool (AVX-512 when the
// CPU has it, else scalar; bit-identical either way).
// nt: 1 = non-temporal stores (the destination is read back from DRAM later),
// 0 = regular stores (it is read again while still cached), -1 = CSAIDX_HOST_NT.
Bf16Flags host_to_bf16(const float* src, uint16_t* dst, size_t n, int nt = -1);

// Scalar reference of one element (tests, tails).
uint16_t host_bf16_rne(float x);

// Threads of a parallel region incl. the caller (CSAIDX_HOST_THREADS,
// default: usable cores / LOCAL_WORLD_SIZE - 1).
int host_threads();

// Runs fn(0) .. fn(parts - 1) on the pool and the calling thread; blocks.
void host_parallel_for(int parts, const std::function<void(int)>& fn);

// Whether the pipelined host entry rounds q on the host (CSAIDX_HOST_ROUND=1 /
// 0; default: on unless several ranks share the node, LOCAL_WORLD_SIZE > 1).
bool host_round_enabled();

// Pinned bf16 staging slabs of that pipeline (CSAIDX_HOST_SLABS, 2..32)
// and the bf16 bytes rounded and copied per piece (CSAIDX_HOST_PIECE_KB).
int host_slab_count();
int64_t host_piece_bytes();
// Ring mode of the pipeline (default; CSAIDX_HOST_RING=0 turns it off): q
// rounded piece by piece (CSAIDX_HOST_PIECE_KB of bf16, default 8 MiB) into
// a small pinned ring (CSAIDX_HOST_RING_PIECES, default 4; regular stores)
// whose pieces are copied right away, so the DMA reads them while they are
// still in the host's last-level cache.
bool host_ring_enabled();
int host_ring_pieces();
// Chunks at the end of the processing order sent as fp32 (pinned q) and
// rounded on the device (CSAIDX_HOST_FP32_TAIL, at most 27; default 0:
// measured slower).
size_t host_fp32_tail(size_t chunks);

}  // namespace csaidx::detail
