// Causal legality (host integer math, causal.cpp:9-28) and tile masking on
// the GPU (causal.cpp:30-79 semantics).
#include "csaidx/causal.hpp"

#include <stdexcept>

#include "device.hpp"

namespace csaidx {

int64_t t_legal(int64_t t, int64_t ratio) {
    if (t < 0 || ratio < 1) throw std::invalid_argument("t_legal: t must be >= 0 and ratio >= 1");
    return (t + 1) / ratio;
}

int64_t k_eff(int64_t t, int64_t ratio, int64_t top_k) {
    if (top_k < 0) throw std::invalid_argument("k_eff: top_k must be >= 0");
    const int64_t legal = t_legal(t, ratio);
    return top_k < legal ? top_k : legal;
}

bool tile_fully_masked(int64_t s0, int64_t rows, int64_t t0, int64_t ratio) {
    if (rows < 1) throw std::invalid_argument("tile_fully_masked: rows must be >= 1");
    return t0 >= t_legal(s0 + rows - 1, ratio);
}

namespace {

// Round-trips a host tile through the device keep-mask kernels.
void apply_device_mask(ScoreTile& tile, const detail::DeviceBuffer& keep) {
    if (tile.scores.empty()) return;
    csaidx_engine* e = detail::engine();
    const int64_t ld = (tile.cols + 3) / 4 * 4;
    detail::DeviceBuffer dev(e, static_cast<size_t>(tile.batch * tile.rows * ld) * sizeof(float));
    for (int64_t r = 0; r < tile.batch * tile.rows; ++r)
        detail::check(csaidx_cuda_copy(e, dev.as<float>() + r * ld, tile.scores.data() + r * tile.cols,
                                       static_cast<size_t>(tile.cols) * sizeof(float)));
    detail::check(csaidx_cuda_apply_bool_mask(e, dev.as<float>(), ld, keep.as<uint8_t>(), tile.batch, tile.rows,
                                              tile.cols));
    for (int64_t r = 0; r < tile.batch * tile.rows; ++r)
        detail::check(csaidx_cuda_copy(e, tile.scores.data() + r * tile.cols, dev.as<float>() + r * ld,
                                       static_cast<size_t>(tile.cols) * sizeof(float)));
    detail::check(csaidx_engine_check(e));
}

}  // namespace

void mask_tile(ScoreTile& tile, int64_t ratio) {
    if (tile.rows < 1 || tile.cols < 1) return;
    if (ratio < 1) throw std::invalid_argument("t_legal: t must be >= 0 and ratio >= 1");
    std::lock_guard<std::mutex> lock(detail::engine_mutex());
    csaidx_engine* e = detail::engine();
    detail::DeviceBuffer keep(e, static_cast<size_t>(tile.rows * tile.cols));
    detail::check(csaidx_cuda_bool_mask(e, keep.as<uint8_t>(), tile.s0, tile.t0, tile.rows, tile.cols, ratio));
    apply_device_mask(tile, keep);
}

MaskTile build_mask_tile(int64_t s0, int64_t t0, int64_t rows, int64_t cols, int64_t ratio, MemoryLedger& ledger) {
    if (rows < 1 || cols < 1 || s0 < 0 || t0 < 0) throw std::invalid_argument("build_mask_tile: bad tile extents");
    MaskTile m;
    m.rows = rows;
    m.cols = cols;
    m.s0 = s0;
    m.t0 = t0;
    m.charge = LedgerCharge(ledger, "mask_tile", static_cast<uint64_t>(rows) * static_cast<uint64_t>(cols));
    m.keep.resize(static_cast<size_t>(rows * cols));
    std::lock_guard<std::mutex> lock(detail::engine_mutex());
    csaidx_engine* e = detail::engine();
    detail::DeviceBuffer keep(e, m.keep.size());
    detail::check(csaidx_cuda_bool_mask(e, keep.as<uint8_t>(), s0, t0, rows, cols, ratio));
    keep.download(m.keep.data(), m.keep.size());
    detail::check(csaidx_engine_check(e));
    return m;
}

void apply_mask_tile(ScoreTile& tile, const MaskTile& mask) {
    if (mask.rows != tile.rows || mask.cols != tile.cols || mask.s0 != tile.s0 || mask.t0 != tile.t0)
        throw std::invalid_argument("apply_mask_tile: mask does not match tile");
    if (tile.rows < 1 || tile.cols < 1) return;
    std::lock_guard<std::mutex> lock(detail::engine_mutex());
    csaidx_engine* e = detail::engine();
    detail::DeviceBuffer keep(e, mask.keep.size());
    keep.upload(mask.keep.data(), mask.keep.size());
    apply_device_mask(tile, keep);
}

}  // namespace csaidx
