// score_tile on the GPU (reference semantics: score.cpp:18-101).
#include "csaidx/score.hpp"

#include <algorithm>
#include <stdexcept>

#include "device.hpp"

namespace csaidx {

bool avx2_kernels_available() { return false; }

ScoreKernel resolve_score_kernel(ScoreKernel requested, int64_t head_dim) {
    (void)head_dim;
    switch (requested) {
        case ScoreKernel::auto_detect: return ScoreKernel::auto_detect;  // device picks tcgen05 or exact
        case ScoreKernel::scalar: return ScoreKernel::scalar;
        case ScoreKernel::avx2:
            throw std::invalid_argument("avx2 kernel requested but this build has no AVX2 kernel (B200 path)");
    }
    throw std::invalid_argument("unknown score kernel");
}

const char* score_kernel_name(ScoreKernel kernel) {
    switch (kernel) {
        case ScoreKernel::auto_detect: return "auto";
        case ScoreKernel::scalar: return "scalar";
        case ScoreKernel::avx2: return "avx2";
    }
    return "unknown";
}

ScoreTile score_tile(const IndexerInputs& inputs, const ProblemDims& dims, int64_t s0, int64_t t0, int64_t rows,
                     int64_t cols, AccumulationMode mode, MemoryLedger& ledger, ScoreKernel kernel) {
    if (rows < 1 || cols < 1 || s0 < 0 || t0 < 0 || s0 + rows > dims.seq_len || t0 + cols > dims.key_blocks)
        throw std::invalid_argument("score_tile: tile out of range");
    const int kcode = detail::kernel_code(kernel, mode);
    const int mcode = detail::mode_code(mode);

    ScoreTile tile;
    tile.batch = dims.batch;
    tile.rows = rows;
    tile.cols = cols;
    tile.s0 = s0;
    tile.t0 = t0;
    tile.charge = LedgerCharge(ledger, "score_tile", chunk_tile_bytes(dims.batch, rows, cols));
    tile.scores.resize(static_cast<size_t>(dims.batch * rows * cols));

    // Stage only the operand rows this tile reads: q / w rows [s0, s0+rows)
    // and kc rows [t0, t0+cols) of every batch, as a compact instance.
    ProblemDims local = dims;
    local.seq_len = rows;
    local.key_blocks = cols;
    std::vector<float> q(static_cast<size_t>(local.q_elems())), kc(static_cast<size_t>(local.kc_elems())),
        w(static_cast<size_t>(local.w_elems()));
    const int64_t qrow = dims.heads * dims.head_dim;
    for (int64_t b = 0; b < dims.batch; ++b) {
        std::copy_n(inputs.q.data() + (b * dims.seq_len + s0) * qrow, rows * qrow, q.data() + b * rows * qrow);
        std::copy_n(inputs.w.data() + (b * dims.seq_len + s0) * dims.heads, rows * dims.heads,
                    w.data() + b * rows * dims.heads);
        std::copy_n(inputs.kc.data() + (b * dims.key_blocks + t0) * dims.head_dim, cols * dims.head_dim,
                    kc.data() + b * cols * dims.head_dim);
    }

    std::lock_guard<std::mutex> lock(detail::engine_mutex());
    csaidx_engine* e = detail::engine();
    const int dtype = detail::operand_dtype(dims, mcode, kcode);
    detail::StagedOperands ops(e, detail::HostView{q.data(), kc.data(), w.data()}, local, dtype,
                               gpu::options().strict_bf16);
    const int64_t ld = (cols + 3) / 4 * 4;
    detail::DeviceBuffer out(e, static_cast<size_t>(dims.batch * rows * ld) * sizeof(float));
    const csaidx_dims cd = detail::to_c(local);
    const detail::DeviceOps o = ops.ops();
    detail::check(csaidx_cuda_score(e, o.q, o.kc, o.dtype, o.w, &cd, 0, rows, 0, cols, mcode, kcode, 0,
                                    out.as<float>(), ld));
    for (int64_t r = 0; r < dims.batch * rows; ++r)
        detail::check(csaidx_cuda_copy(e, tile.scores.data() + r * cols, out.as<float>() + r * ld,
                                       static_cast<size_t>(cols) * sizeof(float)));
    detail::check(csaidx_engine_check(e));  // runtime_error on a non-finite fp32 score
    return tile;
}

}  // namespace csaidx
