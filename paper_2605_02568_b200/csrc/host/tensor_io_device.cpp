// CSAT dump -> HBM (reference tensor_io.cpp is host-only; this is the
// B200-side input producer of SURVEY.md §8 f3). The three sections are
// streamed in 32 MiB pieces: pread into one of two page-locked staging
// buffers, an asynchronous H2D copy on the engine's copy-in lane, and (for
// the tensor-core path) the fp32 -> bf16 rounding kernel on that lane, so
// file reading, PCIe and conversion overlap. With a chunk list only those
// query chunks' q / w rows are read, stacked like the output rows: a
// query-sharded rank reads 1/P of the file's q.
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstring>
#include <stdexcept>
#include <string>

#include "csaidx/gpu.hpp"
#include "csaidx/tensor_io.hpp"
#include "device.hpp"

namespace csaidx::gpu {

namespace {

constexpr uint64_t kPieceBytes = uint64_t{32} << 20;
constexpr int kSlot0 = 60;  // engine event slots of the two staging buffers
constexpr int kCopyLane = 1;

struct Piece {
    uint64_t file_off;
    uint64_t floats;
    void* dst;  // element offset already applied
    bool to_bf16;
};

class Fd {
public:
    explicit Fd(const std::string& path) : fd_(::open(path.c_str(), O_RDONLY | O_CLOEXEC)) {
        if (fd_ < 0) throw std::runtime_error("load_inputs: cannot open " + path + ": " + std::strerror(errno));
    }
    ~Fd() { ::close(fd_); }
    Fd(const Fd&) = delete;
    Fd& operator=(const Fd&) = delete;
    void read_at(void* dst, uint64_t bytes, uint64_t off) const {
        auto* p = static_cast<char*>(dst);
        while (bytes > 0) {
            const ssize_t n = ::pread(fd_, p, bytes, static_cast<off_t>(off));
            if (n < 0 && errno == EINTR) continue;
            if (n <= 0) throw std::runtime_error("load_inputs: short read");
            p += n;
            off += static_cast<uint64_t>(n);
            bytes -= static_cast<uint64_t>(n);
        }
    }

private:
    int fd_;
};

class PinnedPair {
public:
    PinnedPair(csaidx_engine* e, size_t bytes) : e_(e) {
        for (auto& b : buf_) detail::check(csaidx_cuda_host_alloc(e_, bytes, &b));
    }
    ~PinnedPair() {
        for (auto* b : buf_) csaidx_cuda_host_free(e_, b);
    }
    PinnedPair(const PinnedPair&) = delete;
    PinnedPair& operator=(const PinnedPair&) = delete;
    void* operator[](int i) const { return buf_[i]; }

private:
    csaidx_engine* e_;
    void* buf_[2] = {nullptr, nullptr};
};

void split(std::vector<Piece>& out, uint64_t off, uint64_t floats, char* dst, size_t esz, bool conv) {
    const uint64_t step = kPieceBytes / 4;
    for (uint64_t i = 0; i < floats; i += step) {
        const uint64_t n = std::min(step, floats - i);
        out.push_back({off + 4 * i, n, dst + i * esz, conv});
    }
}

void expect_section(const detail::SectionInfo& s, uint8_t tag, std::initializer_list<int64_t> dims) {
    bool ok = s.tag == tag && s.rank == dims.size();
    size_t i = 0;
    for (int64_t d : dims) ok = ok && static_cast<int64_t>(s.dims[i++]) == d;
    if (!ok) throw std::invalid_argument("load_inputs: section " + std::to_string(tag) + " does not match ProblemDims");
}

}  // namespace

void load_inputs_device(const std::string& path, const ProblemDims& dims, const TileConfig& tile,
                        const std::vector<int64_t>* chunk_starts, int dtype, bool strict, void* q, void* kc,
                        float* w) {
    detail::validate_dims(dims);
    if (dtype != CSAIDX_DTYPE_BF16 && dtype != CSAIDX_DTYPE_F32)
        throw std::invalid_argument("load_inputs: unknown operand dtype");
    const auto secs = detail::scan_sections_file(path);
    if (secs.size() != 3) throw std::invalid_argument("load_inputs: expected 3 sections (q, kc, w)");
    const int64_t B = dims.batch, S = dims.seq_len, T = dims.key_blocks, H = dims.heads, D = dims.head_dim;
    expect_section(secs[0], 0, {B, S, H, D});
    expect_section(secs[1], 1, {B, T, D});
    expect_section(secs[2], 2, {B, S, H});
    const detail::ChunkPlan plan = detail::plan_chunks(dims, tile, chunk_starts);
    int64_t out_rows = 0;
    for (int64_t s0 : plan.starts) out_rows += std::min(plan.cs, S - s0);

    const bool conv = dtype == CSAIDX_DTYPE_BF16;
    const size_t esz = conv ? 2 : 4;
    std::vector<Piece> pieces;
    for (int64_t b = 0; b < B; ++b) {
        for (size_t c = 0; c < plan.starts.size(); ++c) {
            const int64_t s0 = plan.starts[c], rows = std::min(plan.cs, S - s0);
            const int64_t lrow = b * out_rows + plan.out_row0[c];
            split(pieces, secs[0].offset + 4 * static_cast<uint64_t>((b * S + s0) * H * D),
                  static_cast<uint64_t>(rows * H * D), static_cast<char*>(q) + lrow * H * D * esz, esz, conv);
        }
    }
    split(pieces, secs[1].offset, static_cast<uint64_t>(B * T * D), static_cast<char*>(kc), esz, conv);
    for (int64_t b = 0; b < B; ++b) {
        for (size_t c = 0; c < plan.starts.size(); ++c) {
            const int64_t s0 = plan.starts[c], rows = std::min(plan.cs, S - s0);
            const int64_t lrow = b * out_rows + plan.out_row0[c];
            split(pieces, secs[2].offset + 4 * static_cast<uint64_t>((b * S + s0) * H),
                  static_cast<uint64_t>(rows * H), reinterpret_cast<char*>(w + lrow * H), 4, false);
        }
    }

    const Fd fd(path);
    std::lock_guard<std::mutex> lock(detail::engine_mutex());
    csaidx_engine* e = detail::engine();
    const PinnedPair staging(e, kPieceBytes);
    detail::DeviceBuffer slab[2];
    if (conv)
        for (auto& sb : slab) sb = detail::DeviceBuffer(e, kPieceBytes);
    try {
        for (size_t i = 0; i < pieces.size(); ++i) {
            const int j = static_cast<int>(i & 1);
            const Piece& pc = pieces[i];
            if (i >= 2) detail::check(csaidx_engine_sync_slot(e, kSlot0 + j));  // staging j is free again
            fd.read_at(staging[j], pc.floats * 4, pc.file_off);
            detail::check(csaidx_engine_use_lane(e, kCopyLane));
            if (pc.to_bf16) {
                detail::check(csaidx_cuda_copy(e, slab[j].as<void>(), staging[j], pc.floats * 4));
                detail::check(csaidx_cuda_to_bf16(e, slab[j].as<float>(), static_cast<uint16_t*>(pc.dst),
                                                  static_cast<int64_t>(pc.floats), strict ? 1 : 0));
            } else {
                detail::check(csaidx_cuda_copy(e, pc.dst, staging[j], pc.floats * 4));
            }
            detail::check(csaidx_engine_signal(e, kSlot0 + j));
            detail::check(csaidx_engine_use_lane(e, 0));
        }
        for (int j = 0; j < 2; ++j) detail::check(csaidx_engine_sync_slot(e, kSlot0 + j));
    } catch (...) {
        csaidx_engine_use_lane(e, 0);
        for (int j = 0; j < 2; ++j) csaidx_engine_sync_slot(e, kSlot0 + j);
        csaidx_engine_check(e);
        throw;
    }
    detail::check(csaidx_engine_check(e));  // latched non-finite / non-bf16 values
}

}  // namespace csaidx::gpu
