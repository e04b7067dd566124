// Selection API (reference semantics: topk.cpp). tile_topk, merge_topk and
// overwrite_topk execute on the GPU select / merge kernels; the bounded heap,
// streaming_topk and oracle_topk are the host-side reference containers the
// theorem tests use (not on the hot path).
#include "csaidx/topk.hpp"

#include <algorithm>
#include <limits>
#include <stdexcept>

#include "device.hpp"

namespace csaidx {

namespace {

constexpr float kNegInf = -std::numeric_limits<float>::infinity();

// With succ as the "less" of std heap routines the succ-minimum sits at the
// front: exactly the entry a better offer evicts; sort_heap gives best-first.
struct WorseFirst {
    bool operator()(const ScoredIndex& a, const ScoredIndex& b) const { return succ(a, b); }
};

int32_t narrow_index(int64_t idx) {
    if (idx < -1 || idx > std::numeric_limits<int32_t>::max())
        throw std::invalid_argument("selection index outside the device index range");
    return static_cast<int32_t>(idx);
}

// Uploads one running row and a tile list, runs the device merge (or the A1
// overwrite), and writes the row back.
void device_merge_row(TopKBuffer& buf, int64_t b, int64_t row, std::span<const ScoredIndex> tile_list,
                      bool overwrite) {
    if (b < 0 || b >= buf.batch || row < 0 || row >= buf.rows) throw std::invalid_argument("merge_topk: row out of range");
    const int64_t k = buf.top_k;
    const int64_t n = std::min<int64_t>(static_cast<int64_t>(tile_list.size()), k);
    std::vector<float> rv(buf.v_row(b, row), buf.v_row(b, row) + k), cv(static_cast<size_t>(std::max<int64_t>(n, 1)));
    std::vector<int32_t> ri(static_cast<size_t>(k)), ci(static_cast<size_t>(std::max<int64_t>(n, 1)));
    for (int64_t e = 0; e < k; ++e) ri[static_cast<size_t>(e)] = narrow_index(buf.i_row(b, row)[e]);
    for (int64_t e = 0; e < n; ++e) {
        cv[static_cast<size_t>(e)] = tile_list[static_cast<size_t>(e)].score;
        ci[static_cast<size_t>(e)] = narrow_index(tile_list[static_cast<size_t>(e)].index);
    }
    if (!overwrite) {
        // Overlap contract (topk.cpp:39-53) includes entries past the first k.
        std::vector<int64_t> seen;
        for (int64_t e = 0; e < k; ++e)
            if (buf.i_row(b, row)[e] != kSentinelIndex) seen.push_back(buf.i_row(b, row)[e]);
        for (const ScoredIndex& s : tile_list)
            if (s.index != kSentinelIndex) seen.push_back(s.index);
        std::sort(seen.begin(), seen.end());
        if (std::adjacent_find(seen.begin(), seen.end()) != seen.end())
            throw std::invalid_argument("merge_topk: overlapping indices between buffer and tile");
    }
    std::lock_guard<std::mutex> lock(detail::engine_mutex());
    csaidx_engine* e = detail::engine();
    detail::DeviceBuffer dv(e, rv.size() * 4), di(e, ri.size() * 4), dcv(e, cv.size() * 4), dci(e, ci.size() * 4);
    dv.upload(rv.data(), rv.size() * 4);
    di.upload(ri.data(), ri.size() * 4);
    dcv.upload(cv.data(), cv.size() * 4);
    dci.upload(ci.data(), ci.size() * 4);
    detail::check(csaidx_cuda_merge(e, dv.as<float>(), di.as<int32_t>(), 1, k, dcv.as<float>(), dci.as<int32_t>(),
                                    std::max<int64_t>(n, 1), n, overwrite ? 1 : 0, 0));
    dv.download(rv.data(), rv.size() * 4);
    di.download(ri.data(), ri.size() * 4);
    detail::check(csaidx_engine_check(e));
    for (int64_t x = 0; x < k; ++x) {
        buf.v_row(b, row)[x] = rv[static_cast<size_t>(x)];
        buf.i_row(b, row)[x] = ri[static_cast<size_t>(x)];
    }
}

}  // namespace

BoundedTopK::BoundedTopK(int64_t capacity) : capacity_(capacity) {
    if (capacity < 1) throw std::invalid_argument("BoundedTopK: capacity must be >= 1");
    heap_.reserve(static_cast<size_t>(capacity));
}

void BoundedTopK::offer(ScoredIndex entry) {
    if (size() < capacity_) {
        heap_.push_back(entry);
        std::push_heap(heap_.begin(), heap_.end(), WorseFirst{});
    } else if (succ(entry, heap_.front())) {
        std::pop_heap(heap_.begin(), heap_.end(), WorseFirst{});
        heap_.back() = entry;
        std::push_heap(heap_.begin(), heap_.end(), WorseFirst{});
    }
}

void BoundedTopK::reset() { heap_.clear(); }

std::vector<ScoredIndex> BoundedTopK::take_sorted() {
    std::sort_heap(heap_.begin(), heap_.end(), WorseFirst{});
    std::vector<ScoredIndex> out;
    out.swap(heap_);
    return out;
}

std::vector<ScoredIndex> streaming_topk(std::span<const ScoredIndex> stream, int64_t k) {
    if (k < 1) throw std::invalid_argument("streaming_topk: k must be >= 1");
    std::vector<int64_t> ids;
    ids.reserve(stream.size());
    for (const ScoredIndex& e : stream) ids.push_back(e.index);
    std::sort(ids.begin(), ids.end());
    if (std::adjacent_find(ids.begin(), ids.end()) != ids.end())
        throw std::invalid_argument("streaming_topk: duplicate index in stream");
    BoundedTopK heap(std::min<int64_t>(k, std::max<int64_t>(1, static_cast<int64_t>(stream.size()))));
    for (const ScoredIndex& e : stream) heap.offer(e);
    return heap.take_sorted();
}

TileTopK tile_topk(const ScoreTile& tile, int64_t top_k, MemoryLedger& ledger) {
    if (top_k < 1) throw std::invalid_argument("tile_topk: top_k must be >= 1");
    TileTopK out;
    out.batch = tile.batch;
    out.rows = tile.rows;
    out.width = std::min(top_k, tile.cols);
    out.charge = LedgerCharge(ledger, "tile_topk_scratch", tile_scratch_bytes(tile.batch, tile.rows, tile.cols, top_k));
    out.entries.resize(static_cast<size_t>(tile.batch * tile.rows * out.width));
    if (out.entries.empty()) return out;

    std::lock_guard<std::mutex> lock(detail::engine_mutex());
    csaidx_engine* e = detail::engine();
    const int64_t nrows = tile.batch * tile.rows;
    const int64_t ld = (tile.cols + 3) / 4 * 4;
    detail::DeviceBuffer scores(e, static_cast<size_t>(nrows * ld) * sizeof(float));
    for (int64_t r = 0; r < nrows; ++r)
        detail::check(csaidx_cuda_copy(e, scores.as<float>() + r * ld, tile.scores.data() + r * tile.cols,
                                       static_cast<size_t>(tile.cols) * sizeof(float)));
    detail::DeviceBuffer val(e, static_cast<size_t>(nrows * out.width) * 4), idx(e, static_cast<size_t>(nrows * out.width) * 4);
    // apply_mask = 0: every column competes; -inf entries become placeholders
    // with real indices, exactly like the reference heap.
    detail::check(csaidx_cuda_select(e, scores.as<float>(), tile.batch, tile.rows, ld, tile.cols, tile.s0, tile.t0, 1,
                                     0, top_k, val.as<float>(), idx.as<int32_t>(), out.width));
    std::vector<float> hv(static_cast<size_t>(nrows * out.width));
    std::vector<int32_t> hi(hv.size());
    val.download(hv.data(), hv.size() * 4);
    idx.download(hi.data(), hi.size() * 4);
    detail::check(csaidx_engine_check(e));
    for (size_t x = 0; x < hv.size(); ++x) out.entries[x] = ScoredIndex{hv[x], hi[x]};
    return out;
}

void merge_topk(TopKBuffer& buf, int64_t b, int64_t row, std::span<const ScoredIndex> tile_list) {
    device_merge_row(buf, b, row, tile_list, false);
}

void overwrite_topk(TopKBuffer& buf, int64_t b, int64_t row, std::span<const ScoredIndex> tile_list) {
    device_merge_row(buf, b, row, tile_list, true);
}

std::vector<ScoredIndex> oracle_topk(std::span<const float> row_scores, int64_t k, int64_t legal) {
    if (k < 1 || legal < 0 || legal > static_cast<int64_t>(row_scores.size()))
        throw std::invalid_argument("oracle_topk: bad k or legal prefix");
    std::vector<ScoredIndex> all(static_cast<size_t>(legal));
    for (int64_t j = 0; j < legal; ++j) all[static_cast<size_t>(j)] = ScoredIndex{row_scores[static_cast<size_t>(j)], j};
    const int64_t take = std::min(k, legal);
    std::partial_sort(all.begin(), all.begin() + take, all.end(), WorseFirst{});
    all.resize(static_cast<size_t>(take));
    return all;
}

}  // namespace csaidx
