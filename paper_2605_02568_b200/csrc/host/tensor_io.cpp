// CSAT input dump (reference tensor_io.cpp:28-140), host side. Headers are
// encoded field by field in little-endian order; payloads stream in 1 MiB
// blocks (no second copy of a multi-GiB tensor), as raw bytes on
// little-endian hosts and byte-swapped otherwise.
#include "csaidx/tensor_io.hpp"

#include <algorithm>
#include <array>
#include <cstring>
#include <fstream>
#include <istream>
#include <ostream>
#include <stdexcept>

namespace csaidx {

namespace {

constexpr size_t kHeaderBytes = 32;
constexpr size_t kBlockFloats = 1 << 18;  // 1 MiB payload blocks

using Header = std::array<uint8_t, kHeaderBytes>;

constexpr bool host_is_little_endian() { return __BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__; }

void store_le32(uint8_t* p, uint32_t v) {
    for (int i = 0; i < 4; ++i) p[i] = static_cast<uint8_t>(v >> (8 * i));
}

uint32_t load_le32(const uint8_t* p) {
    return static_cast<uint32_t>(p[0]) | static_cast<uint32_t>(p[1]) << 8 | static_cast<uint32_t>(p[2]) << 16 |
           static_cast<uint32_t>(p[3]) << 24;
}

Header encode_header(uint8_t tag, const std::vector<uint32_t>& dims) {
    Header h{};
    std::memcpy(h.data(), "CSAT", 4);
    store_le32(h.data() + 4, kTensorFileVersion);
    h[8] = tag;
    h[9] = static_cast<uint8_t>(dims.size());
    for (size_t i = 0; i < dims.size(); ++i) store_le32(h.data() + 12 + 4 * i, dims[i]);
    return h;
}

// Validates one header (reference order of checks) and returns the payload
// element count.
uint64_t decode_header(const Header& h, detail::SectionInfo& s) {
    if (std::memcmp(h.data(), "CSAT", 4) != 0) throw std::runtime_error("read_sections: bad magic");
    if (load_le32(h.data() + 4) != kTensorFileVersion) throw std::runtime_error("read_sections: unsupported version");
    s.tag = h[8];
    s.rank = h[9];
    if (s.rank == 0 || s.rank > 4) throw std::runtime_error("read_sections: bad rank");
    uint64_t elems = 1;
    for (int i = 0; i < 4; ++i) {
        s.dims[i] = load_le32(h.data() + 12 + 4 * i);
        if (i < s.rank) {
            if (s.dims[i] == 0) throw std::runtime_error("read_sections: zero extent");
            elems *= s.dims[i];
        }
    }
    s.elems = elems;
    return elems;
}

void write_payload(std::ostream& os, const std::vector<float>& data) {
    if constexpr (host_is_little_endian()) {
        os.write(reinterpret_cast<const char*>(data.data()), static_cast<std::streamsize>(data.size() * 4));
    } else {
        std::vector<uint8_t> block;
        for (size_t i0 = 0; i0 < data.size(); i0 += kBlockFloats) {
            const size_t n = std::min(kBlockFloats, data.size() - i0);
            block.resize(n * 4);
            for (size_t i = 0; i < n; ++i) {
                uint32_t bits;
                std::memcpy(&bits, &data[i0 + i], 4);
                store_le32(block.data() + 4 * i, bits);
            }
            os.write(reinterpret_cast<const char*>(block.data()), static_cast<std::streamsize>(block.size()));
        }
    }
}

void write_section(std::ostream& os, uint8_t tag, const std::vector<uint32_t>& dims, const std::vector<float>& data) {
    const Header h = encode_header(tag, dims);
    os.write(reinterpret_cast<const char*>(h.data()), kHeaderBytes);
    write_payload(os, data);
}

uint32_t dim32(int64_t v) { return static_cast<uint32_t>(v); }

}  // namespace

void write_inputs(std::ostream& os, const IndexerInputs& inputs, const ProblemDims& d) {
    write_section(os, 0, {dim32(d.batch), dim32(d.seq_len), dim32(d.heads), dim32(d.head_dim)}, inputs.q);
    write_section(os, 1, {dim32(d.batch), dim32(d.key_blocks), dim32(d.head_dim)}, inputs.kc);
    write_section(os, 2, {dim32(d.batch), dim32(d.seq_len), dim32(d.heads)}, inputs.w);
}

uint64_t write_inputs_file(const std::string& path, const IndexerInputs& inputs, const ProblemDims& dims) {
    std::ofstream os(path, std::ios::binary | std::ios::trunc);
    if (!os) throw std::runtime_error("write_inputs_file: cannot open " + path);
    write_inputs(os, inputs, dims);
    os.flush();
    if (!os) throw std::runtime_error("write_inputs_file: write failed for " + path);
    return 3 * kHeaderBytes + 4 * static_cast<uint64_t>(inputs.q.size() + inputs.kc.size() + inputs.w.size());
}

std::vector<TensorSection> read_sections(std::istream& is) {
    std::vector<TensorSection> out;
    Header h{};
    while (is.read(reinterpret_cast<char*>(h.data()), kHeaderBytes)) {
        detail::SectionInfo info;
        const uint64_t elems = decode_header(h, info);
        TensorSection s;
        s.tag = info.tag;
        s.rank = info.rank;
        std::copy(std::begin(info.dims), std::end(info.dims), std::begin(s.dims));
        s.data.resize(elems);
        if (!is.read(reinterpret_cast<char*>(s.data.data()), static_cast<std::streamsize>(elems * 4)))
            throw std::runtime_error("read_sections: truncated payload");
        if constexpr (!host_is_little_endian()) {
            for (auto& f : s.data) {
                uint32_t bits;
                std::memcpy(&bits, &f, 4);
                bits = load_le32(reinterpret_cast<const uint8_t*>(&bits));
                std::memcpy(&f, &bits, 4);
            }
        }
        out.push_back(std::move(s));
    }
    // a clean end reads zero bytes; a partial header is a truncated file
    if (is.gcount() != 0) throw std::runtime_error("read_sections: truncated header");
    if (out.empty()) throw std::runtime_error("read_sections: empty stream");
    return out;
}

namespace detail {

std::vector<SectionInfo> scan_sections_file(const std::string& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw std::runtime_error("read_sections: cannot open " + path);
    is.seekg(0, std::ios::end);
    const uint64_t size = static_cast<uint64_t>(is.tellg());
    is.seekg(0);
    std::vector<SectionInfo> out;
    uint64_t at = 0;
    Header h{};
    while (at < size) {
        if (size - at < kHeaderBytes) throw std::runtime_error("read_sections: truncated header");
        is.seekg(static_cast<std::streamoff>(at));
        is.read(reinterpret_cast<char*>(h.data()), kHeaderBytes);
        SectionInfo s;
        const uint64_t elems = decode_header(h, s);
        s.offset = at + kHeaderBytes;
        if (size - s.offset < elems * 4) throw std::runtime_error("read_sections: truncated payload");
        at = s.offset + elems * 4;
        out.push_back(s);
    }
    if (out.empty()) throw std::runtime_error("read_sections: empty stream");
    return out;
}

}  // namespace detail

}  // namespace csaidx
