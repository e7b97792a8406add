// Host-side .ffcz archive serialisation (format: /root/reference/proj/docs/FORMAT.md).
#pragma once

#include <cstdint>
#include <vector>

namespace ffcz_host {

struct EscapeRec {
    bool frequency;
    std::uint64_t index;
    double re, im;
};

struct ArchiveInput {
    int ndim;
    std::uint64_t dims[3];
    int precision;  // 0 f32, 1 f64
    bool spatial_per_point;
    double spatial_global;
    const double* spatial_values;  // N (host)
    bool freq_per_component;
    double freq_global;
    const double* freq_re;  // N (host, full spectrum)
    const double* freq_im;
    int m;
    bool converged;
    const std::uint8_t* spatial_flags;   std::uint64_t spatial_flag_bytes;
    const std::uint8_t* frequency_flags; std::uint64_t frequency_flag_bytes;
    std::uint64_t n_spatial, n_frequency;
    const std::int32_t* spatial_codes;    // n_spatial
    const std::int32_t* frequency_codes;  // 2 * n_frequency
    const EscapeRec* escapes;
    std::uint64_t n_escapes;
    int zlib_level;
    // pre-encoded Huffman payloads (device encoder); when set, the codes above are not read
    const std::uint8_t* spatial_payload = nullptr;   std::uint64_t spatial_payload_len = 0;
    const std::uint8_t* frequency_payload = nullptr; std::uint64_t frequency_payload_len = 0;
};

// read_archive (archive.cpp:137-225) up to, but not including, the Huffman decode of the index
// streams (that runs on the device): header + CRC-32C, flag streams and index payloads
// (outer_decompress, streams.cpp:34-48), escape records.  Bound arrays point into `bytes`.
struct ParsedArchive {
    int ndim = 0;
    std::uint64_t dims[3] = {1, 1, 1};
    int precision = 0;
    bool spatial_per_point = false, freq_per_component = false, converged = false;
    double spatial_global = 0.0, freq_global = 0.0;
    const std::uint8_t* spatial_values = nullptr;  // N doubles (unaligned) when per point
    const std::uint8_t* freq_re = nullptr;         // N doubles each when per component
    const std::uint8_t* freq_im = nullptr;
    int m = 0;
    std::uint64_t n_spatial = 0, n_frequency = 0;
    std::vector<std::uint8_t> spatial_flags, frequency_flags;       // LSB-first bytes
    std::vector<std::uint8_t> spatial_payload, frequency_payload;   // huffman::encode payloads
    std::vector<EscapeRec> escapes;
};
ParsedArchive parse_archive(const std::uint8_t* bytes, std::size_t len);
// Block directory of a huffman::encode payload (huffman.cpp:156-251): per block its byte offset
// and symbol count; validates the framing.  Returns the total symbol count.
std::uint64_t huffman_blocks(const std::vector<std::uint8_t>& payload,
                             std::vector<std::uint64_t>& block_off,
                             std::vector<std::uint64_t>& block_first);

std::uint32_t crc32c(const std::uint8_t* data, std::size_t len);
// the same on up to 16 host threads (pieces joined by crc32c_combine, deflate.cu)
std::uint32_t crc32c_threads(const std::uint8_t* data, std::uint64_t len);
int host_threads();
std::uint32_t zigzag(std::int32_t v);
// Blockwise canonical Huffman (huffman.cpp:156-251 format)
std::vector<std::uint8_t> huffman_encode(const std::uint32_t* symbols, std::size_t n);
// u64 raw size + zlib stream (streams.cpp:21-32 format)
std::vector<std::uint8_t> outer_compress(const std::uint8_t* raw, std::size_t n, int level);
std::vector<std::uint8_t> write_archive(const ArchiveInput& in);

} // namespace ffcz_host
