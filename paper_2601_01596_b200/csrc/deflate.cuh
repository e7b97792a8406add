// Device outer stage of the .ffcz archive: the streams' zlib framing (streams.cpp:21-32) and the
// header CRC-32C (archive.cpp:61-71 crc32c, FORMAT.md) computed on the GPU.
#pragma once

#include <cstdint>

#include "encode.cuh"

namespace ffcz_gpu {

// outer_compress (streams.cpp:21-32) framing of n device bytes: u64 raw size, then a zlib stream
// that zlib's uncompress() (the reference's outer_decompress, streams.cpp:34-48) accepts.  Every
// 32 KiB of input is one deflate block, encoded by one CTA as the smaller of a stored block and
// a fixed-Huffman block of literals + distance-1 runs (byte-aligned by an empty stored block,
// as Z_SYNC_FLUSH does), so blocks concatenate at byte offsets from one scan.  The adler-32
// trailer is combined from per-block sums.  Asynchronous: the framed stream's length is written
// to *len_dev; *out receives a device buffer (named `tag` in the scratch) of worst-case size
// deflate_bound(n).
void deflate_device(DevScratch& s, const char* tag, const unsigned char* in, unsigned long long n,
                    unsigned char** out, unsigned long long* len_dev);
unsigned long long deflate_bound(unsigned long long n);

// Raw CRC-32C register of n device bytes from state 0 (no pre / post inversion), XOR-ed into
// *acc_dev (which the caller zeroes).  Asynchronous.  crc32c_from_raw() turns it into the
// standard CRC-32C; crc32c_combine() joins standard CRCs of consecutive pieces (host).
void crc32c_raw_device(cudaStream_t st, const unsigned char* p, unsigned long long n,
                       unsigned* acc_dev);

} // namespace ffcz_gpu

namespace ffcz_host {
std::uint32_t crc32c_from_raw(std::uint32_t raw, std::uint64_t n);
std::uint32_t crc32c_combine(std::uint32_t crc1, std::uint32_t crc2, std::uint64_t len2);
// x^(8 * 2^k * unit) mod P (reflected), k < 64, for the device kernels' shift tables
std::uint32_t crc32c_x8n(std::uint64_t n);
std::uint32_t crc32c_multmodp(std::uint32_t a, std::uint32_t b);
} // namespace ffcz_host
