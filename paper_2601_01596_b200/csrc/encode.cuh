// Device-side edit encoding (encode.cu): blockwise canonical Huffman of zigzag'ed int32 codes,
// byte-identical to the reference's huffman::encode (huffman.cpp:156-251).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <functional>

namespace ffcz_gpu {

// Named device scratch buffers (the engine context's pool) and the stream to run on.
struct DevScratch {
    cudaStream_t stream;
    std::function<void*(const char*, size_t)> get;
};

// Encodes n device int32 codes; returns the payload length and a device pointer to it (valid
// until the next call with the same scratch).  Synchronises the stream twice (run and size
// readbacks).
unsigned long long huffman_encode_device(DevScratch& s, const int* codes, unsigned long long n,
                                         unsigned char** payload);

// Decodes a huffman::encode payload (host bytes + its block directory, archive.hpp
// huffman_blocks) into n int32 codes on the device (unzigzag'ed).  Throws Error(kFormat) on a
// corrupt stream.
void huffman_decode_device(DevScratch& s, const unsigned char* payload, unsigned long long len,
                           const unsigned long long* block_off, const unsigned long long* block_first,
                           long long nb, int* codes_out);

} // namespace ffcz_gpu
