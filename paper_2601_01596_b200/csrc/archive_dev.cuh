// Device-assembled .ffcz archive (archive_dev.cu): write_archive (archive.cpp:73-135) whose
// streams are encoded on the GPU from the resident flags and codes.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>

#include "../../include/ffcz_cuda.h"
#include "encode.cuh"

namespace ffcz_gpu {

struct DevArchiveInput {
    int ndim;
    std::uint64_t dims[3];
    int precision;  // 0 f32, 1 f64
    bool spatial_per_point;
    double spatial_global;
    const double* spatial_values;  // N (full field), host or device (bounds_on_device)
    bool freq_per_component;
    double freq_global;
    const double* freq_re;  // N (full spectrum), host or device
    const double* freq_im;
    bool bounds_on_device;
    int m;
    bool converged;
    const unsigned char* spatial_flags;    std::uint64_t spatial_flag_bytes;    // device
    const unsigned char* frequency_flags;  std::uint64_t frequency_flag_bytes;  // device
    std::uint64_t n_spatial, n_frequency;
    const int* spatial_codes;    // device, n_spatial
    const int* frequency_codes;  // device, 2 * n_frequency (Re, Im interleaved)
    const ffcz_cuda_escape* escapes;  // host
    std::uint64_t n_escapes;
};

// Writes the archive into host_alloc(total + 1) (the caller's pinned pool); synchronises the
// scratch stream.
void write_archive_device(DevScratch& s, const DevArchiveInput& in,
                          const std::function<void*(std::size_t)>& host_alloc, std::uint8_t** out,
                          std::uint64_t* out_len);

}  // namespace ffcz_gpu
