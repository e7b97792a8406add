// write_archive (/root/reference/proj/core/src/archive.cpp:73-135, FORMAT.md) with every
// stream produced on the device: the flag bitmaps and the int32 codes never leave HBM until the
// finished archive is copied into the caller's pinned result buffer.
//   index streams: zigzag + canonical Huffman (encode.cu, byte-identical to huffman::encode),
//                  then the device outer stage (deflate.cu)
//   flag streams:  the device outer stage over the resident LSB-first flag bitmaps
//   header CRC-32C: prefix and tail on the host; the bound arrays (N doubles each when per
//                  point / per component) on the device when they are resident there
//                  (crc32c_raw_device), else on host threads; joined by crc32c_combine
// One host sync for the four stream lengths, then every piece lands at its offset in the pinned
// archive (D2H for device pieces, threaded memcpy for host bound arrays).
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <chrono>
#include <cstring>
#include <thread>
#include <vector>

#include "archive.hpp"
#include "archive_dev.cuh"
#include "common.cuh"
#include "deflate.cuh"

namespace ffcz_gpu {

namespace {

template <class T>
void put(std::vector<std::uint8_t>& out, T v) {
    std::uint8_t b[sizeof(T)];
    std::memcpy(b, &v, sizeof(T));
    out.insert(out.end(), b, b + sizeof(T));
}

void memcpy_threads(std::uint8_t* dst, const std::uint8_t* src, std::uint64_t n) {
    const int T = n < (std::uint64_t(64) << 20) ? 1 : ffcz_host::host_threads();
    if (T == 1) {
        std::memcpy(dst, src, n);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) {
        const std::uint64_t a = n * t / T, b = n * (t + 1) / T;
        th.emplace_back([=] { std::memcpy(dst + a, src + a, b - a); });
    }
    for (auto& x : th) x.join();
}

}  // namespace

void write_archive_device(DevScratch& s, const DevArchiveInput& in,
                          const std::function<void*(std::size_t)>& host_alloc, std::uint8_t** out,
                          std::uint64_t* out_len) {
    cudaStream_t st = s.stream;
    // FFCZ_DEBUG_TIMING=1: host timestamps of the archive's phases on stderr (synchronises)
    static const bool dbg_on = std::getenv("FFCZ_DEBUG_TIMING") != nullptr;
    const auto t_start = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!dbg_on) return;
        cudaStreamSynchronize(st);
        std::fprintf(stderr, "[ffcz] archive: %-22s %9.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                               t_start).count());
    };
    std::uint64_t N = 1;
    for (int a = 0; a < in.ndim; ++a) N *= in.dims[a];

    // host-resident bound arrays: CRC-32C on host threads while the device encodes the streams
    std::uint32_t host_bcrc[3] = {0, 0, 0};
    std::thread host_crc;
    if (!in.bounds_on_device) {
        host_crc = std::thread([&] {
            const double* arr[3] = {in.spatial_per_point ? in.spatial_values : nullptr,
                                    in.freq_per_component ? in.freq_re : nullptr,
                                    in.freq_per_component && in.freq_im != in.freq_re ? in.freq_im
                                                                                       : nullptr};
            for (int k = 0; k < 3; ++k)
                if (arr[k])
                    host_bcrc[k] =
                        ffcz_host::crc32c_threads(reinterpret_cast<const std::uint8_t*>(arr[k]), 8 * N);
        });
    }
    struct Join {
        std::thread& t;
        ~Join() { if (t.joinable()) t.join(); }
    } join_guard{host_crc};

    // ---- streams on the device: sf, ff, si, fi (archive.cpp:114-121 order) ---------------------
    auto* lens = static_cast<unsigned long long*>(s.get("arc_lens", 4 * 8));
    auto* crc_acc = static_cast<unsigned*>(s.get("arc_crc", 3 * 4));
    FFCZ_CUDA_CHECK(cudaMemsetAsync(crc_acc, 0, 3 * 4, st));
    unsigned char* dst_ptr[4] = {};
    deflate_device(s, "arc_sf", in.spatial_flags, in.spatial_flag_bytes, &dst_ptr[0], lens + 0);
    deflate_device(s, "arc_ff", in.frequency_flags, in.frequency_flag_bytes, &dst_ptr[1], lens + 1);
    mark("flag streams");
    unsigned char* pay = nullptr;
    unsigned long long pl = huffman_encode_device(s, in.spatial_codes, in.n_spatial, &pay);
    deflate_device(s, "arc_si", pay, pl, &dst_ptr[2], lens + 2);
    mark("spatial index stream");
    pl = huffman_encode_device(s, in.frequency_codes, 2 * in.n_frequency, &pay);
    mark("frequency huffman");
    deflate_device(s, "arc_fi", pay, pl, &dst_ptr[3], lens + 3);
    mark("frequency outer stage");

    // ---- bound arrays: raw CRC on the device when resident there ---------------------------
    const double* arrays[3] = {in.spatial_per_point ? in.spatial_values : nullptr,
                               in.freq_per_component ? in.freq_re : nullptr,
                               in.freq_per_component ? in.freq_im : nullptr};
    const bool im_is_re = arrays[2] && arrays[2] == arrays[1];
    if (in.bounds_on_device) {
        for (int k = 0; k < 3; ++k)
            if (arrays[k] && !(k == 2 && im_is_re))
                crc32c_raw_device(st, reinterpret_cast<const unsigned char*>(arrays[k]), 8 * N,
                                  crc_acc + k);
    }
    unsigned long long hl[4];
    unsigned hcrc[3];
    FFCZ_CUDA_CHECK(cudaMemcpyAsync(hl, lens, sizeof(hl), cudaMemcpyDeviceToHost, st));
    FFCZ_CUDA_CHECK(cudaMemcpyAsync(hcrc, crc_acc, sizeof(hcrc), cudaMemcpyDeviceToHost, st));
    FFCZ_CUDA_CHECK(cudaStreamSynchronize(st));
    std::uint32_t bcrc[3] = {0, 0, 0};
    if (in.bounds_on_device) {
        for (int k = 0; k < 3; ++k)
            if (arrays[k])
                bcrc[k] = ffcz_host::crc32c_from_raw((k == 2 && im_is_re) ? hcrc[1] : hcrc[k], 8 * N);
    } else {
        host_crc.join();
        for (int k = 0; k < 3; ++k) bcrc[k] = host_bcrc[k];
        if (im_is_re) bcrc[2] = bcrc[1];
    }

    // ---- header (archive.cpp:73-112) -----------------------------------------------------------
    std::vector<std::uint8_t> pre;
    const char magic[4] = {'F', 'F', 'C', 'Z'};
    pre.insert(pre.end(), magic, magic + 4);
    put<std::uint16_t>(pre, 1);
    put<std::uint8_t>(pre, static_cast<std::uint8_t>(in.ndim));
    for (int a = 0; a < in.ndim; ++a) put<std::uint64_t>(pre, in.dims[a]);
    put<std::uint8_t>(pre, static_cast<std::uint8_t>(in.precision));
    std::uint8_t tags = 0;
    if (in.spatial_per_point) tags |= 1u;
    if (in.freq_per_component) tags |= 2u;
    if (in.converged) tags |= 4u;
    put<std::uint8_t>(pre, tags);
    if (!in.spatial_per_point) put<double>(pre, in.spatial_global);
    std::vector<std::uint8_t> mid;  // between the spatial and frequency bound arrays
    if (!in.freq_per_component) put<double>(mid, in.freq_global);
    std::vector<std::uint8_t> tail;
    put<std::uint8_t>(tail, static_cast<std::uint8_t>(in.m));
    put<std::uint64_t>(tail, in.n_spatial);
    put<std::uint64_t>(tail, in.n_frequency);
    for (int k = 0; k < 4; ++k) put<std::uint64_t>(tail, hl[k]);
    put<std::uint64_t>(tail, in.n_escapes);

    // CRC over prefix | E | mid | Re | Im | tail (spatial array precedes `mid`)
    std::uint32_t crc = ffcz_host::crc32c(pre.data(), pre.size());
    if (arrays[0]) crc = ffcz_host::crc32c_combine(crc, bcrc[0], 8 * N);
    if (!mid.empty())
        crc = ffcz_host::crc32c_combine(crc, ffcz_host::crc32c(mid.data(), mid.size()), mid.size());
    for (int k = 1; k < 3; ++k)
        if (arrays[k]) crc = ffcz_host::crc32c_combine(crc, bcrc[k], 8 * N);
    crc = ffcz_host::crc32c_combine(crc, ffcz_host::crc32c(tail.data(), tail.size()), tail.size());
    put<std::uint32_t>(tail, crc);

    std::uint64_t esc_bytes = 0;
    for (std::uint64_t i = 0; i < in.n_escapes; ++i) esc_bytes += in.escapes[i].frequency ? 24 : 16;
    const std::uint64_t nbnd = 8 * N * ((arrays[0] ? 1 : 0) + (arrays[1] ? 2 : 0));
    const std::uint64_t total = pre.size() + mid.size() + nbnd + tail.size() + hl[0] + hl[1] +
                                hl[2] + hl[3] + esc_bytes;
    auto* a = static_cast<std::uint8_t*>(host_alloc(total + 1));
    mark("lengths, CRC, host buffer");
    std::uint64_t off = 0;
    auto put_host = [&](const std::uint8_t* p, std::uint64_t n) {
        std::memcpy(a + off, p, n);
        off += n;
    };
    auto put_array = [&](const double* p) {
        if (in.bounds_on_device)
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(a + off, p, 8 * N, cudaMemcpyDeviceToHost, st));
        else
            memcpy_threads(a + off, reinterpret_cast<const std::uint8_t*>(p), 8 * N);
        off += 8 * N;
    };
    put_host(pre.data(), pre.size());
    if (arrays[0]) put_array(arrays[0]);
    put_host(mid.data(), mid.size());
    if (arrays[1]) {
        put_array(arrays[1]);
        put_array(arrays[2]);
    }
    put_host(tail.data(), tail.size());
    for (int k = 0; k < 4; ++k) {
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(a + off, dst_ptr[k], hl[k], cudaMemcpyDeviceToHost, st));
        off += hl[k];
    }
    for (std::uint64_t i = 0; i < in.n_escapes; ++i) {  // archive.cpp:127-133
        const auto& e = in.escapes[i];
        const std::uint64_t packed = e.index | (e.frequency ? (std::uint64_t(1) << 63) : 0);
        std::memcpy(a + off, &packed, 8);
        std::memcpy(a + off + 8, &e.re, 8);
        off += 16;
        if (e.frequency) {
            std::memcpy(a + off, &e.im, 8);
            off += 8;
        }
    }
    FFCZ_CUDA_CHECK(cudaStreamSynchronize(st));
    mark("pieces copied out");
    *out = a;
    *out_len = total;
}

}  // namespace ffcz_gpu
