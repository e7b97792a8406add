// Shared device types and helpers for the FFCz B200 engine (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace ffcz_gpu {

// ---- status / errors ------------------------------------------------------------------------

// Error carrying a C-ABI status code (include/ffcz_cuda.h); thrown inside the library and
// converted at the C boundary.
struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

inline unsigned long long& launch_ticks() {
    static thread_local unsigned long long t = 0;
    return t;
}

enum Status { kOk = 0, kValidation = 1, kSymmetry = 2, kFormat = 3, kIo = 4, kCuda = 5,
              kUnsupported = 6, kOom = 7, kUndefined = 8 };

#define FFCZ_CUDA_CHECK(expr)                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (expr);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            if (e_ == cudaErrorMemoryAllocation)                                               \
                throw ::ffcz_gpu::Error(::ffcz_gpu::kOom, std::string(#expr ": ") +            \
                                                              cudaGetErrorString(e_));         \
            throw ::ffcz_gpu::Error(::ffcz_gpu::kCuda,                                         \
                                    std::string(#expr ": ") + cudaGetErrorString(e_));         \
        }                                                                                      \
    } while (0)

// kernel launches checked on this host thread (the slab ops report their count from it)
#define FFCZ_LAUNCH_CHECK()                                                                    \
    do {                                                                                       \
        ++::ffcz_gpu::launch_ticks();                                                          \
        FFCZ_CUDA_CHECK(cudaGetLastError());                                                   \
    } while (0)

// ---- complex ---------------------------------------------------------------------------------

template <class T> struct cvec;
template <> struct cvec<float> { using type = float2; };
template <> struct cvec<double> { using type = double2; };
template <class T> using cplx = typename cvec<T>::type;

template <class T>
__device__ __forceinline__ cplx<T> mkc(T x, T y) {
    cplx<T> r;
    r.x = x;
    r.y = y;
    return r;
}
template <class C> __device__ __forceinline__ C cadd(C a, C b) { a.x += b.x; a.y += b.y; return a; }
template <class C> __device__ __forceinline__ C csub(C a, C b) { a.x -= b.x; a.y -= b.y; return a; }
template <class C> __device__ __forceinline__ C cconj(C a) { a.y = -a.y; return a; }
template <class C> __device__ __forceinline__ C cmul(C a, C b) {
    C r;
    r.x = a.x * b.x - a.y * b.y;
    r.y = a.x * b.y + a.y * b.x;
    return r;
}
// a * conj(b)
template <class C> __device__ __forceinline__ C cmulc(C a, C b) {
    C r;
    r.x = a.x * b.x + a.y * b.y;
    r.y = a.y * b.x - a.x * b.y;
    return r;
}
template <class C> __device__ __forceinline__ C cscale(C a, decltype(a.x) s) { a.x *= s; a.y *= s; return a; }
// a * i
template <class C> __device__ __forceinline__ C cmuli(C a) { C r; r.x = -a.y; r.y = a.x; return r; }
// a * (-i)
template <class C> __device__ __forceinline__ C cmulmi(C a) { C r; r.x = a.y; r.y = -a.x; return r; }

// ---- misc -----------------------------------------------------------------------------------

__device__ __forceinline__ unsigned long long dbits(double v) {
    return static_cast<unsigned long long>(__double_as_longlong(v));
}
__device__ __forceinline__ double bitsd(unsigned long long b) {
    return __longlong_as_double(static_cast<long long>(b));
}

// Kernels launched speculatively inside the device-resident loop return immediately once the
// convergence decision has set *gate (no host sync per iteration).
__device__ __forceinline__ bool gated(const int* gate) {
    return gate != nullptr && *reinterpret_cast<const volatile int*>(gate) != 0;
}

__host__ __device__ constexpr int ilog2_c(long long v) { return v <= 1 ? 0 : 1 + ilog2_c(v / 2); }
__host__ __device__ constexpr bool is_pow2_c(long long v) { return v > 0 && (v & (v - 1)) == 0; }

inline bool is_pow2(uint64_t v) { return v && !(v & (v - 1)); }
inline uint64_t round_up(uint64_t v, uint64_t m) { return (v + m - 1) / m * m; }

} // namespace ffcz_gpu
