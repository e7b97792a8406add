// Device metrics kernels (metrics.cu); the C-ABI entry points are in engine.cu.
#pragma once

#include <cstring>

#include "kernels.cuh"

namespace ffcz_gpu {

constexpr int kShellSmemBins = 2048;  // per-CTA shared-memory histogram (32 KB) up to this many bins

struct FieldStats {
    double sum[3];                 // sum (y - x)^2, sum x, unused
    unsigned long long max_abs_x;  // double bits (non-negative)
    unsigned long long max_abs_eps;
    unsigned long long lo, hi;     // ord_bits-encoded min / max of x
};
struct SpecStats {
    double sum[2];                 // sum |X|^2, sum |X - Y|^2 over the FULL spectrum
    unsigned long long max_abs_X, max_abs_D;
};

// ordered-integer encoding of a double of any sign (unsigned order == double order)
__device__ __forceinline__ unsigned long long ord_bits(double x) {
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(x));
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
inline double ord_bits_decode(unsigned long long u) {
    u = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
    double d;
    std::memcpy(&d, &u, 8);
    return d;
}

template <class TI>
__global__ void k_field_stats(const TI* __restrict__ x, const TI* __restrict__ y, long long N,
                              double* __restrict__ eps_out, FieldStats* st);
__global__ void k_spec_sums(const double2* __restrict__ X, const double2* __restrict__ Y,
                            const double2* __restrict__ D, HalfGeom hg, SpecStats* st);
__global__ void k_spectrum_bound(const double2* __restrict__ X, long long d0, long long d1,
                                 long long n2, int P, double scale, double floor_v,
                                 double* __restrict__ delta);
__global__ void k_shell_power(const double2* __restrict__ X, long long d0, long long d1,
                              long long n2, int P, int nbins, double* __restrict__ power,
                              unsigned long long* __restrict__ counts);
template <class TI>
__global__ void k_fluct(const TI* __restrict__ x, long long N, double mean, int fallback,
                        double* __restrict__ out);

} // namespace ffcz_gpu
