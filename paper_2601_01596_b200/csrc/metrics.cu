// Device metrics: the reference's evaluation quantities
// (proj/core/src/metrics.cpp) computed on the device from the half spectrum, for at-scale runs
// where the host restatement would need a full complex spectrum per field.
//
//   k_spectrum_bound   spectrum_bound_to_freq_bounds (metrics.cpp:107-128): FULL-grid Delta
//   k_field_stats      psnr's range / squared error (metrics.cpp:64-79), max |eps|, mean, max |x|
//   k_spec_sums        ssnr's energies (metrics.cpp:81-93), rfe's maxima (metrics.cpp:95-105)
//   k_shell_power      power_spectrum's shell sums and counts (metrics.cpp:11-62)
//
// Half-spectrum entries stand for their conjugate mirrors: weight 2 except on the self-mirror
// planes (last-axis index 0 and n2/2).  Magnitudes of mirror pairs are therefore identical here;
// the reference's c2c spectrum differs between a pair only by FFT round-off.  Sums are reduced
// per CTA and combined with one atomic per CTA (order-dependent in the last bits).
#include "metrics.cuh"

namespace ffcz_gpu {

namespace {

__device__ __forceinline__ int hweight(long long k2, long long n2) {
    return (k2 == 0 || 2 * k2 == n2) ? 1 : 2;
}

template <int NV>
__device__ __forceinline__ void block_reduce_sum(double (&v)[NV], double* dst) {
    __shared__ double sh[NV][32];
    __syncthreads();  // the previous reduction's readers are done with the shared slots
#pragma unroll
    for (int i = 0; i < NV; ++i)
        for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
    if (l == 0)
#pragma unroll
        for (int i = 0; i < NV; ++i) sh[i][w] = v[i];
    __syncthreads();
    if (w == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double x = l < nw ? sh[i][l] : 0.0;
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if (l == 0 && x != 0.0) atomicAdd(&dst[i], x);
        }
    }
}

// max of non-negative doubles via their bit patterns (monotone for x >= 0)
__device__ __forceinline__ void block_reduce_max(double v, unsigned long long* dst) {
    __shared__ double sh[32];
    __syncthreads();
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
    if (l == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        double x = l < nw ? sh[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
        if (l == 0) atomicMax(dst, static_cast<unsigned long long>(__double_as_longlong(x)));
    }
}

__device__ __forceinline__ void block_reduce_minmax(double lo, double hi, unsigned long long* dlo,
                                                    unsigned long long* dhi) {
    // ordered-integer encoding of doubles of any sign: flip all bits of negatives, the sign bit
    // of non-negatives; unsigned order then matches double order
    __shared__ double sl[32], sh_[32];
    __syncthreads();
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
    if (l == 0) sl[w] = lo, sh_[w] = hi;
    __syncthreads();
    if (w == 0) {
        double a = l < nw ? sl[l] : sl[0], b = l < nw ? sh_[l] : sh_[0];
        for (int o = 16; o > 0; o >>= 1) {
            a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if (l == 0) {
            atomicMin(dlo, ord_bits(a));
            atomicMax(dhi, ord_bits(b));
        }
    }
}

} // namespace

// psnr / max_spatial / mean inputs over the spatial fields; eps = y - x (FP64) written when
// eps_out != nullptr (it feeds the rfe transform).
template <class TI>
__global__ void k_field_stats(const TI* __restrict__ x, const TI* __restrict__ y, long long N,
                              double* __restrict__ eps_out, FieldStats* st) {
    double lo = INFINITY, hi = -INFINITY, sums[3] = {0.0, 0.0, 0.0};  // se, sum x, (unused)
    double mx = 0.0, me = 0.0;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < N;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double a = static_cast<double>(x[i]);
        lo = fmin(lo, a);
        hi = fmax(hi, a);
        mx = fmax(mx, fabs(a));
        sums[1] += a;
        if (y) {
            const double d = static_cast<double>(y[i]) - a;
            sums[0] += d * d;
            me = fmax(me, fabs(d));
            if (eps_out) eps_out[i] = d;
        }
    }
    block_reduce_sum<3>(sums, st->sum);
    block_reduce_max(mx, &st->max_abs_x);
    block_reduce_max(me, &st->max_abs_eps);
    block_reduce_minmax(lo, hi, &st->lo, &st->hi);
}

// ssnr energies and rfe maxima on half spectra X (original), Y (reconstructed), D (error).
__global__ void k_spec_sums(const double2* __restrict__ X, const double2* __restrict__ Y,
                            const double2* __restrict__ D, HalfGeom hg, SpecStats* st) {
    double sums[2] = {0.0, 0.0};  // sum |X|^2, sum |X - Y|^2 (full-spectrum weights)
    double mxX = 0.0, mxD = 0.0;
    const long long Nc = hg.rows * hg.H;
    for (long long h = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; h < Nc;
         h += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long off = hg.offset_of(h);
        const long long k2 = off % hg.P;
        const double w = hweight(k2, hg.n2);
        const double2 a = X[off];
        sums[0] += w * (a.x * a.x + a.y * a.y);
        mxX = fmax(mxX, hypot(a.x, a.y));
        if (Y) {
            const double2 b = Y[off];
            const double dx = a.x - b.x, dy = a.y - b.y;
            sums[1] += w * (dx * dx + dy * dy);
        }
        if (D) {
            const double2 d = D[off];
            mxD = fmax(mxD, hypot(d.x, d.y));
        }
    }
    block_reduce_sum<2>(sums, st->sum);
    block_reduce_max(mxX, &st->max_abs_X);
    block_reduce_max(mxD, &st->max_abs_D);
}

// spectrum_bound_to_freq_bounds on the FULL grid from the half spectrum, one thread per STORED
// entry: Delta = max(min(|X_k|, |X_mirror(k)|) * scale, floor) written at k and at its mirror
// (the mirror of a stored entry off the self-mirror planes is not stored and has the same
// magnitude; on the planes k2 = 0 and k2 = n2/2 both partners are stored and the min is taken,
// each thread writing its own k).
__global__ void k_spectrum_bound(const double2* __restrict__ X, long long d0, long long d1,
                                 long long n2, int P, double scale, double floor_v,
                                 double* __restrict__ delta) {
    const long long H = n2 / 2 + 1, Nc = d0 * d1 * H;
    for (long long h = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; h < Nc;
         h += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long k2 = h % H, r = h / H, k1 = r % d1, k0 = r / d1;
        const long long m1 = k1 == 0 ? 0 : d1 - k1, m0 = k0 == 0 ? 0 : d0 - k0;
        const long long m2 = k2 == 0 ? 0 : n2 - k2;
        const double2 a = X[r * P + k2];
        double mag = hypot(a.x, a.y);
        if (m2 < H) {  // self-mirror plane: the partner is stored too
            const double2 b = X[(m0 * d1 + m1) * P + m2];
            mag = fmin(mag, hypot(b.x, b.y));
        }
        const double v = fmax(mag * scale, floor_v);
        delta[r * n2 + k2] = v;
        if (m2 >= H) delta[(m0 * d1 + m1) * n2 + m2] = v;
    }
}

// Shell sums: bin = llround(sqrt(sum_a s_a^2)), s_a the centred frequency (k > d/2 wraps to
// k - d); shared-memory histograms per CTA when the bins fit, else global atomics.
__global__ void k_shell_power(const double2* __restrict__ X, long long d0, long long d1,
                              long long n2, int P, int nbins, double* __restrict__ power,
                              unsigned long long* __restrict__ counts) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const bool shared = nbins > 0 && nbins <= kShellSmemBins;
    double* sp = reinterpret_cast<double*>(smem_raw);
    unsigned long long* sc = reinterpret_cast<unsigned long long*>(sp + (shared ? nbins : 0));
    if (shared) {
        for (int b = threadIdx.x; b < nbins; b += blockDim.x) sp[b] = 0.0, sc[b] = 0;
        __syncthreads();
    }
    const long long H = n2 / 2 + 1, Nc = d0 * d1 * H;
    for (long long h = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; h < Nc;
         h += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long k2 = h % H, r = h / H, k1 = r % d1, k0 = r / d1;
        const double s0 = static_cast<double>(k0 > d0 / 2 ? k0 - d0 : k0);
        const double s1 = static_cast<double>(k1 > d1 / 2 ? k1 - d1 : k1);
        const double s2 = static_cast<double>(k2);  // k2 <= n2/2: never wraps
        const int bin = static_cast<int>(llround(sqrt(s0 * s0 + s1 * s1 + s2 * s2)));
        const double2 a = X[r * P + k2];
        const int w = hweight(k2, n2);
        const double p = w * (a.x * a.x + a.y * a.y);
        if (shared) {
            atomicAdd(&sp[bin], p);
            atomicAdd(&sc[bin], static_cast<unsigned long long>(w));
        } else {
            atomicAdd(&power[bin], p);
            atomicAdd(&counts[bin], static_cast<unsigned long long>(w));
        }
    }
    if (shared) {
        __syncthreads();
        for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
            if (sp[b] != 0.0) atomicAdd(&power[b], sp[b]);
            if (sc[b]) atomicAdd(&counts[b], sc[b]);
        }
    }
}

// fluctuation field of power_spectrum: (x - mean) / mean, or x - mean under the zero-mean guard
template <class TI>
__global__ void k_fluct(const TI* __restrict__ x, long long N, double mean, int fallback,
                        double* __restrict__ out) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < N;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double v = static_cast<double>(x[i]) - mean;
        out[i] = fallback ? v : v / mean;
    }
}

template __global__ void k_field_stats<float>(const float*, const float*, long long, double*, FieldStats*);
template __global__ void k_field_stats<double>(const double*, const double*, long long, double*, FieldStats*);
template __global__ void k_fluct<float>(const float*, long long, double, int, double*);
template __global__ void k_fluct<double>(const double*, long long, double, int, double*);

} // namespace ffcz_gpu
