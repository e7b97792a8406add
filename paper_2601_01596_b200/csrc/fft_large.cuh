// Lines too long for the shared-memory passes (fft_engine.cuh / fft_mixed.cuh): power-of-two
// column axes above 4096, other extents above ~6000, rows above 8192 (e.g. the EEG-like 31,000-
// sample 1-D signal of SPEC.md:84; FFTW accepts any extent, transform.cpp:20-50).
//
// Mixed-radix Stockham in global memory: L = r_1 r_2 ... r_S (radix 8 / 4 / 2 for the power of
// two, then 3, 5, 7, then other primes up to 64 as an O(r^2) butterfly), one pass per radix,
// each pass reading and writing every element once (the autosort form: no digit reversal).
// Intermediate passes use a compact j-major scratch layout (element (line l, index j) at
// j * nlines + l: consecutive lines, i.e. consecutive columns, are consecutive addresses, so
// every pass is coalesced for column lines and for rows alike); the first pass reads the field
// layout and the last writes it.  Every twiddle is an exact index into the FP64-derived W_L^q
// table.
//
// Bluestein (chirp-z) when L has a prime factor above 64: X_k = w^{k^2} sum_n (x_n w^{n^2})
// w^{-(k-n)^2}, w = W_{2L}, as a circular convolution of length M = 2^ceil(log2(2L-1)) done with
// the power-of-two Stockham passes; the chirp indices n^2 mod 2L are exact integers.
//
// Long rows: even n2 = 2M packs the real row as z_m = x_2m + i x_2m+1 (one M-point complex
// transform, then the split X_k = Ze_k + W_2M^k Zo_k); odd n2 runs the n2-point complex transform
// of x + 0i.  C2R inverts these steps with the engine's C2R convention (the imaginary parts of
// the k = 0 and Nyquist terms are ignored, the spectrum is extended Hermitian).
#pragma once

#include <vector>

#include "common.cuh"

namespace ffcz_gpu {

template <class T> struct Twiddles;

// Element (line l, index j) of a field-layout line set: l = plane * ncols + col,
// offset = plane * plane_stride + col + j * row_stride; compact: j * nl + l.
struct LineAddr {
    long long row_stride = 0, plane_stride = 0;
    long long ncols = 1;
    long long nl = 1;
    bool compact = true;
    __host__ __device__ long long at(long long l, long long j) const {
        if (compact) return j * nl + l;
        const long long p = l / ncols, c = l - p * ncols;
        return p * plane_stride + c + j * row_stride;
    }
};

namespace large {

// radices of L (each <= 64), or empty when L has a prime factor above 64
std::vector<int> factor(long long L);
long long pow2_ceil(long long v);

template <int R, class T>
__device__ __forceinline__ void dft_r(cplx<T>* v, int r, const cplx<T>* __restrict__ W, long long L,
                                      int dir) {
    constexpr int RM = R ? R : 64;
    cplx<T> y[RM];
    const int rr = R ? R : r;
    const long long step = L / rr;
    for (int a = 0; a < rr; ++a) {
        cplx<T> acc = v[0];
        for (int q = 1; q < rr; ++q) {
            cplx<T> w = W[((a * q) % rr) * step];
            if (dir > 0) w.y = -w.y;
            acc = cadd(acc, cmul(v[q], w));
        }
        y[a] = acc;
    }
    for (int a = 0; a < rr; ++a) v[a] = y[a];
}

// one Stockham pass: ns = product of the radices already applied
template <int R, class T>
__global__ void k_stockham(const cplx<T>* __restrict__ in, LineAddr ai, cplx<T>* __restrict__ out,
                           LineAddr ao, long long nl, long long L, long long ns, int r,
                           const cplx<T>* __restrict__ W, int dir, const int* gate) {
    if (gated(gate)) return;
    constexpr int RM = R ? R : 64;
    const int rr = R ? R : r;
    const long long Lr = L / rr;
    const long long total = nl * Lr;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long l = t % nl, j = t / nl;
        cplx<T> v[RM];
        const long long k = j % ns;
        const long long tstep = L / (ns * rr);  // W_{ns r}^{k q} = W_L^{k q L / (ns r)}
        for (int q = 0; q < rr; ++q) {
            cplx<T> x = in[ai.at(l, j + q * Lr)];
            if (ns > 1 && q) {
                cplx<T> w = W[(k * q * tstep) % L];
                if (dir > 0) w.y = -w.y;
                x = cmul(x, w);
            }
            v[q] = x;
        }
        dft_r<R, T>(v, rr, W, L, dir);
        const long long base = (j / ns) * ns * rr + k;
        for (int a = 0; a < rr; ++a) out[ao.at(l, base + a * ns)] = v[a];
    }
}

template <class T>
__global__ void k_copy_lines(const cplx<T>* __restrict__ in, LineAddr ai, cplx<T>* __restrict__ out,
                             LineAddr ao, long long nl, long long L, T scale, const int* gate) {
    if (gated(gate)) return;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nl * L;
         t += (long long)gridDim.x * blockDim.x) {
        const long long l = t % nl, j = t / nl;
        out[ao.at(l, j)] = cscale(in[ai.at(l, j)], scale);
    }
}

// Bluestein helpers: W2 = W_{2L}^q table
template <class T>
__global__ void k_chirp_in(const cplx<T>* __restrict__ in, LineAddr ai, cplx<T>* __restrict__ a,
                           long long nl, long long L, long long M, const cplx<T>* __restrict__ W2,
                           int dir, const int* gate) {
    if (gated(gate)) return;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nl * M;
         t += (long long)gridDim.x * blockDim.x) {
        const long long l = t % nl, n = t / nl;
        cplx<T> v = mkc<T>(T(0), T(0));
        if (n < L) {
            cplx<T> w = W2[static_cast<long long>((static_cast<unsigned long long>(n) * n) % (2 * L))];
            if (dir > 0) w.y = -w.y;
            v = cmul(in[ai.at(l, n)], w);
        }
        a[n * nl + l] = v;
    }
}

template <class T>
__global__ void k_chirp_kernel(cplx<T>* __restrict__ b, long long L, long long M,
                               const cplx<T>* __restrict__ W2, int dir, const int* gate) {
    if (gated(gate)) return;
    for (long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x; m < M;
         m += (long long)gridDim.x * blockDim.x) {
        const long long d = m < L ? m : (M - m < L ? M - m : -1);
        cplx<T> v = mkc<T>(T(0), T(0));
        if (d >= 0) {
            v = W2[static_cast<long long>((static_cast<unsigned long long>(d) * d) % (2 * L))];
            if (dir < 0) v.y = -v.y;  // w^{-d^2} for the forward transform
        }
        b[m] = v;
    }
}

template <class T>
__global__ void k_pointwise(cplx<T>* __restrict__ a, const cplx<T>* __restrict__ fb, long long nl,
                            long long M, const int* gate) {
    if (gated(gate)) return;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nl * M;
         t += (long long)gridDim.x * blockDim.x)
        a[t] = cmul(a[t], fb[t / nl]);
}

template <class T>
__global__ void k_chirp_out(const cplx<T>* __restrict__ c, cplx<T>* __restrict__ out, LineAddr ao,
                            long long nl, long long L, const cplx<T>* __restrict__ W2, int dir,
                            T scale, const int* gate) {
    if (gated(gate)) return;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nl * L;
         t += (long long)gridDim.x * blockDim.x) {
        const long long l = t % nl, k = t / nl;
        cplx<T> w = W2[static_cast<long long>((static_cast<unsigned long long>(k) * k) % (2 * L))];
        if (dir > 0) w.y = -w.y;
        out[ao.at(l, k)] = cscale(cmul(c[k * nl + l], w), scale);
    }
}

// packed real rows: z_m = x_2m + i x_2m+1 into compact lines (even n2), or x + 0i (odd n2)
template <class T>
__global__ void k_pack_rows(const T* __restrict__ x, long long in_stride, cplx<T>* __restrict__ z,
                            long long nrows, long long n2, const int* gate) {
    if (gated(gate)) return;
    const bool even = (n2 & 1) == 0;
    const long long Lz = even ? n2 / 2 : n2;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nrows * Lz;
         t += (long long)gridDim.x * blockDim.x) {
        const long long r = t % nrows, m = t / nrows;
        const T* row = x + r * in_stride;
        z[m * nrows + r] = even ? mkc<T>(row[2 * m], row[2 * m + 1]) : mkc<T>(row[m], T(0));
    }
}

// R2C split of the packed transform Z (compact) into the half row X_0..X_M (even n2)
template <class T>
__global__ void k_r2c_split(const cplx<T>* __restrict__ Z, cplx<T>* __restrict__ out,
                            long long out_stride, long long nrows, long long n2,
                            const cplx<T>* __restrict__ Wn2, const int* gate) {
    if (gated(gate)) return;
    const long long M = n2 / 2;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nrows * (M + 1);
         t += (long long)gridDim.x * blockDim.x) {
        const long long r = t % nrows, k = t / nrows;
        const cplx<T> a = Z[(k % M) * nrows + r];
        const cplx<T> b = cconj(Z[((M - k) % M) * nrows + r]);
        const cplx<T> ze = cscale(cadd(a, b), T(0.5));
        const cplx<T> zo = cscale(cmulmi(csub(a, b)), T(0.5));  // (a - b) / (2i)
        out[r * out_stride + k] = cadd(ze, cmul(Wn2[k], zo));
    }
}

// odd n2: keep X_0..X_{n2/2} of the complex transform
template <class T>
__global__ void k_r2c_take(const cplx<T>* __restrict__ Z, cplx<T>* __restrict__ out,
                           long long out_stride, long long nrows, long long n2, const int* gate) {
    if (gated(gate)) return;
    const long long H = n2 / 2 + 1;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nrows * H;
         t += (long long)gridDim.x * blockDim.x) {
        const long long r = t % nrows, k = t / nrows;
        out[r * out_stride + k] = Z[k * nrows + r];
    }
}

// C2R merge: half rows -> packed Z (even n2), or the Hermitian-extended full spectrum (odd n2)
template <class T>
__global__ void k_c2r_merge(const cplx<T>* __restrict__ X, long long in_stride,
                            cplx<T>* __restrict__ Z, long long nrows, long long n2,
                            const cplx<T>* __restrict__ Wn2, const int* gate) {
    if (gated(gate)) return;
    const bool even = (n2 & 1) == 0;
    const long long M = even ? n2 / 2 : n2;
    const long long H = n2 / 2;  // last stored index
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nrows * M;
         t += (long long)gridDim.x * blockDim.x) {
        const long long r = t % nrows, k = t / nrows;
        const cplx<T>* row = X + r * in_stride;
        auto xk = [&](long long q) {  // X_q with the C2R convention (real DC and Nyquist)
            cplx<T> v = row[q];
            if (q == 0 || (even && q == H)) v.y = T(0);
            return v;
        };
        cplx<T> z;
        if (even) {
            const cplx<T> a = xk(k), b = cconj(xk(M - k));
            const cplx<T> ze = cscale(cadd(a, b), T(0.5));
            const cplx<T> zo = cscale(cmulc(csub(a, b), Wn2[k]), T(0.5));  // * W_2M^{-k}
            z = cadd(ze, cmuli(zo));
        } else {
            z = k <= H ? xk(k) : cconj(xk(n2 - k));
        }
        Z[k * nrows + r] = z;
    }
}

template <class T>
__global__ void k_unpack_rows(const cplx<T>* __restrict__ z, T* __restrict__ x,
                              long long out_stride, long long nrows, long long n2, T scale, const int* gate) {
    if (gated(gate)) return;
    const bool even = (n2 & 1) == 0;
    const long long Lz = even ? n2 / 2 : n2;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nrows * Lz;
         t += (long long)gridDim.x * blockDim.x) {
        const long long r = t % nrows, m = t / nrows;
        const cplx<T> v = z[m * nrows + r];
        T* row = x + r * out_stride;
        if (even) {
            row[2 * m] = T(2) * v.x * scale;
            row[2 * m + 1] = T(2) * v.y * scale;
        } else {
            row[m] = v.x * scale;
        }
    }
}

}  // namespace large

// Complex transform of nl lines of length L (dir -1 forward, +1 inverse, unnormalised) from the
// `ai` layout of src to the `ao` layout of dst (src == dst allowed).  Scratch: per call,
// (plain cudaMalloc, freed after the stream drains).
template <class T>
void large_lines(long long L, int dir, const cplx<T>* src, LineAddr ai, cplx<T>* dst, LineAddr ao,
                 long long nl, Twiddles<T>& tw, const int* gate, cudaStream_t st);

template <class T>
void large_row_r2c(long long n2, const T* in, long long in_stride, cplx<T>* out,
                   long long out_stride, long long nrows, Twiddles<T>& tw, const int* gate,
                   cudaStream_t st);
template <class T>
void large_row_c2r(long long n2, const cplx<T>* in, long long in_stride, T* out,
                   long long out_stride, long long nrows, T scale, Twiddles<T>& tw,
                   const int* gate, cudaStream_t st);

}  // namespace ffcz_gpu
