// Host side of the long-line transforms (fft_large.cuh): factorisation, pass sequencing,
// Bluestein, packed real rows.  FP64 and FP32 instantiations.
#include <algorithm>

#include "fft_large.cuh"
#include "fft_plan.cuh"

namespace ffcz_gpu {

namespace large {

std::vector<int> factor(long long L) {
    std::vector<int> r;
    long long m = L;
    while (m % 8 == 0) { r.push_back(8); m /= 8; }
    if (m % 4 == 0) { r.push_back(4); m /= 4; }
    if (m % 2 == 0) { r.push_back(2); m /= 2; }
    for (int p = 3; p <= 64 && m > 1; p += 2)
        while (m % p == 0) { r.push_back(p); m /= p; }
    if (m > 1) return {};  // a prime factor above 64: Bluestein
    return r;
}

long long pow2_ceil(long long v) {
    long long p = 1;
    while (p < v) p <<= 1;
    return p;
}

namespace {

unsigned grid_of(long long n) {
    return static_cast<unsigned>(std::max<long long>(1, std::min<long long>((n + 255) / 256, 148 * 32)));
}

template <class T>
void stage(int r, const cplx<T>* in, LineAddr ai, cplx<T>* out, LineAddr ao, long long nl,
           long long L, long long ns, const cplx<T>* W, int dir, const int* gate, cudaStream_t st) {
    const unsigned g = grid_of(nl * (L / r));
    switch (r) {
#define R_CASE(R)                                                                              \
    case R:                                                                                    \
        k_stockham<R, T><<<g, 256, 0, st>>>(in, ai, out, ao, nl, L, ns, r, W, dir, gate);      \
        break;
        R_CASE(2) R_CASE(3) R_CASE(4) R_CASE(5) R_CASE(7) R_CASE(8)
#undef R_CASE
        default:
            k_stockham<0, T><<<g, 256, 0, st>>>(in, ai, out, ao, nl, L, ns, r, W, dir, gate);
    }
    FFCZ_LAUNCH_CHECK();
}

template <class T>
// Device scratch of one call: plain allocations, released after the stream has drained (these
// passes are a correctness path for rare extents; a stream-ordered pool allocation here was the
// one suspect left for an intermittent wrong Bluestein result seen in two full-suite runs)
struct Scratch {
    cudaStream_t st;
    std::vector<void*> bufs;
    cplx<T>* get(long long n) {
        void* p = nullptr;
        FFCZ_CUDA_CHECK(cudaMalloc(&p, sizeof(cplx<T>) * std::max<long long>(1, n)));
        bufs.push_back(p);
        return static_cast<cplx<T>*>(p);
    }
    ~Scratch() {
        if (bufs.empty()) return;
        cudaStreamSynchronize(st);
        for (void* p : bufs) cudaFree(p);
    }
};

LineAddr compact(long long nl) {
    LineAddr a;
    a.compact = true;
    a.nl = nl;
    return a;
}

}  // namespace
}  // namespace large

template <class T>
void large_lines(long long L, int dir, const cplx<T>* src, LineAddr ai, cplx<T>* dst, LineAddr ao,
                 long long nl, Twiddles<T>& tw, const int* gate, cudaStream_t st) {
    using namespace large;
    large::Scratch<T> sc{st, {}};
    const std::vector<int> rad = factor(L);
    if (L == 1) {
        k_copy_lines<T><<<grid_of(nl), 256, 0, st>>>(src, ai, dst, ao, nl, 1, T(1), gate);
        FFCZ_LAUNCH_CHECK();
        return;
    }
    if (!rad.empty()) {
        const cplx<T>* W = tw.table_for(L);
        const int S = static_cast<int>(rad.size());
        const LineAddr ac = compact(nl);
        cplx<T>* buf[2] = {sc.get(nl * L), S > 2 ? sc.get(nl * L) : nullptr};
        const cplx<T>* in = src;
        LineAddr a_in = ai;
        long long ns = 1;
        for (int s = 0; s < S; ++s) {
            const bool last = s == S - 1;
            cplx<T>* out = last ? dst : buf[s & 1];
            LineAddr a_out = last ? ao : ac;
            if (last && S == 1 && src == dst) {  // one out-of-place pass, in place: via scratch
                out = buf[0];
                a_out = ac;
            }
            stage<T>(rad[s], in, a_in, out, a_out, nl, L, ns, W, dir, gate, st);
            ns *= rad[s];
            in = out;
            a_in = a_out;
        }
        if (S == 1 && src == dst) {
            k_copy_lines<T><<<grid_of(nl * L), 256, 0, st>>>(buf[0], ac, dst, ao, nl, L, T(1), gate);
            FFCZ_LAUNCH_CHECK();
        }
        return;
    }
    // Bluestein: circular convolution of length M >= 2L - 1 with power-of-two passes
    const long long M = pow2_ceil(2 * L - 1);
    const cplx<T>* W2 = tw.table_for(2 * L);
    const LineAddr ac = compact(nl), a1 = compact(1);
    cplx<T>* a = sc.get(nl * M);
    cplx<T>* b = sc.get(M);
    k_chirp_in<T><<<grid_of(nl * M), 256, 0, st>>>(src, ai, a, nl, L, M, W2, dir, gate);
    k_chirp_kernel<T><<<grid_of(M), 256, 0, st>>>(b, L, M, W2, dir, gate);
    FFCZ_LAUNCH_CHECK();
    large_lines<T>(M, -1, b, a1, b, a1, 1, tw, gate, st);
    large_lines<T>(M, -1, a, ac, a, ac, nl, tw, gate, st);
    k_pointwise<T><<<grid_of(nl * M), 256, 0, st>>>(a, b, nl, M, gate);
    FFCZ_LAUNCH_CHECK();
    large_lines<T>(M, +1, a, ac, a, ac, nl, tw, gate, st);
    k_chirp_out<T><<<grid_of(nl * L), 256, 0, st>>>(a, dst, ao, nl, L, W2, dir,
                                                    T(1) / static_cast<T>(M), gate);
    FFCZ_LAUNCH_CHECK();
}

template <class T>
void large_row_r2c(long long n2, const T* in, long long in_stride, cplx<T>* out,
                   long long out_stride, long long nrows, Twiddles<T>& tw, const int* gate,
                   cudaStream_t st) {
    using namespace large;
    large::Scratch<T> sc{st, {}};
    const bool even = (n2 & 1) == 0;
    const long long Lz = even ? n2 / 2 : n2;
    cplx<T>* z = sc.get(nrows * Lz);
    const LineAddr ac = compact(nrows);
    k_pack_rows<T><<<grid_of(nrows * Lz), 256, 0, st>>>(in, in_stride, z, nrows, n2, gate);
    FFCZ_LAUNCH_CHECK();
    large_lines<T>(Lz, -1, z, ac, z, ac, nrows, tw, gate, st);
    if (even)
        k_r2c_split<T><<<grid_of(nrows * (Lz + 1)), 256, 0, st>>>(z, out, out_stride, nrows, n2,
                                                                  tw.table_for(n2), gate);
    else
        k_r2c_take<T><<<grid_of(nrows * (n2 / 2 + 1)), 256, 0, st>>>(z, out, out_stride, nrows,
                                                                     n2, gate);
    FFCZ_LAUNCH_CHECK();
}

template <class T>
void large_row_c2r(long long n2, const cplx<T>* in, long long in_stride, T* out,
                   long long out_stride, long long nrows, T scale, Twiddles<T>& tw,
                   const int* gate, cudaStream_t st) {
    using namespace large;
    large::Scratch<T> sc{st, {}};
    const bool even = (n2 & 1) == 0;
    const long long Lz = even ? n2 / 2 : n2;
    cplx<T>* z = sc.get(nrows * Lz);
    const LineAddr ac = compact(nrows);
    k_c2r_merge<T><<<grid_of(nrows * Lz), 256, 0, st>>>(in, in_stride, z, nrows, n2,
                                                        tw.table_for(n2), gate);
    FFCZ_LAUNCH_CHECK();
    large_lines<T>(Lz, +1, z, ac, z, ac, nrows, tw, gate, st);
    k_unpack_rows<T><<<grid_of(nrows * Lz), 256, 0, st>>>(z, out, out_stride, nrows, n2, scale,
                                                          gate);
    FFCZ_LAUNCH_CHECK();
}

#define FFCZ_LARGE_INST(T)                                                                     \
    template void large_lines<T>(long long, int, const cplx<T>*, LineAddr, cplx<T>*, LineAddr,  \
                                 long long, Twiddles<T>&, const int*, cudaStream_t);            \
    template void large_row_r2c<T>(long long, const T*, long long, cplx<T>*, long long,         \
                                   long long, Twiddles<T>&, const int*, cudaStream_t);          \
    template void large_row_c2r<T>(long long, const cplx<T>*, long long, T*, long long,         \
                                   long long, T, Twiddles<T>&, const int*, cudaStream_t);
FFCZ_LARGE_INST(double)
FFCZ_LARGE_INST(float)
#undef FFCZ_LARGE_INST

}  // namespace ffcz_gpu
