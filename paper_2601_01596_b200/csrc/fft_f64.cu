// FP64 instantiations of the FFT engine + shared host helpers (geometry, twiddle tables).
#include <cmath>

#include "fft_dispatch.cuh"

namespace ffcz_gpu {

Geometry make_geometry(int ndim, const uint64_t* dims, int pitch_align) {
    if (ndim < 1 || ndim > 3)
        throw Error(kValidation, "dims must have 1 to 3 axes, got " + std::to_string(ndim));
    Geometry g;
    g.ndim = ndim;
    for (int a = 0; a < ndim; ++a) {
        if (dims[a] == 0) throw Error(kValidation, "dims must have positive extents");
        g.d[3 - ndim + a] = static_cast<long long>(dims[a]);
    }
    g.N = g.d[0] * g.d[1] * g.d[2];
    g.rows = g.d[0] * g.d[1];
    g.n2 = g.d[2];
    g.H = static_cast<int>(g.n2 / 2 + 1);
    g.P = static_cast<int>(round_up(g.H, pitch_align));
    return g;
}

template <class T>
void Twiddles<T>::init() {
    std::lock_guard<std::mutex> lk(mu);
    if (W) return;
    std::vector<cplx<T>> h(kLmax);
    for (int q = 0; q < kLmax; ++q) {
        const long double a = -2.0L * 3.14159265358979323846264338327950288L * q / kLmax;
        h[q].x = static_cast<T>(std::cos(a));
        h[q].y = static_cast<T>(std::sin(a));
    }
    FFCZ_CUDA_CHECK(cudaMalloc(&W, sizeof(cplx<T>) * kLmax));
    FFCZ_CUDA_CHECK(cudaMemcpy(W, h.data(), sizeof(cplx<T>) * kLmax, cudaMemcpyHostToDevice));
}

template <class T>
const cplx<T>* Twiddles<T>::table_for(long long L) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = direct.find(L);
    if (it != direct.end()) return it->second;
    std::vector<cplx<T>> h(L);
    for (long long q = 0; q < L; ++q) {
        const long double a = -2.0L * 3.14159265358979323846264338327950288L * q / L;
        h[q].x = static_cast<T>(std::cos(a));
        h[q].y = static_cast<T>(std::sin(a));
    }
    cplx<T>* d = nullptr;
    FFCZ_CUDA_CHECK(cudaMalloc(&d, sizeof(cplx<T>) * L));
    FFCZ_CUDA_CHECK(cudaMemcpy(d, h.data(), sizeof(cplx<T>) * L, cudaMemcpyHostToDevice));
    direct[L] = d;
    return d;
}

template <class T>
Twiddles<T>::~Twiddles() {
    if (W) cudaFree(W);
    for (auto& kv : direct) cudaFree(kv.second);
}

template struct Twiddles<double>;
template struct Twiddles<float>;

template struct FftPlan<double>;
template void launch_col<double, HookNone>(long long, int, const double2*, double2*, long long,
                                           long long, long long, int, Twiddles<double>&,
                                           const int*, HookNone, cudaStream_t);
template void launch_col<double, HookFReduce>(long long, int, const double2*, double2*, long long,
                                              long long, long long, int, Twiddles<double>&,
                                              const int*, HookFReduce, cudaStream_t);
template void launch_col<double, HookFClip<double>>(long long, int, const double2*, double2*,
                                                    long long, long long, long long, int,
                                                    Twiddles<double>&, const int*,
                                                    HookFClip<double>, cudaStream_t);
template void launch_row_r2c<double>(long long, const double*, long long, double2*, long long,
                                     long long, Twiddles<double>&, const int*, cudaStream_t);
template void launch_row_c2r<double>(long long, const double2*, long long, double*, long long,
                                     long long, double, Twiddles<double>&, const int*,
                                     cudaStream_t);
template void launch_row_fused<double, HookSClip<double>>(long long, double2*, long long,
                                                          long long, long long, double,
                                                          Twiddles<double>&, const int*,
                                                          HookSClip<double>, cudaStream_t);

} // namespace ffcz_gpu
