// FP64 instantiations of the FFT engine + shared host helpers (geometry, twiddle tables).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "fft_dispatch.cuh"

namespace ffcz_gpu {

// L2 sector promotion of the column-pass boxes (FFCZ_TMA_PROMO=none|64|128|256, A/B): 128 B
// measured 1.7 % faster than 256 B on the 1024^3 outer axis (profiles/r02_passbench_promo.jsonl)
static CUtensorMapL2promotion l2_promotion() {
    static const CUtensorMapL2promotion p = [] {
        const char* e = std::getenv("FFCZ_TMA_PROMO");
        const std::string v = e ? e : "128";
        if (v == "none") return CU_TENSOR_MAP_L2_PROMOTION_NONE;
        if (v == "64") return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
        if (v == "128") return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
        return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }();
    return p;
}

bool encode_col_map(CUtensorMap* map, const void* base, int scalar_bytes, long long ncols,
                    long long L, long long row_stride, long long nplanes, long long plane_stride,
                    int B, int LB, bool complex) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) return false;
    const int per = complex ? 2 : 1;                     // scalars per element
    const long long eb = static_cast<long long>(per) * scalar_bytes;  // bytes per element
    if ((reinterpret_cast<uintptr_t>(base) & 15) || (row_stride * eb) % 16 ||
        (plane_stride * eb) % 16 || (B * eb) % 16)
        return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(per * ncols), static_cast<cuuint64_t>(L),
                                static_cast<cuuint64_t>(nplanes)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(row_stride * eb),
                                   static_cast<cuuint64_t>(plane_stride * eb)};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(per * B), static_cast<cuuint32_t>(LB), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode(map, scalar_bytes == 8   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                   : scalar_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                       : CU_TENSOR_MAP_DATA_TYPE_UINT8,
                              3, const_cast<void*>(base), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

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

namespace {

constexpr long double kTwoPi = 6.283185307179586476925286766559005768L;

template <class T>
cplx<T>* upload(const std::vector<cplx<T>>& h) {
    cplx<T>* d = nullptr;
    FFCZ_CUDA_CHECK(cudaMalloc(&d, sizeof(cplx<T>) * std::max<size_t>(1, h.size())));
    FFCZ_CUDA_CHECK(cudaMemcpy(d, h.data(), sizeof(cplx<T>) * h.size(), cudaMemcpyHostToDevice));
    return d;
}

// exp(-2 pi i num / den), evaluated in long double and rounded once
template <class T>
cplx<T> wexp(long long num, long long den) {
    const long double a = -kTwoPi * static_cast<long double>(num % den) / static_cast<long double>(den);
    cplx<T> w;
    w.x = static_cast<T>(std::cos(a));
    w.y = static_cast<T>(std::sin(a));
    return w;
}

} // namespace

template <class T>
const cplx<T>* Twiddles<T>::stage_table(int L, int E) {
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(L, E);
    auto it = stage.find(key);
    if (it != stage.end()) return it->second;
    std::vector<cplx<T>> h;
    for (int ns = 1; ns < L;) {
        const int R = (L / ns >= E) ? E : L / ns;
        if (ns > 1)
            for (int k = 0; k < ns; ++k) h.push_back(wexp<T>(k, static_cast<long long>(ns) * R));
        ns *= R;
    }
    if (h.empty()) h.push_back(wexp<T>(0, 1));
    return stage[key] = upload<T>(h);
}

template <class T>
const cplx<T>* Twiddles<T>::post_table(int M) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = post.find(M);
    if (it != post.end()) return it->second;
    std::vector<cplx<T>> h(M + 1);
    for (int k = 0; k <= M; ++k) h[k] = wexp<T>(k, 2LL * M);
    return post[M] = upload<T>(h);
}

template <class T>
const cplx<T>* Twiddles<T>::table_for(long long L) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = direct.find(L);
    if (it != direct.end()) return it->second;
    std::vector<cplx<T>> h(L);
    for (long long q = 0; q < L; ++q) h[q] = wexp<T>(q, L);
    return direct[L] = upload<T>(h);
}

template <class T>
Twiddles<T>::~Twiddles() {
    for (auto& kv : stage) cudaFree(kv.second);
    for (auto& kv : post) cudaFree(kv.second);
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
template bool launch_row_r2c_eps0<float>(long long, const float*, const float*, double2*,
                                         long long, long long, Twiddles<double>&, SpatialB, double,
                                         double, Ctl*, cudaStream_t, const double*);
template bool launch_row_r2c_eps0<double>(long long, const double*, const double*, double2*,
                                          long long, long long, Twiddles<double>&, SpatialB,
                                          double, double, Ctl*, cudaStream_t, const double*);
template void launch_row_r2c<double>(long long, const double*, long long, double2*, long long,
                                     long long, Twiddles<double>&, const int*, cudaStream_t);
template void launch_row_c2r<double>(long long, const double2*, long long, double*, long long,
                                     long long, double, Twiddles<double>&, const int*,
                                     cudaStream_t);
template void launch_row_fused<double, HookSClip<double>>(long long, double2*, long long,
                                                          long long, long long, double,
                                                          Twiddles<double>&, const int*,
                                                          HookSClip<double>, cudaStream_t, double2*);
} // namespace ffcz_gpu
