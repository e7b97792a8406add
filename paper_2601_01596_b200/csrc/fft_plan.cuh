// Host-side pass planning and launch dispatch for the FFT engine.
#pragma once

#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "fft_engine.cuh"
#include "kernels.cuh"

namespace ffcz_gpu {

constexpr int kLmax = 8192;   // largest pow2 row length n2 / column length handled by the radix path

// Elements per thread E (= radix of the full Stockham stages) for an L-point line: the fewest
// stages (= fewest shared-memory exchanges) with at most 64 registers of line data
// (FP64: 8 or 16 complex, FP32: 16 or 32), the smaller E on a tie.
__host__ __device__ constexpr int nstages_c(int L, int E) {
    int s = 0;
    for (int ns = 1; ns < L; ns *= (L / ns >= E ? E : L / ns)) ++s;
    return s;
}
#ifndef FFCZ_E64_MAX
#define FFCZ_E64_MAX 16
#endif
template <class T>
__host__ __device__ constexpr int pick_E(int L) {
    constexpr int lo = sizeof(T) == 8 ? 8 : 16;
    constexpr int hi = sizeof(T) == 8 ? FFCZ_E64_MAX : 32;
    if (L <= lo) return L;
    return (hi > lo && nstages_c(L, hi) < nstages_c(L, lo)) ? hi : lo;
}

// Geometry of a field and its pitched half spectrum.
struct Geometry {
    int ndim = 0;
    long long d[3] = {1, 1, 1};  // dims padded to 3-D at the FRONT: (d0, d1, d2), d2 = last axis
    long long N = 0;             // samples
    long long rows = 0;          // d0 * d1
    long long n2 = 0;            // last axis
    int H = 0;                   // n2/2 + 1
    int P = 0;                   // pitch in complex elements
    long long half_elems() const { return rows * P; }
    long long Nc() const { return rows * H; }
    HalfGeom hg() const { return HalfGeom{rows, H, P, n2, 1.0 / H}; }
};

Geometry make_geometry(int ndim, const uint64_t* dims, int pitch_align);

// Twiddle tables, FP64-derived (long double on the host, rounded once).
template <class T>
struct Twiddles {
    std::map<std::pair<int, int>, cplx<T>*> stage;  // (L, E) -> Stockham stage table
    std::map<int, cplx<T>*> post;                   // M -> W_{2M}^k, k in [0, M]
    std::map<long long, cplx<T>*> direct;           // L -> W_L^q, q < L (direct passes)
    std::mutex mu;
    const cplx<T>* stage_table(int L, int E);
    const cplx<T>* post_table(int M);
    const cplx<T>* table_for(long long L);
    void init() {}
    ~Twiddles();
};

inline bool radix_col_ok(long long L) { return is_pow2(L) && L >= 16 && L <= 4096; }
inline bool radix_row_ok(long long n2) { return is_pow2(n2) && n2 >= 32 && n2 <= kLmax; }

// ---- launchers (fft_dispatch*.cu) -----------------------------------------------------------------
// Column pass along an axis of the half spectrum.  dir = -1 forward, +1 inverse.
template <class T, class Hook>
void launch_col(long long L, int dir, const cplx<T>* src, cplx<T>* dst, long long row_stride,
                long long plane_stride, long long nplanes, int ncols, Twiddles<T>& tw,
                const int* gate, Hook hook, cudaStream_t st);
// Round-trip column pass (k_col_tma1_rt: forward, hook.mid, inverse) into dst != src.
template <class T, class Hook>
void launch_col_rt(long long L, const cplx<T>* src, cplx<T>* dst, long long row_stride,
                   long long plane_stride, long long nplanes, int ncols, Twiddles<T>& tw,
                   const int* gate, Hook hook, cudaStream_t st);
// F = moved ? delta - FFT_axis(src) : 0 along one column axis (k_col_tma1_frebuild).
template <class T>
void launch_col_frebuild(long long L, const cplx<T>* src, const cplx<T>* delta, cplx<T>* F,
                         const unsigned char* moved, long long row_stride, long long plane_stride,
                         long long nplanes, int ncols, Twiddles<T>& tw, cudaStream_t st);
// Row R2C: real rows (stride in_stride) -> half rows (stride out_stride).
template <class T>
void launch_row_r2c(long long n2, const T* in, long long in_stride, cplx<T>* out,
                    long long out_stride, long long nrows, Twiddles<T>& tw, const int* gate,
                    cudaStream_t st);
// Row R2C with an output hook (tiled hooks skip the rows of converged frames).
template <class T, class Hook>
void launch_row_r2c_hook(long long n2, const T* in, long long in_stride, cplx<T>* out,
                         long long out_stride, long long nrows, Twiddles<T>& tw, const int* gate,
                         Hook hook, cudaStream_t st);
// First R2C of correct() with compute_error + preconditions fused in (FP64 output); with S,
// the R2C of eps0 + S instead (the gate's F rebuild), no checks.
template <class TI>
bool launch_row_r2c_eps0(long long n2, const TI* orig, const TI* dec, double2* out,
                         long long out_stride, long long nrows, Twiddles<double>& tw, SpatialB sb,
                         double fscale, double slack, Ctl* ctl, cudaStream_t st,
                         const double* S = nullptr);
// Row C2R: half rows -> real rows, scaled.
template <class T>
void launch_row_c2r(long long n2, const cplx<T>* in, long long in_stride, T* out,
                    long long out_stride, long long nrows, T scale, Twiddles<T>& tw,
                    const int* gate, cudaStream_t st);
// C2R with a real-output epilogue hook (radix path only).
template <class T, class Hook>
void launch_row_c2r_hook(long long n2, const cplx<T>* in, long long in_stride, T* out,
                         long long out_stride, long long nrows, T scale, Twiddles<T>& tw,
                         const int* gate, Hook hook, cudaStream_t st);
// Fused C2R -> hook(real) -> R2C, in place on the half rows or into `out` (radix path only).
template <class T, class Hook>
void launch_row_fused(long long n2, cplx<T>* data, long long stride, long long nrows,
                      long long real_stride, T scale, Twiddles<T>& tw, const int* gate, Hook hook,
                      cudaStream_t st,
                      cplx<T>* out = nullptr);

// Whole-field transforms built from the passes.
template <class T>
struct FftPlan {
    Geometry g;
    Twiddles<T>* tw;
    // x (N reals) -> half (pitched)
    void r2c(const T* x, cplx<T>* half, const int* gate, cudaStream_t st) const;
    // half (pitched, preserved if work != half) -> x (N reals) * scale; work is clobbered
    void c2r(const cplx<T>* half, cplx<T>* work, T* x, T scale, const int* gate,
             cudaStream_t st) const;
    // single column pass along field axis `axis` (< ndim-1 in the padded 3-D frame)
    template <class Hook>
    void col(int axis3, int dir, const cplx<T>* src, cplx<T>* dst, const int* gate, Hook hook,
             cudaStream_t st) const {
        const long long L = g.d[axis3];
        if (L == 1) {
            if (src != dst)
                FFCZ_CUDA_CHECK(cudaMemcpyAsync(dst, src, sizeof(cplx<T>) * g.half_elems(),
                                                cudaMemcpyDeviceToDevice, st));
            return;
        }
        long long row_stride, plane_stride, nplanes;
        if (axis3 == 1) {  // rows inside a d1 x P plane, planes = d0
            row_stride = g.P;
            plane_stride = g.d[1] * g.P;
            nplanes = g.d[0];
        } else {           // axis 0: rows stride d1*P, planes = d1
            row_stride = g.d[1] * g.P;
            plane_stride = g.P;
            nplanes = g.d[1];
        }
        launch_col<T, Hook>(L, dir, src, dst, row_stride, plane_stride, nplanes, g.H, *tw, gate,
                            hook, st);
    }
    // column axis `axis3` as one round trip (forward, hook.mid, inverse) from src into dst
    template <class Hook>
    void col_rt(int axis3, const cplx<T>* src, cplx<T>* dst, const int* gate, Hook hook,
                cudaStream_t st) const {
        long long row_stride, plane_stride, nplanes;
        axis_strides(axis3, row_stride, plane_stride, nplanes);
        launch_col_rt<T, Hook>(g.d[axis3], src, dst, row_stride, plane_stride, nplanes, g.H, *tw,
                               gate, hook, st);
    }
    void col_frebuild(int axis3, const cplx<T>* src, const cplx<T>* delta, cplx<T>* F,
                      const unsigned char* moved, cudaStream_t st) const {
        long long row_stride, plane_stride, nplanes;
        axis_strides(axis3, row_stride, plane_stride, nplanes);
        launch_col_frebuild<T>(g.d[axis3], src, delta, F, moved, row_stride, plane_stride, nplanes,
                               g.H, *tw, st);
    }
    bool rt_ok(int axis3) const {
        const long long L = g.d[axis3];
        return sizeof(T) == 8 && is_pow2(L) && L >= 16 && L <= 4096;
    }
    void axis_strides(int axis3, long long& row_stride, long long& plane_stride,
                      long long& nplanes) const {
        if (axis3 == 1) {
            row_stride = g.P;
            plane_stride = g.d[1] * g.P;
            nplanes = g.d[0];
        } else {
            row_stride = g.d[1] * g.P;
            plane_stride = g.P;
            nplanes = g.d[1];
        }
    }
    bool fused_ok() const;
};

} // namespace ffcz_gpu
