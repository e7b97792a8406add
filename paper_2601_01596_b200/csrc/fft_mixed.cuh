// Mixed-radix Stockham passes for extents that are not powers of two (SURVEY.md §8(f) item 3:
// S3D 500^3, EEG-length rows).  The reference transforms any extent through FFTW
// (proj/core/src/transform.cpp:20-50); here an extent L = 4^a 2^b 3^c 5^d 7^e p... is factored
// into radix stages run on a tile of lines staged in shared memory (ping-pong buffers, one
// __syncthreads per stage), radices 2/3/4/5/7 as register butterflies with exact constants and
// any other prime factor as an O(r) stage read straight from shared memory.  Every twiddle is an
// exact index into the per-L FP64-derived table W_L^q (Twiddles::table_for).  The inverse is
// conj(DFT(conj x)) (conjugation is exact), so only forward butterflies exist.
//
// Unlike the power-of-two passes these carry no fused hooks; the engine runs the clips as
// separate elementwise kernels for such shapes (engine.cu, fused_ok() == false).
#pragma once

#include "common.cuh"

namespace ffcz_gpu {

constexpr int kMixedMaxStages = 28;

struct MixedPlan {
    int L = 0;
    int nst = 0;
    int r[kMixedMaxStages] = {};
    // k = j mod ns at stage s without a division: floor(j / ns) = umulhi(j, mul[s]) with
    // mul = floor(2^32 / ns) + 1, exact while j * ns < 2^32 (L <= 65536); ns = 1 -> k = 0
    unsigned mul[kMixedMaxStages] = {};
};

// Factor L: radix 8 then 4 first (fewest stages), then 2, 3, 5, 7, then the remaining primes.
inline MixedPlan make_mixed_plan(long long L) {
    MixedPlan p;
    p.L = static_cast<int>(L);
    long long rem = L;
    auto take = [&](int r) {
        while (rem % r == 0 && p.nst < kMixedMaxStages) {
            p.r[p.nst++] = r;
            rem /= r;
        }
    };
    take(8);
    take(4);
    take(2);
    take(3);
    take(5);
    take(7);
    for (long long q = 11; q * q <= rem; q += 2) take(static_cast<int>(q));
    if (rem > 1 && p.nst < kMixedMaxStages) p.r[p.nst++] = static_cast<int>(rem);
    unsigned long long ns = 1;
    for (int s = 0; s < p.nst; ++s) {
        p.mul[s] = ns == 1 ? 0u : static_cast<unsigned>((1ull << 32) / ns + 1);
        ns *= static_cast<unsigned long long>(p.r[s]);
    }
    return p;
}

namespace mixed {

// Shared-memory position of line element i: one padding slot after every 8 elements.  The early
// Stockham stages store butterfly j's outputs R elements apart (R = 2, 4, 8), which put the
// lanes of a warp on the same banks (8-way conflicts: the passes were shared-memory bound at
// 84.5 % L1/TEX, profiles/r01_ncu_mixed_radix_500_v2.txt); with the pad, rows j*R land on
// alternating bank halves and every warp access is the minimum number of wavefronts.
__host__ __device__ __forceinline__ int sw(int i) { return i + (i >> 3); }
// padded line length (slots) of an L-element line
__host__ __device__ __forceinline__ int padded(int L) { return L + (L >> 3) + 1; }
// the column tiles use the padded positions; the row passes (one line per warp group, lanes on
// consecutive butterflies) measured slower with them (0.35 -> 0.31 of HBM at 500^3) and keep
// the dense layout
template <bool PAD> __device__ __forceinline__ int at(int i) { return PAD ? sw(i) : i; }

template <class C> __device__ __forceinline__ C conjc(C a) { a.y = -a.y; return a; }

// forward DFT of R points held in registers
template <class T, int R>
__device__ __forceinline__ void bfly(cplx<T>* a) {
    if constexpr (R == 2) {
        const cplx<T> s = cadd(a[0], a[1]), d = csub(a[0], a[1]);
        a[0] = s;
        a[1] = d;
    } else if constexpr (R == 8) {
        // two radix-4 DFTs of the even / odd samples, merged with W8^k = exp(-i pi k / 4)
        cplx<T> e[4] = {a[0], a[2], a[4], a[6]}, o[4] = {a[1], a[3], a[5], a[7]};
        bfly<T, 4>(e);
        bfly<T, 4>(o);
        const T c = T(0.70710678118654752440);
        cplx<T> w[4];
        w[0] = o[0];
        w[1] = mkc<T>(c * (o[1].x + o[1].y), c * (o[1].y - o[1].x));   // o (1 - i) / sqrt2
        w[2] = mkc<T>(o[2].y, -o[2].x);                                  // o (-i)
        w[3] = mkc<T>(c * (o[3].y - o[3].x), -c * (o[3].x + o[3].y));  // o (-1 - i) / sqrt2
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            a[k] = cadd(e[k], w[k]);
            a[k + 4] = csub(e[k], w[k]);
        }
    } else if constexpr (R == 4) {
        const cplx<T> s02 = cadd(a[0], a[2]), d02 = csub(a[0], a[2]);
        const cplx<T> s13 = cadd(a[1], a[3]), d13 = cmulmi(csub(a[1], a[3]));  // -i (a1 - a3)
        a[0] = cadd(s02, s13);
        a[2] = csub(s02, s13);
        a[1] = cadd(d02, d13);
        a[3] = csub(d02, d13);
    } else {
        // odd R: X_u = a0 + sum_{t=1}^{(R-1)/2} (a_t + a_{R-t}) cos(2 pi t u / R)
        //                                     - i (a_t - a_{R-t}) sin(2 pi t u / R)
        constexpr int H = (R - 1) / 2;
        double cs[R], sn[R];
        if constexpr (R == 3) {
            const double c[3] = {1.0, -0.5, -0.5};
            const double s[3] = {0.0, 0.86602540378443864676, -0.86602540378443864676};
#pragma unroll
            for (int k = 0; k < 3; ++k) cs[k] = c[k], sn[k] = s[k];
        } else if constexpr (R == 5) {
            const double c[5] = {1.0, 0.30901699437494742410, -0.80901699437494742410,
                                 -0.80901699437494742410, 0.30901699437494742410};
            const double s[5] = {0.0, 0.95105651629515357212, 0.58778525229247312917,
                                 -0.58778525229247312917, -0.95105651629515357212};
#pragma unroll
            for (int k = 0; k < 5; ++k) cs[k] = c[k], sn[k] = s[k];
        } else {
            static_assert(R == 7, "register butterflies exist for radix 2, 3, 4, 5, 7, 8");
            const double c[7] = {1.0,
                                 0.62348980185873353053,
                                 -0.22252093395631440429,
                                 -0.90096886790241912624,
                                 -0.90096886790241912624,
                                 -0.22252093395631440429,
                                 0.62348980185873353053};
            const double s[7] = {0.0,
                                 0.78183148246802980871,
                                 0.97492791218182360702,
                                 0.43388373911755812048,
                                 -0.43388373911755812048,
                                 -0.97492791218182360702,
                                 -0.78183148246802980871};
#pragma unroll
            for (int k = 0; k < 7; ++k) cs[k] = c[k], sn[k] = s[k];
        }
        cplx<T> sp[H + 1], sm[H + 1];
#pragma unroll
        for (int t = 1; t <= H; ++t) {
            sp[t] = cadd(a[t], a[R - t]);
            sm[t] = csub(a[t], a[R - t]);
        }
        cplx<T> X[R];
        X[0] = a[0];
#pragma unroll
        for (int t = 1; t <= H; ++t) X[0] = cadd(X[0], sp[t]);
#pragma unroll
        for (int u = 1; u <= H; ++u) {
            T re = a[0].x, im = a[0].y, pr = 0, pi = 0;
#pragma unroll
            for (int t = 1; t <= H; ++t) {
                const int k = (t * u) % R;
                re += sp[t].x * T(cs[k]);
                im += sp[t].y * T(cs[k]);
                // -i * sm * sin  ->  (sm.y sin, -sm.x sin)
                pr += sm[t].y * T(sn[k]);
                pi -= sm[t].x * T(sn[k]);
            }
            X[u] = mkc<T>(re + pr, im + pi);
            X[R - u] = mkc<T>(re - pr, im - pi);
        }
#pragma unroll
        for (int u = 0; u < R; ++u) a[u] = X[u];
    }
}

// This thread's place in a tile: line `line`, butterflies j = jt, jt + TL, ... (active only
// when line < nlines).  Element (i, line) of a buffer sits at i * si + line * sl.
struct TileLane {
    int line, jt, TL;
};

__device__ __forceinline__ int mod_ns(int j, int ns, unsigned mul) {
    return ns == 1 ? 0 : j - static_cast<int>(__umulhi(static_cast<unsigned>(j), mul)) * ns;
}

// One Stockham stage: butterfly j reads j + t m (t < R), twiddles by W_{ns R}^{k t}
// (k = j mod ns), writes (j - k) R + k + t ns.
template <class T, int R, bool PAD>
__device__ __forceinline__ void stage_reg(const cplx<T>* __restrict__ in, cplx<T>* __restrict__ out,
                                          int L, int ns, unsigned mul, int si, int sl,
                                          TileLane tl, const cplx<T>* __restrict__ wl, int wmul,
                                          bool cin) {
    const int m = L / R, wstep = L / (ns * R) * wmul;
    const int lo = tl.line * sl;
    for (int j = tl.jt; j < m; j += tl.TL) {
        const int k = mod_ns(j, ns, mul);
        cplx<T> a[R];
#pragma unroll
        for (int t = 0; t < R; ++t) {
            a[t] = in[at<PAD>(j + t * m) * si + lo];
            if (cin) a[t].y = -a[t].y;
            if (t > 0 && k > 0) a[t] = cmul(a[t], __ldg(&wl[k * t * wstep]));
        }
        bfly<T, R>(a);
        const int o = (j - k) * R + k;
#pragma unroll
        for (int t = 0; t < R; ++t) out[at<PAD>(o + t * ns) * si + lo] = a[t];
    }
}

// Generic prime radix: each output of a butterfly sums its R twiddled inputs from shared memory.
template <class T, bool PAD>
__device__ __forceinline__ void stage_gen(const cplx<T>* __restrict__ in, cplx<T>* __restrict__ out,
                                          int L, int R, int ns, unsigned mul, int si, int sl,
                                          TileLane tl, const cplx<T>* __restrict__ wl, int wmul,
                                          bool cin) {
    const int m = L / R, wstep = L / (ns * R);
    const int lo = tl.line * sl;
    for (int j = tl.jt; j < m; j += tl.TL) {
        const int k = mod_ns(j, ns, mul);
        for (int u = 0; u < R; ++u) {
            // X_u = sum_t a_t W_{ns R}^{k t} W_R^{t u} = sum_t a_t W_L^{t (k wstep + u m)}
            const int step = k * wstep + u * m;  // < 2L
            T ax = 0, ay = 0;
            int q = 0;
            for (int t = 0; t < R; ++t) {
                cplx<T> x = in[at<PAD>(j + t * m) * si + lo];
                if (cin) x.y = -x.y;
                const cplx<T> p = cmul(x, __ldg(&wl[q * wmul]));
                ax += p.x;
                ay += p.y;
                q += step;
                while (q >= L) q -= L;
            }
            out[at<PAD>((j - k) * R + k + u * ns) * si + lo] = mkc<T>(ax, ay);
        }
    }
}

// Runs every stage; returns the buffer holding the natural-order result.  wl[q * wmul] = W_L^q
// (wmul = 2 when the table is the 2L-point one of a packed real row).  Every thread of the CTA
// calls it (idle lanes included: the stage barriers are CTA-wide).
template <class T, bool PAD>
__device__ cplx<T>* run_stages(cplx<T>* A, cplx<T>* B, const MixedPlan& p, int si, int sl,
                               int nlines, TileLane tl, const cplx<T>* __restrict__ wl,
                               int wmul = 1, bool conj_in = false) {
    const bool on = tl.line < nlines;
    int ns = 1;
    for (int s = 0; s < p.nst; ++s) {
        const int r = p.r[s];
        const unsigned mul = p.mul[s];
        const bool cin = conj_in && s == 0;
        if (on) {
            switch (r) {
                case 2: stage_reg<T, 2, PAD>(A, B, p.L, ns, mul, si, sl, tl, wl, wmul, cin); break;
                case 3: stage_reg<T, 3, PAD>(A, B, p.L, ns, mul, si, sl, tl, wl, wmul, cin); break;
                case 4: stage_reg<T, 4, PAD>(A, B, p.L, ns, mul, si, sl, tl, wl, wmul, cin); break;
                case 8: stage_reg<T, 8, PAD>(A, B, p.L, ns, mul, si, sl, tl, wl, wmul, cin); break;
                case 5: stage_reg<T, 5, PAD>(A, B, p.L, ns, mul, si, sl, tl, wl, wmul, cin); break;
                case 7: stage_reg<T, 7, PAD>(A, B, p.L, ns, mul, si, sl, tl, wl, wmul, cin); break;
                default: stage_gen<T, PAD>(A, B, p.L, r, ns, mul, si, sl, tl, wl, wmul, cin); break;
            }
        }
        __syncthreads();
        cplx<T>* t = A;
        A = B;
        B = t;
        ns *= r;
    }
    return A;
}

} // namespace mixed

constexpr int kMixedU = 8;  // global loads in flight per thread while a tile is staged

// Column pass: a tile of B adjacent columns x L rows per CTA, ping-pong buffers of L*B.  Thread
// t works on column t mod B (consecutive threads: adjacent columns of one row, so loads and
// stores are B-element runs).
template <class T>
__global__ void __launch_bounds__(256) k_col_mixed(const cplx<T>* __restrict__ src,
                                                   cplx<T>* __restrict__ dst, MixedPlan p,
                                                   long long row_stride, long long plane_stride,
                                                   int ncols, int B, const cplx<T>* __restrict__ wl,
                                                   int dir, const int* gate) {
    if (gated(gate)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int L = p.L;
    cplx<T>* A = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* Bf = A + static_cast<size_t>(mixed::padded(L)) * B;
    const long long base = static_cast<long long>(blockIdx.y) * plane_stride +
                           static_cast<long long>(blockIdx.x) * B;
    const int nb = min(B, ncols - static_cast<int>(blockIdx.x) * B);
    const int TL = blockDim.x / B;
    mixed::TileLane tl{static_cast<int>(threadIdx.x) % B, static_cast<int>(threadIdx.x) / B, TL};
    if (tl.jt >= TL) tl.line = B;  // idle lane
    const int b = tl.line;
    if (b < B) {
        for (int i0 = tl.jt; i0 < L; i0 += kMixedU * TL) {
            cplx<T> v[kMixedU];
#pragma unroll
            for (int u = 0; u < kMixedU; ++u) {
                const int i = i0 + u * TL;
                v[u] = (i < L && b < nb) ? src[base + i * row_stride + b] : mkc<T>(T(0), T(0));
            }
#pragma unroll
            for (int u = 0; u < kMixedU; ++u) {
                const int i = i0 + u * TL;
                if (i < L) A[mixed::sw(i) * B + b] = dir < 0 ? v[u] : mixed::conjc(v[u]);
            }
        }
    }
    __syncthreads();
    const cplx<T>* R = mixed::run_stages<T, true>(A, Bf, p, B, 1, B, tl, wl);
    if (b < nb)
        for (int i = tl.jt; i < L; i += TL)
            dst[base + i * row_stride + b] =
                dir < 0 ? R[mixed::sw(i) * B + b] : mixed::conjc(R[mixed::sw(i) * B + b]);
}

__device__ __forceinline__ void cp_async_elem(void* dst, const void* src, int bytes, bool valid) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    const int n = valid ? bytes : 0;  // 0: zero-fill
    if (bytes == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n)
                     : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(n)
                     : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Persistent, pipelined column pass: three tile buffers rotate so that the cp.async copy of the
// CTA's next tile is in flight while the current tile runs its stages (ping-pong between the
// current and the spare buffer) and is stored.  Tiles: (plane, block of B columns).
template <class T>
__global__ void __launch_bounds__(256) k_col_mixed_pipe(const cplx<T>* __restrict__ src,
                                                        cplx<T>* __restrict__ dst, MixedPlan p,
                                                        long long row_stride,
                                                        long long plane_stride, int ncols, int B,
                                                        long long ntiles,
                                                        const cplx<T>* __restrict__ wl, int dir,
                                                        const int* gate) {
    if (gated(gate)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int L = p.L;
    const size_t tile_elems = static_cast<size_t>(mixed::padded(L)) * B;
    cplx<T>* buf0 = reinterpret_cast<cplx<T>*>(smem_raw);
    const int nblk = (ncols + B - 1) / B;
    const int TL = blockDim.x / B;
    mixed::TileLane tl{static_cast<int>(threadIdx.x) % B, static_cast<int>(threadIdx.x) / B, TL};
    if (tl.jt >= TL) tl.line = B;
    const int b = tl.line;
    auto tile_base = [&](long long tile, int& nb) {
        const long long plane = tile / nblk;
        const int cb = static_cast<int>(tile - plane * nblk);
        nb = min(B, ncols - cb * B);
        return plane * plane_stride + static_cast<long long>(cb) * B;
    };
    auto issue = [&](long long tile, cplx<T>* buf) {
        if (b < B) {
            int nb;
            const long long base = tile_base(tile, nb);
            const bool ok = b < nb;
            const cplx<T>* g = src + base + (ok ? b : 0);
            for (int i = tl.jt; i < L; i += TL)
                cp_async_elem(&buf[mixed::sw(i) * B + b], g + i * row_stride, sizeof(cplx<T>), ok);
        }
        cp_async_commit();
    };
    long long tile = blockIdx.x;
    if (tile >= ntiles) return;
    issue(tile, buf0);
    for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
        cplx<T>* cur = buf0 + tile_elems * (it % 3);
        cplx<T>* nxt = buf0 + tile_elems * ((it + 1) % 3);
        cplx<T>* spare = buf0 + tile_elems * ((it + 2) % 3);
        const long long next = tile + gridDim.x;
        if (next < ntiles) issue(next, nxt);
        else cp_async_commit();
        cp_async_wait1();
        __syncthreads();
        const cplx<T>* R = mixed::run_stages<T, true>(cur, spare, p, B, 1, B, tl, wl, 1, dir > 0);
        int nb;
        const long long base = tile_base(tile, nb);
        if (b < nb)
            for (int i = tl.jt; i < L; i += TL)
                dst[base + i * row_stride + b] =
                    dir < 0 ? R[mixed::sw(i) * B + b] : mixed::conjc(R[mixed::sw(i) * B + b]);
        __syncthreads();
    }
}

// Row tiles: thread t works on row t / TL of the tile, positions t mod TL + TL n.
__device__ __forceinline__ mixed::TileLane row_lane(int R) {
    const int TL = blockDim.x / R;
    return mixed::TileLane{static_cast<int>(threadIdx.x) / TL, static_cast<int>(threadIdx.x) % TL,
                           TL};
}

// Row R2C, R rows per CTA.  Even n2 = 2M: the row is packed as z[n] = x[2n] + i x[2n+1], one
// M-point transform Z, then X[k] = E[k] + W_n2^k O[k] with E[k] = (Z[k] + conj Z[M-k]) / 2 and
// O[k] = (Z[k] - conj Z[M-k]) / 2i (p = plan of M, wl = the n2-point table, stride 2 for the
// stages).  Odd n2: a full n2-point complex transform of (x, 0) (p = plan of n2).  Buffers hold
// R lines of stride sl = p.L + 1.
template <class T>
__global__ void __launch_bounds__(256) k_row_r2c_mixed(const T* __restrict__ in,
                                                       long long in_stride,
                                                       cplx<T>* __restrict__ out,
                                                       long long out_stride, long long nrows,
                                                       int n2, int R, MixedPlan p,
                                                       const cplx<T>* __restrict__ wl,
                                                       const int* gate) {
    if (gated(gate)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const bool packed = (n2 & 1) == 0;
    const int L = p.L, sl = L + 1, h = n2 / 2 + 1;
    cplx<T>* A = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* Bf = A + static_cast<size_t>(sl) * R;
    const long long row0 = static_cast<long long>(blockIdx.x) * R;
    const int nr = static_cast<int>(nrows - row0 < R ? nrows - row0 : R);
    const mixed::TileLane tl = row_lane(R);
    const int r = tl.line;
    if (r < R) {
        const T* row = in + (row0 + r) * in_stride;
        for (int i0 = tl.jt; i0 < L; i0 += kMixedU * tl.TL) {
            T v0[kMixedU], v1[kMixedU];
#pragma unroll
            for (int u = 0; u < kMixedU; ++u) {
                const int i = i0 + u * tl.TL;
                const bool ok = i < L && r < nr;
                v0[u] = ok ? row[packed ? 2 * i : i] : T(0);
                v1[u] = (ok && packed) ? row[2 * i + 1] : T(0);
            }
#pragma unroll
            for (int u = 0; u < kMixedU; ++u) {
                const int i = i0 + u * tl.TL;
                if (i < L) A[r * sl + (i)] = mkc<T>(v0[u], v1[u]);
            }
        }
    }
    __syncthreads();
    const cplx<T>* Z = mixed::run_stages<T, false>(A, Bf, p, 1, sl, R, tl, wl, packed ? 2 : 1);
    if (r < nr) {
        for (int k = tl.jt; k < h; k += tl.TL) {
            cplx<T> X;
            if (packed) {
                const cplx<T> zk = Z[r * sl + (k == L ? 0 : k)], zn = Z[r * sl + (k == 0 ? 0 : L - k)];
                const T hf = T(0.5);
                const cplx<T> ze = mkc<T>((zk.x + zn.x) * hf, (zk.y - zn.y) * hf);
                const cplx<T> zo = mkc<T>((zk.y + zn.y) * hf, (zn.x - zk.x) * hf);
                X = cadd(ze, cmul(zo, __ldg(&wl[k])));
            } else {
                X = Z[r * sl + (k)];
            }
            out[(row0 + r) * out_stride + k] = X;
        }
    }
}

// Row C2R (imaginary parts of bin 0 and, for even n2, bin n2/2 ignored, as every C2R).  Even
// n2 = 2M: Z[k] = (X[k] + conj X[M-k]) + i (X[k] - conj X[M-k]) conj(W_n2^k), z = M-point
// inverse of Z, x[2n] = Re z[n], x[2n+1] = Im z[n].  Odd n2: the half row is mirrored to the full
// Hermitian row and transformed with n2 points.  The inverse is conj(DFT(conj .)).
template <class T>
__global__ void __launch_bounds__(256) k_row_c2r_mixed(const cplx<T>* __restrict__ in,
                                                       long long in_stride, T* __restrict__ out,
                                                       long long out_stride, long long nrows,
                                                       int n2, int R, MixedPlan p,
                                                       const cplx<T>* __restrict__ wl, T scale,
                                                       const int* gate) {
    if (gated(gate)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const bool packed = (n2 & 1) == 0;
    const int L = p.L, sl = L + 1, h = n2 / 2 + 1;
    cplx<T>* A = reinterpret_cast<cplx<T>*>(smem_raw);
    cplx<T>* Bf = A + static_cast<size_t>(sl) * R;
    const long long row0 = static_cast<long long>(blockIdx.x) * R;
    const int nr = static_cast<int>(nrows - row0 < R ? nrows - row0 : R);
    const mixed::TileLane tl = row_lane(R);
    const int r = tl.line;
    // stage the half rows (packed: into Bf; odd: conj X[k] into A and X[k] at the mirror)
    if (r < R) {
        const cplx<T>* row = in + (row0 + r) * in_stride;
        for (int k0 = tl.jt; k0 < h; k0 += kMixedU * tl.TL) {
            cplx<T> v[kMixedU];
#pragma unroll
            for (int u = 0; u < kMixedU; ++u) {
                const int k = k0 + u * tl.TL;
                v[u] = (k < h && r < nr) ? row[k] : mkc<T>(T(0), T(0));
                if (k == 0 || (packed && k == h - 1)) v[u].y = T(0);
            }
#pragma unroll
            for (int u = 0; u < kMixedU; ++u) {
                const int k = k0 + u * tl.TL;
                if (k >= h) continue;
                if (packed) {
                    Bf[r * sl + (k)] = v[u];
                } else {
                    A[r * sl + (k)] = mixed::conjc(v[u]);
                    if (k > 0 && n2 - k >= h) A[r * sl + (n2 - k)] = v[u];
                }
            }
        }
    }
    __syncthreads();
    if (packed) {
        if (r < R) {
            for (int k = tl.jt; k < L; k += tl.TL) {
                const cplx<T> xk = Bf[r * sl + (k)], xn = Bf[r * sl + (L - k)];
                const cplx<T> s = mkc<T>(xk.x + xn.x, xk.y - xn.y);   // X[k] + conj X[M-k]
                const cplx<T> d = mkc<T>(xk.x - xn.x, xk.y + xn.y);   // X[k] - conj X[M-k]
                const cplx<T> o = cmulc(d, __ldg(&wl[k]));           // d * conj W^k
                A[r * sl + (k)] = mixed::conjc(mkc<T>(s.x - o.y, s.y + o.x));  // conj(s + i o)
            }
        }
        __syncthreads();
    }
    const cplx<T>* z = mixed::run_stages<T, false>(A, Bf, p, 1, sl, R, tl, wl, packed ? 2 : 1);
    if (r < nr) {
        T* orow = out + (row0 + r) * out_stride;
        if (packed) {
            for (int i = tl.jt; i < L; i += tl.TL) {
                const cplx<T> v = z[r * sl + (i)];  // conj z: (x[2i], -x[2i+1])
                orow[2 * i] = v.x * scale;
                orow[2 * i + 1] = -v.y * scale;
            }
        } else {
            for (int i = tl.jt; i < n2; i += tl.TL) orow[i] = z[r * sl + (i)].x * scale;
        }
    }
}

} // namespace ffcz_gpu
