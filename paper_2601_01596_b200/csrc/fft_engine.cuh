// Hand-written FFT engine for sm_100a: batched 1-D passes of a separable R2C/C2R transform.
//
// Replaces the reference's FFTW c2c call (`run_c2c`, /root/reference/proj/core/src/transform.cpp:20-50)
// with a half-spectrum (R2C/C2R) decomposition; SURVEY.md §0.5 / App. B establish that an FP64
// half-spectrum loop is observationally identical to the reference's full c2c loop.
//
// Layout in HBM: a real field is row-major n0 x n1 x n2 (last axis fastest);
// its half spectrum is row-major n0 x n1 x P complex with P = round_up(n2/2+1, 128 B/elem) so every
// row starts 128-byte aligned (the Nyquist column k2 = n2/2 is a ragged last tile).
//
// Every pass is one kernel that reads each element once and writes it once (16 B/complex FP32,
// 32 B FP64 — the per-pass algorithmic traffic of SURVEY.md §8d).  Inside a pass:
//  * each thread owns E elements of one line in registers, strided by T = L/E
//    (v[m] = x[t + T*m]); global loads/stores of that set are coalesced because consecutive
//    lanes own consecutive columns (column passes) or consecutive elements (row passes);
//  * the line is transformed by Stockham radix-E stages (radix <= 32 butterflies fully in
//    registers with compile-time twiddles), exchanging through padded shared memory between
//    stages (row i lives at i + i/E: the stride-E writes of stage 1 hit distinct banks);
//  * inter-stage twiddles come from one FP64-derived table W[q] = exp(-2*pi*i*q/LMAX).
// Fusion hooks (pre/post functors) let the projection loop put its clip / reduction into the
// pass that produces or consumes the data.
#pragma once

#include <cooperative_groups.h>

#include <utility>

#include "common.cuh"
#include "tma.cuh"

namespace ffcz_gpu {

// cos(2*pi*q/32), q in [0, 16)
__host__ __device__ constexpr double cos32(int q) {
    return q == 0   ? 1.0
           : q == 1 ? 0.98078528040323044912618223613424
           : q == 2 ? 0.92387953251128675612818318939679
           : q == 3 ? 0.83146961230254523707878837761791
           : q == 4 ? 0.70710678118654752440084436210485
           : q == 5 ? 0.55557023301960222474283081394853
           : q == 6 ? 0.38268343236508977172845998403040
           : q == 7 ? 0.19509032201612826784828486847702
           : q == 8 ? 0.0
                    : -cos32(16 - q);
}
// sin(2*pi*q/32), q in [0, 16)
__host__ __device__ constexpr double sin32(int q) { return q <= 8 ? cos32(8 - q) : cos32(q - 8); }

// a * exp(DIR * 2*pi*i * Q/32)
template <int DIR, int Q, class C>
__device__ __forceinline__ C twq(C a) {
    using T = decltype(a.x);
    if constexpr (Q == 0) {
        return a;
    } else if constexpr (Q == 8) {
        return DIR < 0 ? cmulmi(a) : cmuli(a);
    } else {
        constexpr T c = static_cast<T>(cos32(Q));
        constexpr T s = static_cast<T>(DIR * sin32(Q));
        C r;
        r.x = a.x * c - a.y * s;
        r.y = a.x * s + a.y * c;
        return r;
    }
}

__host__ __device__ constexpr int brev_c(int i, int bits) {
    int r = 0;
    for (int b = 0; b < bits; ++b)
        if (i & (1 << b)) r |= 1 << (bits - 1 - b);
    return r;
}

template <int DIR, int R, int LEN, class C>
__device__ __forceinline__ void dit_stages(C* a) {
    if constexpr (LEN <= R) {
        [&]<int... S>(std::integer_sequence<int, S...>) {
            (
                [&] {
                    constexpr int s0 = S * LEN;
                    [&]<int... J>(std::integer_sequence<int, J...>) {
                        (
                            [&] {
                                C u = a[s0 + J];
                                C v = twq<DIR, J*(32 / LEN)>(a[s0 + J + LEN / 2]);
                                a[s0 + J] = cadd(u, v);
                                a[s0 + J + LEN / 2] = csub(u, v);
                            }(),
                            ...);
                    }(std::make_integer_sequence<int, LEN / 2>{});
                }(),
                ...);
        }(std::make_integer_sequence<int, R / LEN>{});
        dit_stages<DIR, R, LEN * 2>(a);
    }
}

// In-register DFT of R (power of two, <= 32) points, natural order in and out.
// DIR = -1: forward exp(-2 pi i nk/R); DIR = +1: unnormalised inverse.
template <int DIR, int R, class C>
__device__ __forceinline__ void dft_reg(C* a) {
    static_assert(R >= 1 && R <= 32 && is_pow2_c(R), "radix");
    if constexpr (R > 1) {
        constexpr int bits = ilog2_c(R);
        [&]<int... I>(std::integer_sequence<int, I...>) {
            (
                [&] {
                    constexpr int j = brev_c(I, bits);
                    if constexpr (j > I) {
                        C tmp = a[I];
                        a[I] = a[j];
                        a[j] = tmp;
                    }
                }(),
                ...);
        }(std::make_integer_sequence<int, R>{});
        dit_stages<DIR, R, 2>(a);
    }
}

// ---- shared-memory exchangers ---------------------------------------------------------------

// Column passes: smem tile [row i][column b], one padding row every E rows.
template <class T, int E>
struct XchCol {
    cplx<T>* s;   // already offset by the thread's column b
    int B;
    __device__ __forceinline__ static int row(int i) { return i + i / E; }
    __device__ __forceinline__ void sync() const { __syncthreads(); }
    __device__ __forceinline__ void st(int i, cplx<T> v) const { s[row(i) * B] = v; }
    __device__ __forceinline__ cplx<T> ld(int i) const { return s[row(i) * B]; }
};

// Column passes with a scalar exchange buffer: real and imaginary parts are exchanged in two
// rounds through (L + L/E) x B scalars, half the shared memory of XchCol (k_col_tma1).
template <class T, int E>
struct XchColS {
    static constexpr bool kSplit = true;
    T* s;   // already offset by the thread's column b
    int B;
    __device__ __forceinline__ static int row(int i) { return i + i / E; }
    __device__ __forceinline__ void sync() const { __syncthreads(); }
    __device__ __forceinline__ void st(int i, T v) const { s[row(i) * B] = v; }
    __device__ __forceinline__ T ld(int i) const { return s[row(i) * B]; }
};

template <class X>
constexpr bool xch_split() {
    if constexpr (requires { X::kSplit; })
        return X::kSplit;
    else
        return false;
}

// Row passes: one padded line per row; element i lives at i + i/E.
template <class T, int E>
struct XchRow {
    cplx<T>* s;
    __device__ __forceinline__ static int pos(int i) { return i + i / E; }
    __device__ __forceinline__ void sync() const { __syncthreads(); }
    __device__ __forceinline__ void st(int i, cplx<T> v) const { s[pos(i)] = v; }
    __device__ __forceinline__ cplx<T> ld(int i) const { return s[pos(i)]; }
};

// Row passes whose line fits one warp (the warp-shuffle kernels, L/E <= 32 threads per row): the
// row's padded buffer is private to its warp, so its exchanges need only a warp barrier — the
// rows of a CTA no longer wait for each other at every Stockham stage.
template <class T, int E>
struct XchRowW {
    static constexpr bool kTwTree = true;  // twiddle powers by squaring (see stockham)
    cplx<T>* s;
    __device__ __forceinline__ static int pos(int i) { return i + i / E; }
    __device__ __forceinline__ void sync() const { __syncwarp(); }
    __device__ __forceinline__ void st(int i, cplx<T> v) const { s[pos(i)] = v; }
    __device__ __forceinline__ cplx<T> ld(int i) const { return s[pos(i)]; }
};

// ---- Stockham radix-E passes over a line of L points held as v[m] = x[t + T*m] ---------------
// Stage radices are E, E, ..., E, L/E^k (remainder last so stage 1 writes have stride E, the
// pattern the padding is built for).  Inter-stage twiddles: one load of w = exp(-2 pi i k/(NS R))
// per butterfly from a per-(L, E) table laid out stage by stage ([k], so consecutive lanes read
// consecutive entries: one coalesced, L1-resident request per warp), then w^r by successive
// products in registers (<= 15 products, a few ulp) — shared-memory/L1 bandwidth, not FLOPs,
// bounds these passes.
template <int L, int E>
__host__ __device__ constexpr int stage_tw_offset(int NS) {
    int off = 0;
    for (int ns = 1; ns < NS;) {
        const int R = (L / ns >= E) ? E : L / ns;
        if (ns > 1) off += ns;
        ns *= R;
    }
    return off;
}

template <class X>
constexpr bool tw_tree() {
#ifdef FFCZ_TW_TREE
    return true;
#else
    if constexpr (requires { X::kTwTree; })
        return X::kTwTree;
    else
        return false;
#endif
}

template <class T, int L, int E, int NS, int DIR, class X>
__device__ __forceinline__ void stockham(cplx<T> (&v)[E], int t, const cplx<T>* __restrict__ tw,
                                         const X& xch) {
    constexpr int R = (L / NS >= E) ? E : (L / NS);
    constexpr int NB = E / R;
    constexpr int TT = L / E;
    static_assert(R >= 2 && L % (NS * R) == 0, "stage");
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        cplx<T> a[R];
#pragma unroll
        for (int r = 0; r < R; ++r) a[r] = v[i + r * NB];
        if constexpr (NS > 1) {
            const int j = t + TT * i;
            const int k = j & (NS - 1);
            constexpr int OFF = stage_tw_offset<L, E>(NS);
            const cplx<T> w1 = tw[OFF + k];
            if constexpr (!tw_tree<X>()) {
                cplx<T> w = w1;
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    a[r] = DIR < 0 ? cmul(a[r], w) : cmulc(a[r], w);
                    if (r + 1 < R) w = cmul(w, w1);
                }
            } else {
                // powers by squaring where r is even (w^r = (w^(r/2))^2): dependency depth 6
                // for R = 16 instead of the 14 of successive products (the warp-per-row passes:
                // fused row pass -3 %; the column passes measured +2-3 % and keep the chain,
                // profiles/r02_ab_twiddle_tree.txt)
                cplx<T> w[R];
                w[1] = w1;
#pragma unroll
                for (int r = 2; r < R; ++r)
                    w[r] = (r & 1) ? cmul(w[r - 1], w1) : cmul(w[r / 2], w[r / 2]);
#pragma unroll
                for (int r = 1; r < R; ++r) a[r] = DIR < 0 ? cmul(a[r], w[r]) : cmulc(a[r], w[r]);
            }
        }
        dft_reg<DIR, R>(a);
#pragma unroll
        for (int r = 0; r < R; ++r) v[i + r * NB] = a[r];
    }
    if constexpr (NS * R < L) {
        if constexpr (xch_split<X>()) {
            // two scalar rounds (Re, then Im); v keeps the pre-exchange slot order for the Im
            // round because only the .x halves have been replaced
#pragma unroll
            for (int part = 0; part < 2; ++part) {
                xch.sync();
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    const int j = t + TT * i;
                    const int base = (j / NS) * NS * R + (j & (NS - 1));
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        xch.st(base + r * NS, part == 0 ? v[i + r * NB].x : v[i + r * NB].y);
                }
                xch.sync();
#pragma unroll
                for (int m = 0; m < E; ++m) {
                    if (part == 0) v[m].x = xch.ld(t + TT * m);
                    else v[m].y = xch.ld(t + TT * m);
                }
            }
        } else {
            xch.sync();
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const int j = t + TT * i;
                const int base = (j / NS) * NS * R + (j & (NS - 1));
#pragma unroll
                for (int r = 0; r < R; ++r) xch.st(base + r * NS, v[i + r * NB]);
            }
            xch.sync();
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = xch.ld(t + TT * m);
        }
        stockham<T, L, E, NS * R, DIR>(v, t, tw, xch);
    }
}

// ---- hooks ------------------------------------------------------------------------------------
// pre(v, off, c): on a loaded element before the transform; post(v, off, c): on a transformed
// element before the store (off = element offset in the half-spectrum layout, c = k2 column).
// finish(): once per CTA after all stores (block-level reductions); must be CTA-uniform.
struct HookNone {
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    template <class C> __device__ __forceinline__ void post(C&, long long, int) {}
    __device__ __forceinline__ void finish() {}
};

// Optional per-CTA setup (e.g. reading loop state once): hook.begin() when the hook has one.
template <class H>
__device__ __forceinline__ void hook_begin(H& h) {
    if constexpr (requires { h.begin(); }) h.begin();
}

// A tiled hook (kTiled, batched frames) is asked per tile whether to skip it (its frame has
// converged) and brackets every processed tile with tile_begin(unit) / tile_end() (CTA-uniform;
// unit = plane for column passes, first row for row passes).
template <class H>
constexpr bool hook_tiled() {
    if constexpr (requires { H::kTiled; })
        return H::kTiled;
    else
        return false;
}

// A hook may declare `static constexpr bool kNoStore = true` when the pass output is consumed
// by the hook alone (e.g. the verify reduction): the store is skipped (half a pass of traffic).
template <class H>
constexpr bool hook_stores() {
    if constexpr (requires { H::kNoStore; })
        return !H::kNoStore;
    else
        return true;
}

// ---- column pass: L-point c2c along a strided axis of the half spectrum -------------------------
// Tile = L rows x B consecutive columns (columns = k2 < ncols inside one plane).
// Threads holding 32 registers of line data run 512 per CTA, 64 registers 256.
template <class T, int E>
constexpr int max_threads() { return E * sizeof(cplx<T>) <= 128 ? 512 : 256; }

// Launched with blockDim.x = (L/E) * B threads and (L + L/E) * B elements of dynamic smem.
// Persistent: a grid sized to the resident-CTA capacity walks the tiles (tile = B consecutive
// columns of one plane), so a pass launched after convergence retires in microseconds and
// block reductions fold many tiles before their single atomic.
template <class T, int L, int E, int DIR, class Hook>
__global__ void __launch_bounds__(max_threads<T, E>(), 512 / max_threads<T, E>())
    k_col(const cplx<T>* __restrict__ src, cplx<T>* __restrict__ dst, long long row_stride,
          long long plane_stride, int ncols, int B, long long ntiles,
          const cplx<T>* __restrict__ tw, const int* gate, Hook hook) {
    if (gated(gate)) return;
    hook_begin(hook);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* s = reinterpret_cast<cplx<T>*>(smem_raw);
    constexpr int TT = L / E;
    const int b = threadIdx.x % B;
    const int t = threadIdx.x / B;
    const int tiles_c = (ncols + B - 1) / B;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long plane = tile / tiles_c;
        if constexpr (hook_tiled<Hook>()) {
            if (hook.tile_skip(plane)) continue;
            hook.tile_begin(plane);
        }
        const int c = static_cast<int>(tile - plane * tiles_c) * B + b;
        const bool valid = c < ncols;
        const long long base = plane * plane_stride + c;
        cplx<T> v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const long long off = base + static_cast<long long>(t + TT * m) * row_stride;
            if (valid) {
                v[m] = src[off];
                hook.pre(v[m], off, c);
            } else {
                v[m] = mkc<T>(T(0), T(0));
            }
        }
        stockham<T, L, E, 1, DIR>(v, t, tw, XchCol<T, E>{s + b, B});
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const long long off = base + static_cast<long long>(t + TT * m) * row_stride;
            if (valid) {
                hook.post(v[m], off, c);
                if constexpr (hook_stores<Hook>()) dst[off] = v[m];
            }
        }
        if constexpr (hook_tiled<Hook>()) {
            hook.tile_end();
            __syncthreads();  // the next tile's exchange reuses the shared tile
        }
    }
    hook.finish();
}

// Hooks that compare against the frequency bound declare kDelta and take Delta(off) as an
// argument (pre_d / post_d), so the staged pass can hand them the value from its TMA side tile.
template <class H>
constexpr bool hook_delta() {
    if constexpr (requires { H::kDelta; })
        return H::kDelta;
    else
        return false;
}

// TMA-staged column pass.  Same tile and register layout as k_col, but the tile is brought into
// shared memory by 3-D TMA boxes (cp.async.bulk.tensor, mbarrier completion, <= 256 rows per
// box), double-buffered: while tile k is transformed out of buffer k%2 (which then serves as its
// exchange buffer), tile k+1 is already landing in the other buffer, and tile k+2 is issued the
// moment buffer k%2 is free — so HBM always has a tile in flight per SM (the load/compute/store
// serialisation measured in profiles/r01_summary.md).  Out-of-range columns of the ragged last
// tile arrive zero-filled.  With `has_side`, the per-component bound Delta (one FP64 lane in the
// same pitched layout) rides along as a side tile on the same mbarrier, so the check / clip hooks
// never wait on a dependent global load.
// smem: 2 x (L + L/E) x B complex [+ 2 x L x B doubles side] + 2 mbarriers.
template <class T, int L, int E, int DIR, class Hook>
__global__ void __launch_bounds__(max_threads<T, E>(), 1)
    k_col_tma(const __grid_constant__ CUtensorMap map, const __grid_constant__ CUtensorMap side_map,
              int has_side, cplx<T>* __restrict__ dst, long long row_stride, long long plane_stride,
              int ncols, int B, long long ntiles, const cplx<T>* __restrict__ tw, const int* gate,
              Hook hook) {
    if (gated(gate)) return;
    hook_begin(hook);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int TT = L / E;
    constexpr int LB = L < 256 ? L : 256;
    constexpr bool kDelta = hook_delta<Hook>();
    const int b = threadIdx.x % B;
    const int t = threadIdx.x / B;
    const int tiles_c = (ncols + B - 1) / B;
    const int buf_elems = (L + L / E) * B;
    cplx<T>* bufs = reinterpret_cast<cplx<T>*>(smem_raw);
    double* sides = reinterpret_cast<double*>(bufs + 2 * buf_elems);
    const int side_elems = has_side ? L * B : 0;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sides + 2 * side_elems);
    const unsigned tile_bytes = static_cast<unsigned>(L) * B * sizeof(cplx<T>) +
                                static_cast<unsigned>(side_elems) * sizeof(double);
    auto issue = [&](long long tile, int slot) {
        const long long plane = tile / tiles_c;
        const int c0 = static_cast<int>(tile - plane * tiles_c) * B;
        mbar_arrive_expect_tx(&bars[slot], tile_bytes);
#pragma unroll
        for (int j = 0; j < L / LB; ++j) {
            tma_load_3d(bufs + slot * buf_elems + j * LB * B, &map, &bars[slot], 2 * c0, j * LB,
                        static_cast<int>(plane));
            if (has_side)
                tma_load_3d(sides + slot * side_elems + j * LB * B, &side_map, &bars[slot], c0,
                            j * LB, static_cast<int>(plane));
        }
    };
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&map);
        if (has_side) tma_prefetch_desc(&side_map);
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (blockIdx.x < ntiles) issue(blockIdx.x, 0);
        if (blockIdx.x + gridDim.x < ntiles) issue(blockIdx.x + gridDim.x, 1);
    }
    unsigned phase = 0;  // bit s = parity of the next completion of buffer s
    int slot = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, slot ^= 1) {
        cplx<T>* s = bufs + slot * buf_elems;
        const double* sd = sides + slot * side_elems;
        mbar_wait(&bars[slot], (phase >> slot) & 1u);
        phase ^= 1u << slot;
        const long long plane = tile / tiles_c;
        if constexpr (hook_tiled<Hook>()) {
            if (hook.tile_skip(plane)) {  // frame done: drop the tile, keep the pipeline going
                fence_proxy_async_smem();
                __syncthreads();
                if (threadIdx.x == 0 && tile + 2 * gridDim.x < ntiles) issue(tile + 2 * gridDim.x, slot);
                continue;
            }
            hook.tile_begin(plane);
        }
        const int c = static_cast<int>(tile - plane * tiles_c) * B + b;
        const bool valid = c < ncols;
        const long long base = plane * plane_stride + c;
        auto delta = [&](int m, long long off) {
            if constexpr (kDelta) {
                if (has_side) {
                    const double x = sd[(t + TT * m) * B + b];
                    return make_double2(x, x);
                }
                return hook.fb.at2(off);
            } else {
                return make_double2(0.0, 0.0);
            }
        };
        cplx<T> v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) {
            v[m] = s[(t + TT * m) * B + b];
            if (valid) {
                const long long off = base + static_cast<long long>(t + TT * m) * row_stride;
                if constexpr (kDelta) hook.pre_d(v[m], off, c, delta(m, off));
                else hook.pre(v[m], off, c);
            }
        }
        stockham<T, L, E, 1, DIR>(v, t, tw, XchCol<T, E>{s + b, B});
        if constexpr (!kDelta) {
            fence_proxy_async_smem();  // this thread's exchange writes before the async refill
            __syncthreads();           // every thread is done with buffer `slot`
            if (threadIdx.x == 0 && tile + 2 * gridDim.x < ntiles) issue(tile + 2 * gridDim.x, slot);
        }
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const long long off = base + static_cast<long long>(t + TT * m) * row_stride;
            if (valid) {
                if constexpr (kDelta) hook.post_d(v[m], off, c, delta(m, off));
                else hook.post(v[m], off, c);
                if constexpr (hook_stores<Hook>()) dst[off] = v[m];
            }
        }
        if constexpr (kDelta) {  // the side tile is read in the store loop: refill after it
            fence_proxy_async_smem();
            __syncthreads();
            if (threadIdx.x == 0 && tile + 2 * gridDim.x < ntiles) issue(tile + 2 * gridDim.x, slot);
        }
        if constexpr (hook_tiled<Hook>()) hook.tile_end();
    }
    hook.finish();
}

// TMA-staged column pass for tiles too large to double-buffer (FP64 L >= 1024 at B = 8 columns,
// FP32 L >= 1024 at B = 16: 128-B row segments, which the first-axis pass needs to stay near the
// DRAM page / TLB sweet spot — 64-B segments measured 0.38 of HBM at 1024^3).  One dense TMA
// landing buffer (L x B complex) plus a separate scalar exchange buffer (XchColS): the next
// tile's box load is issued as soon as this tile's elements are in registers, so it lands while
// the current tile is transformed, hooked and stored.  Delta of kDelta hooks is read from global
// memory (the per-component side tile stays with k_col_tma).
// smem: L x B complex + (L + L/E) x B scalars + 1 mbarrier.
template <class T, int L, int E, int DIR, class Hook, int NT>
__global__ void __launch_bounds__(NT, (NT < 512 ? 512 / NT : 1))
    k_col_tma1(const __grid_constant__ CUtensorMap map, cplx<T>* __restrict__ dst,
               long long row_stride, long long plane_stride, int ncols, int B, long long ntiles,
               const cplx<T>* __restrict__ tw, const int* gate, Hook hook) {
    if (gated(gate)) return;
    hook_begin(hook);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int TT = L / E;
    constexpr int LB = L < 256 ? L : 256;
    constexpr bool kDelta = hook_delta<Hook>();
    const int b = threadIdx.x % B;
    const int t = threadIdx.x / B;
    const int tiles_c = (ncols + B - 1) / B;
    cplx<T>* land = reinterpret_cast<cplx<T>*>(smem_raw);
    T* xs = reinterpret_cast<T*>(land + L * B);
    uint64_t* bar = reinterpret_cast<uint64_t*>(
        smem_raw + ((static_cast<size_t>(L) * B * sizeof(cplx<T>) +
                     static_cast<size_t>(L + L / E) * B * sizeof(T) + 15) & ~size_t(15)));
    const unsigned tile_bytes = static_cast<unsigned>(L) * B * sizeof(cplx<T>);
    auto issue = [&](long long tile) {
        const long long plane = tile / tiles_c;
        const int c0 = static_cast<int>(tile - plane * tiles_c) * B;
        mbar_arrive_expect_tx(bar, tile_bytes);
#pragma unroll
        for (int j = 0; j < L / LB; ++j)
            tma_load_3d(land + j * LB * B, &map, bar, 2 * c0, j * LB, static_cast<int>(plane));
    };
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&map);
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < ntiles) issue(blockIdx.x);
    unsigned phase = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        mbar_wait(bar, phase);
        phase ^= 1u;
        const long long plane = tile / tiles_c;
        if constexpr (hook_tiled<Hook>()) {
            if (hook.tile_skip(plane)) {  // frame done: drop the tile, keep the pipeline going
                fence_proxy_async_smem();
                __syncthreads();
                if (threadIdx.x == 0 && tile + gridDim.x < ntiles) issue(tile + gridDim.x);
                continue;
            }
            hook.tile_begin(plane);
        }
        const int c = static_cast<int>(tile - plane * tiles_c) * B + b;
        const bool valid = c < ncols;
        const long long base = plane * plane_stride + c;
        cplx<T> v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[m] = land[(t + TT * m) * B + b];
        fence_proxy_async_smem();  // generic reads of the landing buffer before the async refill
        __syncthreads();
        if (threadIdx.x == 0 && tile + gridDim.x < ntiles) issue(tile + gridDim.x);
        if (valid) {
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const long long off = base + static_cast<long long>(t + TT * m) * row_stride;
                if constexpr (kDelta) hook.pre_d(v[m], off, c, hook.fb.at2(off));
                else hook.pre(v[m], off, c);
            }
        }
        stockham<T, L, E, 1, DIR>(v, t, tw, XchColS<T, E>{xs + b, B});
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const long long off = base + static_cast<long long>(t + TT * m) * row_stride;
            if (valid) {
                if constexpr (kDelta) hook.post_d(v[m], off, c, hook.fb.at2(off));
                else hook.post(v[m], off, c);
                if constexpr (hook_stores<Hook>()) dst[off] = v[m];
            }
        }
        if constexpr (hook_tiled<Hook>()) hook.tile_end();
    }
    hook.finish();
}

// Round trip along one column axis (k_col_tma1's tile walk): forward L-point transform, the
// hook's check / clip on the spectrum values (hook.mid), inverse transform, store into another
// buffer — the loop's K3a (check) and K3b (clip + first inverse pass) as ONE read and ONE write
// of the half spectrum instead of two of each.  The hook's 1-B marks of the tile land by TMA too
// (a second map, MB >= 16 columns wide, its own mbarrier): they are read from shared memory in
// the check / clip, and the next tile's marks are requested right after it, so they land during
// the inverse transform and the stores (no dependent global load, no registers held across the
// forward transform).  hook.fwd_only() (CTA-uniform) stores the forward values instead:
// the same instructions re-form the spectrum bit for bit (the recovery launch after the loop's
// last, discarded clip; HookRT).
// smem: L x B complex (landing) + (L + L/E) x B scalars (exchange) + L x MB marks + 2 mbarriers.
template <class T, int L, int E>
constexpr size_t col_rt_smem_bytes(int B, int MB) {
    return ((static_cast<size_t>(L) * B * sizeof(cplx<T>) +
             static_cast<size_t>(L + L / E) * B * sizeof(T) + static_cast<size_t>(L) * MB + 15) &
            ~size_t(15)) + 32;
}

template <class T, int L, int E, class Hook, int NT>
__global__ void __launch_bounds__(NT, 1)
    k_col_tma1_rt(const __grid_constant__ CUtensorMap map, const __grid_constant__ CUtensorMap mmap,
                  cplx<T>* __restrict__ dst, long long row_stride, long long plane_stride,
                  int ncols, int B, int MB, long long ntiles, const cplx<T>* __restrict__ tw,
                  const int* gate, const Hook hook) {
    if (gated(gate)) return;
    const bool first = hook.is_first();
    double peak = 0.0, ex = 0.0;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int TT = L / E;
    constexpr int LB = L < 256 ? L : 256;
    const int b = threadIdx.x % B;
    const int t = threadIdx.x / B;
    const int tiles_c = (ncols + B - 1) / B;
    const bool fwd_only = hook.fwd_only();
    cplx<T>* land = reinterpret_cast<cplx<T>*>(smem_raw);
    T* xs = reinterpret_cast<T*>(land + L * B);
    unsigned char* mk = reinterpret_cast<unsigned char*>(xs + (L + L / E) * B);
    uint64_t* bar = reinterpret_cast<uint64_t*>(
        smem_raw + ((static_cast<size_t>(L) * B * sizeof(cplx<T>) +
                     static_cast<size_t>(L + L / E) * B * sizeof(T) + static_cast<size_t>(L) * MB +
                     15) & ~size_t(15)));
    uint64_t* mbar = bar + 1;
    auto issue = [&](long long tile) {
        const long long plane = tile / tiles_c;
        const int c0 = static_cast<int>(tile - plane * tiles_c) * B;
        mbar_arrive_expect_tx(bar, static_cast<unsigned>(L) * B * sizeof(cplx<T>));
#pragma unroll
        for (int j = 0; j < L / LB; ++j)
            tma_load_3d(land + j * LB * B, &map, bar, 2 * c0, j * LB, static_cast<int>(plane));
    };
    auto issue_marks = [&](long long tile) {
        const long long plane = tile / tiles_c;
        const int c0 = static_cast<int>(tile - plane * tiles_c) * B;
        mbar_arrive_expect_tx(mbar, static_cast<unsigned>(L) * MB);
#pragma unroll
        for (int j = 0; j < L / LB; ++j)
            tma_load_3d(mk + j * LB * MB, &mmap, mbar, c0 - c0 % MB, j * LB,
                        static_cast<int>(plane));
    };
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&map);
        tma_prefetch_desc(&mmap);
        mbar_init(bar, 1);
        mbar_init(mbar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < ntiles) {
        issue(blockIdx.x);
        issue_marks(blockIdx.x);
    }
    unsigned phase = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        mbar_wait(bar, phase);
        const long long plane = tile / tiles_c;
        const int c0 = static_cast<int>(tile - plane * tiles_c) * B;
        const int c = c0 + b;
        const bool valid = c < ncols;
        const long long base = plane * plane_stride + c;
        const int mcol = c0 % MB + b;
        cplx<T> v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[m] = land[(t + TT * m) * B + b];
        fence_proxy_async_smem();  // generic reads of the landing buffer before the async refill
        __syncthreads();
        if (threadIdx.x == 0 && tile + gridDim.x < ntiles) issue(tile + gridDim.x);
        stockham<T, L, E, 1, -1>(v, t, tw, XchColS<T, E>{xs + b, B});
        mbar_wait(mbar, phase);
        phase ^= 1u;
        if (valid) {
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const long long off = base + static_cast<long long>(t + TT * m) * row_stride;
                hook.mid(v[m], off, hook.fb.at2(off), mk[(t + TT * m) * MB + mcol], first, peak,
                         ex);
            }
        }
        fence_proxy_async_smem();  // generic reads of the marks before their async refill
        __syncthreads();
        if (threadIdx.x == 0 && tile + gridDim.x < ntiles) issue_marks(tile + gridDim.x);
        if (!fwd_only) {
            // a fresh twiddle pointer: keeps the compiler from carrying the forward transform's
            // twiddle powers across the hook into the inverse (CSE; 560 B of spills)
            const cplx<T>* twi;
            asm volatile("mov.b64 %0, %1;" : "=l"(twi) : "l"(tw));
            stockham<T, L, E, 1, +1>(v, t, twi, XchColS<T, E>{xs + b, B});
        }
        if (valid) {
            // (the store addresses re-formed from an opaque base: not the hook's 16 live offsets)
            cplx<T>* out;
            asm volatile("mov.b64 %0, %1;" : "=l"(out) : "l"(dst + base));
#pragma unroll
            for (int m = 0; m < E; ++m) out[static_cast<long long>(t + TT * m) * row_stride] = v[m];
        }
    }
    hook.finish(peak, ex);
}

// The gate's F rebuild on the completing axis (HookFRebuild's arithmetic, k_col_tma1's tile walk):
// forward transform of FFT(eps0 + S)'s partial spectrum, then F = mark ? delta_final - v : 0, no
// store of v.  The tile's marks land with it (UINT8 map); delta_final's tile lands in the same
// landing buffer once the tile is in registers (during the transform), so the hook issues no
// dependent global load — HookFRebuild's two per-element loads held the pass at 10.3 ms at 1024^3
// (2.6 TB/s).  The next tile is requested after the F stores (no overlap of its load with this
// tile's transform: the landing buffer holds delta until then).
// smem: as k_col_tma1_rt (landing + exchange + L x MB marks + 2 mbarriers).
template <class T, int L, int E, int NT>
__global__ void __launch_bounds__(NT, 1)
    k_col_tma1_frebuild(const __grid_constant__ CUtensorMap map,
                        const __grid_constant__ CUtensorMap mmap,
                        const __grid_constant__ CUtensorMap dmap, cplx<T>* __restrict__ F,
                        long long row_stride, long long plane_stride, int ncols, int B, int MB,
                        long long ntiles, const cplx<T>* __restrict__ tw) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int TT = L / E;
    constexpr int LB = L < 256 ? L : 256;
    const int b = threadIdx.x % B;
    const int t = threadIdx.x / B;
    const int tiles_c = (ncols + B - 1) / B;
    cplx<T>* land = reinterpret_cast<cplx<T>*>(smem_raw);
    T* xs = reinterpret_cast<T*>(land + L * B);
    unsigned char* mk = reinterpret_cast<unsigned char*>(xs + (L + L / E) * B);
    uint64_t* bar = reinterpret_cast<uint64_t*>(
        smem_raw + ((static_cast<size_t>(L) * B * sizeof(cplx<T>) +
                     static_cast<size_t>(L + L / E) * B * sizeof(T) + static_cast<size_t>(L) * MB +
                     15) & ~size_t(15)));
    uint64_t* dbar = bar + 1;
    const unsigned data_bytes = static_cast<unsigned>(L) * B * sizeof(cplx<T>);
    auto issue = [&](long long tile) {  // the tile's partial spectrum + its marks
        const long long plane = tile / tiles_c;
        const int c0 = static_cast<int>(tile - plane * tiles_c) * B;
        mbar_arrive_expect_tx(bar, data_bytes + static_cast<unsigned>(L) * MB);
#pragma unroll
        for (int j = 0; j < L / LB; ++j) {
            tma_load_3d(land + j * LB * B, &map, bar, 2 * c0, j * LB, static_cast<int>(plane));
            tma_load_3d(mk + j * LB * MB, &mmap, bar, c0 - c0 % MB, j * LB,
                        static_cast<int>(plane));
        }
    };
    auto issue_delta = [&](long long tile) {
        const long long plane = tile / tiles_c;
        const int c0 = static_cast<int>(tile - plane * tiles_c) * B;
        mbar_arrive_expect_tx(dbar, data_bytes);
#pragma unroll
        for (int j = 0; j < L / LB; ++j)
            tma_load_3d(land + j * LB * B, &dmap, dbar, 2 * c0, j * LB, static_cast<int>(plane));
    };
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&map);
        tma_prefetch_desc(&mmap);
        tma_prefetch_desc(&dmap);
        mbar_init(bar, 1);
        mbar_init(dbar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < ntiles) issue(blockIdx.x);
    unsigned phase = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        mbar_wait(bar, phase);
        const long long plane = tile / tiles_c;
        const int c0 = static_cast<int>(tile - plane * tiles_c) * B;
        const int c = c0 + b;
        const bool valid = c < ncols;
        const long long base = plane * plane_stride + c;
        const int mcol = c0 % MB + b;
        cplx<T> v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[m] = land[(t + TT * m) * B + b];
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) issue_delta(tile);
        stockham<T, L, E, 1, -1>(v, t, tw, XchColS<T, E>{xs + b, B});
        mbar_wait(dbar, phase);
        phase ^= 1u;
        if (valid) {
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int i = t + TT * m;
                const cplx<T> d = land[i * B + b];
                F[base + static_cast<long long>(i) * row_stride] =
                    mk[i * MB + mcol] ? mkc<T>(d.x - v[m].x, d.y - v[m].y) : mkc<T>(T(0), T(0));
            }
        }
        fence_proxy_async_smem();  // generic reads of delta / marks before the next async fill
        __syncthreads();
        if (threadIdx.x == 0 && tile + gridDim.x < ntiles) issue(tile + gridDim.x);
    }
}

// Column pass of an L-point line split over a 2-CTA cluster (DSMEM): CTA h of the pair lands
// rows [h L/2, (h+1) L/2) of a B-column tile by TMA, so a tile can be twice as wide as one SM's
// shared memory allows (FP64: L = 1024 at 16 columns = 256-B rows, L = 2048 at 8 columns =
// 128-B rows — the outer / 2048-point passes measured 0.38-0.67 of HBM at 64-128-B rows).
// One decimation-in-frequency radix-2 stage across the pair: CTA 0 forms u_i = x_i + x_{i+L/2},
// CTA 1 forms v_i = (x_i - x_{i+L/2}) W_L^{+-i}, reading the partner's landing tile through
// distributed shared memory; each then runs an L/2-point Stockham transform and stores rows
// 2q + h.  The next tile's box is issued once both CTAs have read the landing buffers, so it
// lands during the L/2-point transform and the stores.  Pre-hooks run on the landing tile
// (owner only) before the exchange; post-hooks on the stored elements.
// smem per CTA: (L/2) x B complex (landing) + (L/2 + L/2/E) x B scalars (exchange) + mbarrier.
template <class T, int L, int E, int DIR, class Hook, int NT>
__global__ void __launch_bounds__(NT, 1)
    k_col_c2(const __grid_constant__ CUtensorMap map, cplx<T>* __restrict__ dst,
             long long row_stride, long long plane_stride, int ncols, int B, long long ntiles,
             const cplx<T>* __restrict__ tw, const cplx<T>* __restrict__ twl, const int* gate,
             Hook hook) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    if (gated(gate)) return;  // uniform over the pair: both CTAs read the same flag
    hook_begin(hook);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int LH = L / 2;
    constexpr int TT = LH / E;
    constexpr int LB = LH < 256 ? LH : 256;
    const unsigned h = cluster.block_rank();
    const int b = threadIdx.x % B;
    const int t = threadIdx.x / B;
    const int tiles_c = (ncols + B - 1) / B;
    cplx<T>* land = reinterpret_cast<cplx<T>*>(smem_raw);
    T* xs = reinterpret_cast<T*>(land + LH * B);
    uint64_t* bar = reinterpret_cast<uint64_t*>(
        smem_raw + ((static_cast<size_t>(LH) * B * sizeof(cplx<T>) +
                     static_cast<size_t>(LH + LH / E) * B * sizeof(T) + 15) & ~size_t(15)));
    const cplx<T>* peer = cluster.map_shared_rank(land, h ^ 1u);
    const unsigned tile_bytes = static_cast<unsigned>(LH) * B * sizeof(cplx<T>);
    const long long pair = blockIdx.x / 2, npairs = gridDim.x / 2;
    auto issue = [&](long long tile) {
        const long long plane = tile / tiles_c;
        const int c0 = static_cast<int>(tile - plane * tiles_c) * B;
        mbar_arrive_expect_tx(bar, tile_bytes);
#pragma unroll
        for (int j = 0; j < LH / LB; ++j)
            tma_load_3d(land + j * LB * B, &map, bar, 2 * c0, static_cast<int>(h) * LH + j * LB,
                        static_cast<int>(plane));
    };
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&map);
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0 && pair < ntiles) issue(pair);
    unsigned phase = 0;
    for (long long tile = pair; tile < ntiles; tile += npairs) {
        mbar_wait(bar, phase);
        phase ^= 1u;
        const long long plane = tile / tiles_c;
        bool skip = false;
        if constexpr (hook_tiled<Hook>()) {
            skip = hook.tile_skip(plane);
            if (!skip) hook.tile_begin(plane);
        }
        const int c = static_cast<int>(tile - plane * tiles_c) * B + b;
        const bool valid = c < ncols;
        const long long base = plane * plane_stride + c;
        if (!skip && valid) {  // pre-hooks on the owned half, in place
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int i = t + TT * m;
                const long long off = base + static_cast<long long>(h * LH + i) * row_stride;
                cplx<T> x = land[i * B + b];
                hook.pre(x, off, c);
                land[i * B + b] = x;
            }
        }
        cluster.sync();  // both halves landed and pre-hooked
        cplx<T> v[E];
        if (!skip) {
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int i = t + TT * m;
                const cplx<T> mine = land[i * B + b], other = peer[i * B + b];
                const cplx<T> a = h ? other : mine, bb = h ? mine : other;  // x_i, x_{i+L/2}
                if (h == 0) {
                    v[m] = cadd(a, bb);
                } else {
                    const cplx<T> w = twl[i];  // W_L^i = exp(-2 pi i i / L)
                    v[m] = DIR < 0 ? cmul(csub(a, bb), w) : cmulc(csub(a, bb), w);
                }
            }
        }
        fence_proxy_async_smem();
        cluster.sync();  // both CTAs are done with both landing tiles
        if (threadIdx.x == 0 && tile + npairs < ntiles) issue(tile + npairs);
        if (skip) continue;
        stockham<T, LH, E, 1, DIR>(v, t, tw, XchColS<T, E>{xs + b, B});
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const long long r = 2LL * (t + TT * m) + h;
            const long long off = base + r * row_stride;
            if (valid) {
                hook.post(v[m], off, c);
                if constexpr (hook_stores<Hook>()) dst[off] = v[m];
            }
        }
        if constexpr (hook_tiled<Hook>()) hook.tile_end();
    }
    hook.finish();
    cluster.sync();  // no CTA exits while its partner may still read its shared memory
}

template <class T, int L, int E>
constexpr size_t col_c2_smem_bytes(int B) {
    return ((static_cast<size_t>(L / 2) * B * sizeof(cplx<T>) +
             static_cast<size_t>(L / 2 + L / 2 / E) * B * sizeof(T) + 15) & ~size_t(15)) + 16;
}

template <class T, int L, int E>
constexpr size_t col_tma1_smem_bytes(int B) {
    return ((static_cast<size_t>(L) * B * sizeof(cplx<T>) +
             static_cast<size_t>(L + L / E) * B * sizeof(T) + 15) & ~size_t(15)) + 16;
}

template <class T, int L, int E>
constexpr size_t col_tma_smem_bytes(int B, bool side) {
    return 2 * static_cast<size_t>(L + L / E) * B * sizeof(cplx<T>) +
           (side ? 2 * static_cast<size_t>(L) * B * sizeof(double) : 0) + 2 * sizeof(uint64_t);
}

template <class T, int L, int E>
constexpr size_t col_smem_bytes(int B) {
    return static_cast<size_t>(L + L / E) * B * sizeof(cplx<T>);
}

// ---- row passes: last (contiguous) axis, n2 = 2M real <-> M+1 complex ---------------------------
// The n2 reals of a row are read as M complex z[j] = x[2j] + i x[2j+1]; an M-point FFT plus the
// split/merge with W_{2M}^k gives X[0..M] (classic packed real FFT).

template <int M, int E>
constexpr int row_smem_elems() { return M + M / E + 2; }

// Split Z (in smem, natural order at XchRow positions) into X[k] = Ze + W_{2M}^k Zo.
// twp[k] = W_{2M}^k = exp(-2 pi i k / 2M), k in [0, M]
template <class T, int M, int E>
__device__ __forceinline__ cplx<T> r2c_split(const cplx<T>* s, int k, const cplx<T>* __restrict__ twp) {
    using X = XchRow<T, E>;
    const cplx<T> zk = s[X::pos(k)];
    const cplx<T> zn = s[X::pos((M - k) & (M - 1))];
    const T h = T(0.5);
    cplx<T> ze = mkc<T>((zk.x + zn.x) * h, (zk.y - zn.y) * h);
    cplx<T> zo = mkc<T>((zk.y + zn.y) * h, (zn.x - zk.x) * h);
    const cplx<T> w = twp[k];
    return cadd(ze, cmul(zo, w));
}

// Merge X[k], X[M-k] (smem) into Z[k] = (X_k + conj X_{M-k}) + i (X_k - conj X_{M-k}) W^{-k};
// imaginary parts of X[0] and X[M] are dropped (= Re of the full c2c inverse).
template <class T, int M, int E>
__device__ __forceinline__ cplx<T> c2r_merge(const cplx<T>* s, int k, const cplx<T>* __restrict__ twp) {
    using X = XchRow<T, E>;
    cplx<T> a = s[X::pos(k)];
    cplx<T> b = s[X::pos(M - k)];
    if (k == 0) {
        a.y = T(0);
        b.y = T(0);
    }
    const cplx<T> ze = mkc<T>(a.x + b.x, a.y - b.y);
    const cplx<T> d = mkc<T>(a.x - b.x, a.y + b.y);
    const cplx<T> w = twp[k];
    const cplx<T> zo = cmulc(d, w);
    return mkc<T>(ze.x - zo.y, ze.y + zo.x);
}

// Real-output hook for C2R rows: post_real(x0, x1, n) gets the two scaled reals of sample pair
// (n, n+1) and may modify them before the store.
struct RealHookNone {
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    template <class T> __device__ __forceinline__ void post_real(T&, T&, long long) {}
    __device__ __forceinline__ void finish() {}
};

// Plain R2C of rows (FP32 or FP64 real input of the same type).
// Launched with blockDim.x = (M/E) * rows-per-CTA threads, row_smem_elems() per row of smem.
template <class T, int M, int E, class Hook>
__global__ void __launch_bounds__(max_threads<T, E>(), 512 / max_threads<T, E>())
    k_row_r2c(const T* __restrict__ in, long long in_stride, cplx<T>* __restrict__ out,
              long long out_stride, long long nrows, const cplx<T>* __restrict__ tw,
              const cplx<T>* __restrict__ twp, const int* gate, Hook hook) {
    if (gated(gate)) return;
    hook_begin(hook);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int TT = M / E;
    const int t = threadIdx.x % TT;
    const int rb = threadIdx.x / TT;
    const long long ntiles = (nrows + (blockDim.x / TT) - 1) / (blockDim.x / TT);
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        __syncthreads();  // smem of the previous tile fully consumed
        if constexpr (hook_tiled<Hook>()) {
            const long long u = tile * (blockDim.x / TT);
            if (hook.tile_skip(u)) continue;
            hook.tile_begin(u);
        }
        const long long row = tile * (blockDim.x / TT) + rb;
        const bool valid = row < nrows;
        cplx<T>* s = reinterpret_cast<cplx<T>*>(smem_raw) + rb * row_smem_elems<M, E>();
        const cplx<T>* src = reinterpret_cast<const cplx<T>*>(in + (valid ? row : 0) * in_stride);
        cplx<T> v[E];
    #pragma unroll
        for (int m = 0; m < E; ++m) v[m] = valid ? src[t + TT * m] : mkc<T>(T(0), T(0));
        const XchRow<T, E> x{s};
        stockham<T, M, E, 1, -1>(v, t, tw, x);
        __syncthreads();
    #pragma unroll
        for (int m = 0; m < E; ++m) x.st(t + TT * m, v[m]);
        __syncthreads();
        if (valid) {
            cplx<T>* dst = out + row * out_stride;
    #pragma unroll
            for (int m = 0; m < E; ++m) {
                const int k = t + TT * m;
                cplx<T> X = r2c_split<T, M, E>(s, k, twp);
                hook.post(X, row * out_stride + k, k);
                dst[k] = X;
            }
            if (t == 0) {
                const cplx<T> z0 = s[0];
                cplx<T> X = mkc<T>(z0.x - z0.y, T(0));
                hook.post(X, row * out_stride + M, M);
                dst[M] = X;
            }
        }
        if constexpr (hook_tiled<Hook>()) hook.tile_end();
    }
    hook.finish();
}

// Plain C2R of rows: out = scale * (unnormalised inverse along the last axis).
// Launched with blockDim.x = (M/E) * rows-per-CTA threads, row_smem_elems() per row of smem.
template <class T, int M, int E, class Hook>
__global__ void __launch_bounds__(max_threads<T, E>(), 512 / max_threads<T, E>())
    k_row_c2r(const cplx<T>* __restrict__ in, long long in_stride, T* __restrict__ out,
              long long out_stride, long long nrows, const cplx<T>* __restrict__ tw,
              const cplx<T>* __restrict__ twp, T scale, const int* gate, Hook hook) {
    if (gated(gate)) return;
    hook_begin(hook);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int TT = M / E;
    const int t = threadIdx.x % TT;
    const int rb = threadIdx.x / TT;
    const long long ntiles = (nrows + (blockDim.x / TT) - 1) / (blockDim.x / TT);
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        __syncthreads();  // smem of the previous tile fully consumed
        if constexpr (hook_tiled<Hook>()) {
            const long long u = tile * (blockDim.x / TT);
            if (hook.tile_skip(u)) continue;
            hook.tile_begin(u);
        }
        const long long row = tile * (blockDim.x / TT) + rb;
        const bool valid = row < nrows;
        cplx<T>* s = reinterpret_cast<cplx<T>*>(smem_raw) + rb * row_smem_elems<M, E>();
        const XchRow<T, E> x{s};
        const cplx<T>* src = in + (valid ? row : 0) * in_stride;
    #pragma unroll
        for (int m = 0; m < E; ++m) {
            const int k = t + TT * m;
            cplx<T> X = valid ? src[k] : mkc<T>(T(0), T(0));
            hook.pre(X, row * in_stride + k, k);
            x.st(k, X);
        }
        if (t == 0) {
            cplx<T> X = valid ? src[M] : mkc<T>(T(0), T(0));
            hook.pre(X, row * in_stride + M, M);
            x.st(M, X);
        }
        __syncthreads();
        cplx<T> v[E];
    #pragma unroll
        for (int m = 0; m < E; ++m) v[m] = c2r_merge<T, M, E>(s, t + TT * m, twp);
        stockham<T, M, E, 1, +1>(v, t, tw, x);
        if (valid) {
            cplx<T>* dst = reinterpret_cast<cplx<T>*>(out + row * out_stride);
    #pragma unroll
            for (int m = 0; m < E; ++m) {
                const int j = t + TT * m;
                T x0 = v[m].x * scale, x1 = v[m].y * scale;
                hook.post_real(x0, x1, row * out_stride + 2 * j);
                dst[j] = mkc<T>(x0, x1);
            }
        }
        if constexpr (hook_tiled<Hook>()) hook.tile_end();
    }
    hook.finish();
}

// Fused last-axis pass of the projection loop: C2R -> (scale, s-cube clip via hook) -> R2C,
// in place on the half spectrum (or into `out`).  The real epsilon never round-trips HBM except for the hook's
// own write.
// Launched with blockDim.x = (M/E) * rows-per-CTA threads, row_smem_elems() per row of smem.
template <class T, int M, int E, class Hook>
__global__ void __launch_bounds__(max_threads<T, E>(), 512 / max_threads<T, E>())
    k_row_c2r_r2c(cplx<T>* data, long long stride, long long nrows, long long real_stride,
                  const cplx<T>* __restrict__ tw, const cplx<T>* __restrict__ twp, T scale,
                  const int* gate, Hook hook, cplx<T>* out) {
    if (gated(gate)) return;
    hook_begin(hook);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int TT = M / E;
    const int t = threadIdx.x % TT;
    const int rb = threadIdx.x / TT;
    const long long ntiles = (nrows + (blockDim.x / TT) - 1) / (blockDim.x / TT);
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        __syncthreads();  // smem of the previous tile fully consumed
        if constexpr (hook_tiled<Hook>()) {
            const long long u = tile * (blockDim.x / TT);
            if (hook.tile_skip(u)) continue;
            hook.tile_begin(u);
        }
        const long long row = tile * (blockDim.x / TT) + rb;
        const bool valid = row < nrows;
        cplx<T>* s = reinterpret_cast<cplx<T>*>(smem_raw) + rb * row_smem_elems<M, E>();
        const XchRow<T, E> x{s};
        cplx<T>* rowp = data + (valid ? row : 0) * stride;
    #pragma unroll
        for (int m = 0; m < E; ++m) {
            const int k = t + TT * m;
            x.st(k, valid ? rowp[k] : mkc<T>(T(0), T(0)));
        }
        if (t == 0) x.st(M, valid ? rowp[M] : mkc<T>(T(0), T(0)));
        __syncthreads();
        cplx<T> v[E];
    #pragma unroll
        for (int m = 0; m < E; ++m) v[m] = c2r_merge<T, M, E>(s, t + TT * m, twp);
        stockham<T, M, E, 1, +1>(v, t, tw, x);
    #pragma unroll
        for (int m = 0; m < E; ++m) {
            const int j = t + TT * m;
            T x0 = v[m].x * scale, x1 = v[m].y * scale;
            if (valid) hook.post_real(x0, x1, row * real_stride + 2 * j);
            v[m] = mkc<T>(x0, x1);
        }
        stockham<T, M, E, 1, -1>(v, t, tw, x);
        __syncthreads();
    #pragma unroll
        for (int m = 0; m < E; ++m) x.st(t + TT * m, v[m]);
        __syncthreads();
        if (valid) {
            cplx<T>* rowo = out ? out + row * stride : rowp;
    #pragma unroll
            for (int m = 0; m < E; ++m) {
                const int k = t + TT * m;
                rowo[k] = r2c_split<T, M, E>(s, k, twp);
            }
            if (t == 0) {
                const cplx<T> z0 = s[0];
                rowo[M] = mkc<T>(z0.x - z0.y, T(0));
            }
        }
        if constexpr (hook_tiled<Hook>()) hook.tile_end();
    }
    hook.finish();
}

// Input prefetch for C2R epilogue hooks (k_row_c2r_sh): a hook with kPrefetch names two input
// fields (prefetch_src(k, first_sample)), their scalar size (prefetch_scalar_bytes) and takes the
// shared-memory copies per tile (use_prefetch(orig_s, dec_s, first_sample)).
template <class H>
constexpr bool hook_prefetch() {
    if constexpr (requires { H::kPrefetch; })
        return H::kPrefetch;
    else
        return false;
}

// ---- row passes with warp-shuffle pairing (M/E <= 32) --------------------------------------------
// The split/merge needs X[k] and X[M-k] together.  Instead of a shared-memory round trip, rows are
// loaded in a "paired" layout: thread t holds X[t + T m] in slot m and X[M - t - T m] in slot
// E-1-m (m < E/2; descending addresses are still coalesced), so the merge is thread-local; one
// exchange of E/2 values with the partner lane (T - t) mod T converts to the natural layout the
// Stockham stages need (and back for the split).  Thread 0 additionally owns the self-paired
// index M/2 and, through slot E-1, the Nyquist X[M].

template <class T>
__device__ __forceinline__ cplx<T> shfl_c(cplx<T> v, int src, int width) {
    v.x = __shfl_sync(0xffffffffu, v.x, src, width);
    v.y = __shfl_sync(0xffffffffu, v.y, src, width);
    return v;
}

// X_k, X_{M-k}, W_{2M}^k -> Z_k  (c2r_merge on registers; `dc` drops Im of X_0 and X_M)
template <class T>
__device__ __forceinline__ cplx<T> merge_pair(cplx<T> a, cplx<T> b, cplx<T> w, bool dc) {
    if (dc) {
        a.y = T(0);
        b.y = T(0);
    }
    const cplx<T> ze = mkc<T>(a.x + b.x, a.y - b.y);
    const cplx<T> d = mkc<T>(a.x - b.x, a.y + b.y);
    const cplx<T> zo = cmulc(d, w);
    return mkc<T>(ze.x - zo.y, ze.y + zo.x);
}

// Z_k, Z_{M-k}, W_{2M}^k -> X_k (r2c_split on registers)
template <class T>
__device__ __forceinline__ cplx<T> split_pair(cplx<T> zk, cplx<T> zn, cplx<T> w) {
    const T h = T(0.5);
    const cplx<T> ze = mkc<T>((zk.x + zn.x) * h, (zk.y - zn.y) * h);
    const cplx<T> zo = mkc<T>((zk.y + zn.y) * h, (zn.x - zk.x) * h);
    return cadd(ze, cmul(zo, w));
}

template <class T, int M, int E>
__device__ __forceinline__ void load_pairs(const cplx<T>* __restrict__ rowp, int t, bool valid,
                                           cplx<T> (&v)[E], cplx<T>& mid) {
    constexpr int TT = M / E;
#pragma unroll
    for (int m = 0; m < E / 2; ++m) {
        v[m] = valid ? rowp[t + TT * m] : mkc<T>(T(0), T(0));
        v[E - 1 - m] = valid ? rowp[M - t - TT * m] : mkc<T>(T(0), T(0));
    }
    mid = (valid && t == 0) ? rowp[M / 2] : mkc<T>(T(0), T(0));
}

template <class T, int M, int E>
__device__ __forceinline__ void merge_pairs(cplx<T> (&v)[E], cplx<T>& mid, int t,
                                            const cplx<T>* __restrict__ twp) {
    constexpr int TT = M / E;
#pragma unroll
    for (int m = 0; m < E / 2; ++m) {
        const int k = t + TT * m;
        const cplx<T> a = v[m], b = v[E - 1 - m];
        const bool dc = (k == 0);
        v[m] = merge_pair<T>(a, b, twp[k], dc);
        v[E - 1 - m] = merge_pair<T>(b, a, twp[M - k], false);  // unused when k == 0
    }
    if (t == 0) mid = merge_pair<T>(mid, mid, twp[M / 2], false);
}

// paired -> natural (v[m] = Z[t + T m]); ascending so thread 0 reads slots not yet replaced
template <class T, int M, int E>
__device__ __forceinline__ void pairs_to_natural(cplx<T> (&v)[E], cplx<T> mid, int t) {
    constexpr int TT = M / E;
    const int src = (TT - t) & (TT - 1);
#pragma unroll
    for (int m = 0; m < E / 2; ++m) {
        cplx<T> send = v[E - 1 - m];
        if (t == 0) send = (m + 1 < E / 2) ? v[E - 2 - m] : mid;
        v[E - 1 - m] = shfl_c<T>(send, src, TT);
    }
}

// natural -> paired; descending so thread 0 reads slots not yet replaced.  Returns Z[M/2] in
// thread 0.
template <class T, int M, int E>
__device__ __forceinline__ cplx<T> natural_to_pairs(cplx<T> (&v)[E], int t) {
    constexpr int TT = M / E;
    const int src = (TT - t) & (TT - 1);
    const cplx<T> mid = v[E / 2];
#pragma unroll
    for (int m = E / 2 - 1; m >= 0; --m) {
        cplx<T> send = v[E - 1 - m];
        if (t == 0) send = (m == 0) ? v[0] : v[E - m];
        v[E - 1 - m] = shfl_c<T>(send, src, TT);
    }
    return mid;
}

template <class T, int M, int E, class Hook>
__device__ __forceinline__ void split_store(cplx<T> (&v)[E], cplx<T> mid, int t, bool valid,
                                            cplx<T>* rowp, long long row_off,
                                            const cplx<T>* __restrict__ twp, Hook& hook) {
    constexpr int TT = M / E;
#pragma unroll
    for (int m = 0; m < E / 2; ++m) {
        const int k = t + TT * m;
        const cplx<T> zk = v[m], zn = v[E - 1 - m];
        cplx<T> xk, xn;
        if (k == 0) {
            xk = mkc<T>(zk.x + zk.y, T(0));
            xn = mkc<T>(zk.x - zk.y, T(0));
        } else {
            xk = split_pair<T>(zk, zn, twp[k]);
            xn = split_pair<T>(zn, zk, twp[M - k]);
        }
        if (valid) {
            hook.post(xk, row_off + k, k);
            hook.post(xn, row_off + (M - k), M - k);
            rowp[k] = xk;
            rowp[M - k] = xn;
        }
    }
    if (valid && t == 0) {
        cplx<T> xm = split_pair<T>(mid, mid, twp[M / 2]);
        hook.post(xm, row_off + M / 2, M / 2);
        rowp[M / 2] = xm;
    }
}

template <class T, int M, int E, class Hook>
__global__ void __launch_bounds__(max_threads<T, E>(), 512 / max_threads<T, E>())
    k_row_r2c_sh(const T* __restrict__ in, long long in_stride, cplx<T>* __restrict__ out,
                 long long out_stride, long long nrows, const cplx<T>* __restrict__ tw,
                 const cplx<T>* __restrict__ twp, const int* gate, Hook hook) {
    if (gated(gate)) return;
    hook_begin(hook);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int TT = M / E;
    const int t = threadIdx.x % TT;
    const int rb = threadIdx.x / TT;
    const long long ntiles = (nrows + (blockDim.x / TT) - 1) / (blockDim.x / TT);
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        // (a CTA barrier only where the tile is shared: prefetch buffers, per-frame skips)
        if constexpr (hook_tiled<Hook>()) __syncthreads();
        else __syncwarp();
        if constexpr (hook_tiled<Hook>()) {
            const long long u = tile * (blockDim.x / TT);
            if (hook.tile_skip(u)) continue;
            hook.tile_begin(u);
        }
        const long long row = tile * (blockDim.x / TT) + rb;
        const bool valid = row < nrows;
        cplx<T>* s = reinterpret_cast<cplx<T>*>(smem_raw) + rb * row_smem_elems<M, E>();
        const cplx<T>* src = reinterpret_cast<const cplx<T>*>(in + (valid ? row : 0) * in_stride);
        cplx<T> v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[m] = valid ? src[t + TT * m] : mkc<T>(T(0), T(0));
        stockham<T, M, E, 1, -1>(v, t, tw, XchRowW<T, E>{s});
        const cplx<T> mid = natural_to_pairs<T, M, E>(v, t);
        split_store<T, M, E>(v, mid, t, valid, out + (valid ? row : 0) * out_stride,
                             row * out_stride, twp, hook);
        if constexpr (hook_tiled<Hook>()) hook.tile_end();
    }
    hook.finish();
}

// First forward pass of correct() with compute_error fused in (pipeline.cpp:31-42): rows of
// eps0 = dec - orig are formed in registers from the two input fields (never stored), the two
// preconditions are checked on the way (first failing index -> bad1 / bad2), and the R2C
// proceeds as k_row_r2c_sh.  Saves the separate eps0 pass (read 2 fields + write eps).
template <class TI, int M, int E, class SB, class CTL>
__global__ void __launch_bounds__(max_threads<double, E>(), 512 / max_threads<double, E>())
    k_row_r2c_eps0_sh(const TI* __restrict__ orig, const TI* __restrict__ dec, long long n2,
                      double2* __restrict__ out, long long out_stride, long long nrows,
                      const double2* __restrict__ tw, const double2* __restrict__ twp, SB sb,
                      double fscale, double slack, CTL* ctl, const double* __restrict__ S) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int TT = M / E;
    const int t = threadIdx.x % TT;
    const int rb = threadIdx.x / TT;
    const long long ntiles = (nrows + (blockDim.x / TT) - 1) / (blockDim.x / TT);
    HookNone none;
    unsigned long long bad1 = ~0ull, bad2 = ~0ull;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        __syncwarp();  // (each warp's rows use only its own buffer)
        const long long row = tile * (blockDim.x / TT) + rb;
        const bool valid = row < nrows;
        double2* s = reinterpret_cast<double2*>(smem_raw) + rb * row_smem_elems<M, E>();
        double2 v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const long long n = (valid ? row : 0) * n2 + 2 * (t + TT * m);
            double e0 = 0.0, e1 = 0.0;
            if (valid) {
                if constexpr (sizeof(TI) == 4) {
                    const float2 o = *reinterpret_cast<const float2*>(orig + n);
                    const float2 d = *reinterpret_cast<const float2*>(dec + n);
                    e0 = static_cast<double>(d.x) - static_cast<double>(o.x);
                    e1 = static_cast<double>(d.y) - static_cast<double>(o.y);
                } else {
                    const double2 o = *reinterpret_cast<const double2*>(orig + n);
                    const double2 d = *reinterpret_cast<const double2*>(dec + n);
                    e0 = d.x - o.x;
                    e1 = d.y - o.y;
                }
                if (S) {  // the gate's F rebuild input eps0 + S (k_eps0_plus_s), no checks
                    const double2 sv = *reinterpret_cast<const double2*>(S + n);
                    e0 += sv.x;
                    e1 += sv.y;
                    v[m] = make_double2(e0, e1);
                    continue;
                }
                const double E0 = sb.at(n), E1 = sb.at(n + 1);
                if (fabs(e0) > E0 * (1.0 + 0x1p-20) && static_cast<unsigned long long>(n) < bad1) bad1 = n;
                if (fabs(e1) > E1 * (1.0 + 0x1p-20) && static_cast<unsigned long long>(n + 1) < bad1) bad1 = n + 1;
                if (fabs(e0) > E0 * fscale * (1.0 + slack) && static_cast<unsigned long long>(n) < bad2) bad2 = n;
                if (fabs(e1) > E1 * fscale * (1.0 + slack) && static_cast<unsigned long long>(n + 1) < bad2) bad2 = n + 1;
            }
            v[m] = make_double2(e0, e1);
        }
        stockham<double, M, E, 1, -1>(v, t, tw, XchRowW<double, E>{s});
        const double2 mid = natural_to_pairs<double, M, E>(v, t);
        split_store<double, M, E>(v, mid, t, valid, out + (valid ? row : 0) * out_stride,
                                  row * out_stride, twp, none);
    }
    if (bad1 != ~0ull && ctl) atomicMin(&ctl->bad1, bad1);
    if (bad2 != ~0ull && ctl) atomicMin(&ctl->bad2, bad2);
}

template <class T, int M, int E, class Hook>
__global__ void __launch_bounds__(max_threads<T, E>(), 512 / max_threads<T, E>())
    k_row_c2r_sh(const cplx<T>* __restrict__ in, long long in_stride, T* __restrict__ out,
                 long long out_stride, long long nrows, const cplx<T>* __restrict__ tw,
                 const cplx<T>* __restrict__ twp, T scale, const int* gate, Hook hook) {
    if (gated(gate)) return;
    hook_begin(hook);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int TT = M / E;
    const int t = threadIdx.x % TT;
    const int rb = threadIdx.x / TT;
    const long long ntiles = (nrows + (blockDim.x / TT) - 1) / (blockDim.x / TT);
    // hooks that read input fields per output sample (escape repair / verify) get the tile's rows
    // of those fields prefetched into shared memory by bulk copies issued at the start of the
    // tile, so the loads land while the rows are transformed (hook_prefetch)
    constexpr bool kPf = hook_prefetch<Hook>();
    const int R = blockDim.x / TT;
    const long long n2r = 2LL * M;  // reals per row
    unsigned char* pf_base = smem_raw + static_cast<size_t>(row_smem_elems<M, E>()) * R * sizeof(cplx<T>);
    uint64_t* pf_bar = nullptr;
    size_t pf_bytes_row = 0;
    if constexpr (kPf) {
        pf_bytes_row = static_cast<size_t>(n2r) * hook.prefetch_scalar_bytes();
        pf_bar = reinterpret_cast<uint64_t*>(pf_base + 2 * pf_bytes_row * R);
        if (threadIdx.x == 0) {
            mbar_init(pf_bar, 1);
            fence_mbar_init();
        }
    }
    unsigned pf_phase = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        // (a CTA barrier only where the tile is shared: prefetch buffers, per-frame skips)
        if constexpr (hook_prefetch<Hook>() || hook_tiled<Hook>()) __syncthreads();
        else __syncwarp();
        if constexpr (hook_tiled<Hook>()) {
            const long long u = tile * (blockDim.x / TT);
            if (hook.tile_skip(u)) continue;
            hook.tile_begin(u);
        }
        const long long row0 = tile * R;
        if constexpr (kPf) {
            if (threadIdx.x == 0) {
                const long long nr = nrows - row0 < R ? nrows - row0 : R;
                const unsigned bytes = static_cast<unsigned>(pf_bytes_row * nr);
                fence_proxy_async_smem();
                mbar_arrive_expect_tx(pf_bar, 2 * bytes);
                bulk_load(pf_base, hook.prefetch_src(0, row0 * out_stride), bytes, pf_bar);
                bulk_load(pf_base + pf_bytes_row * R, hook.prefetch_src(1, row0 * out_stride), bytes,
                          pf_bar);
            }
        }
        const long long row = row0 + rb;
        const bool valid = row < nrows;
        cplx<T>* s = reinterpret_cast<cplx<T>*>(smem_raw) + rb * row_smem_elems<M, E>();
        cplx<T> v[E], mid;
        load_pairs<T, M, E>(in + (valid ? row : 0) * in_stride, t, valid, v, mid);
        merge_pairs<T, M, E>(v, mid, t, twp);
        pairs_to_natural<T, M, E>(v, mid, t);
        stockham<T, M, E, 1, +1>(v, t, tw, XchRowW<T, E>{s});
        if constexpr (kPf) {
            mbar_wait(pf_bar, pf_phase);
            pf_phase ^= 1u;
            hook.use_prefetch(pf_base, pf_base + pf_bytes_row * R, row0 * out_stride);
        }
        if (valid) {
            cplx<T>* dst = reinterpret_cast<cplx<T>*>(out + row * out_stride);
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int j = t + TT * m;
                T x0 = v[m].x * scale, x1 = v[m].y * scale;
                hook.post_real(x0, x1, row * out_stride + 2 * j);
                dst[j] = mkc<T>(x0, x1);
            }
        }
        if constexpr (hook_tiled<Hook>()) hook.tile_end();
    }
    hook.finish();
}

template <class T, int M, int E, class Hook>
__global__ void __launch_bounds__(max_threads<T, E>(), 512 / max_threads<T, E>())
    k_row_c2r_r2c_sh(cplx<T>* data, long long stride, long long nrows, long long real_stride,
                     const cplx<T>* __restrict__ tw, const cplx<T>* __restrict__ twp, T scale,
                     const int* gate, Hook hook, cplx<T>* out) {
    if (gated(gate)) return;
    hook_begin(hook);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int TT = M / E;
    const int t = threadIdx.x % TT;
    const int rb = threadIdx.x / TT;
    const long long ntiles = (nrows + (blockDim.x / TT) - 1) / (blockDim.x / TT);
    HookNone none;
    // input fields of the hook prefetched per tile by bulk copies (as k_row_c2r_sh)
    constexpr bool kPf = hook_prefetch<Hook>();
    const int R = blockDim.x / TT;
    unsigned char* pf_base = smem_raw + static_cast<size_t>(row_smem_elems<M, E>()) * R * sizeof(cplx<T>);
    uint64_t* pf_bar = nullptr;
    size_t pf_bytes_row = 0;
    if constexpr (kPf) {
        pf_bytes_row = static_cast<size_t>(2LL * M) * hook.prefetch_scalar_bytes();
        pf_bar = reinterpret_cast<uint64_t*>(pf_base + 2 * pf_bytes_row * R);
        if (threadIdx.x == 0) {
            mbar_init(pf_bar, 1);
            fence_mbar_init();
        }
    }
    unsigned pf_phase = 0;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        // (a CTA barrier only where the tile is shared: prefetch buffers, per-frame skips)
        if constexpr (hook_prefetch<Hook>() || hook_tiled<Hook>()) __syncthreads();
        else __syncwarp();
        if constexpr (hook_tiled<Hook>()) {
            const long long u = tile * (blockDim.x / TT);
            if (hook.tile_skip(u)) continue;
            hook.tile_begin(u);
        }
        if constexpr (kPf) {
            const long long row0 = tile * R;
            if (threadIdx.x == 0) {
                const long long nr = nrows - row0 < R ? nrows - row0 : R;
                const unsigned bytes = static_cast<unsigned>(pf_bytes_row * nr);
                fence_proxy_async_smem();
                mbar_arrive_expect_tx(pf_bar, 2 * bytes);
                bulk_load(pf_base, hook.prefetch_src(0, row0 * real_stride), bytes, pf_bar);
                bulk_load(pf_base + pf_bytes_row * R, hook.prefetch_src(1, row0 * real_stride),
                          bytes, pf_bar);
            }
        }
        const long long row = tile * (blockDim.x / TT) + rb;
        const bool valid = row < nrows;
        cplx<T>* s = reinterpret_cast<cplx<T>*>(smem_raw) + rb * row_smem_elems<M, E>();
        const XchRowW<T, E> x{s};
        cplx<T>* rowp = data + (valid ? row : 0) * stride;
        cplx<T> v[E], mid;
        load_pairs<T, M, E>(rowp, t, valid, v, mid);
        merge_pairs<T, M, E>(v, mid, t, twp);
        pairs_to_natural<T, M, E>(v, mid, t);
        stockham<T, M, E, 1, +1>(v, t, tw, x);
        if constexpr (kPf) {
            mbar_wait(pf_bar, pf_phase);
            pf_phase ^= 1u;
            hook.use_prefetch(pf_base, pf_base + pf_bytes_row * R, tile * R * real_stride);
        }
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int j = t + TT * m;
            T x0 = v[m].x * scale, x1 = v[m].y * scale;
            if (valid) hook.post_real(x0, x1, row * real_stride + 2 * j);
            v[m] = mkc<T>(x0, x1);
        }
        if constexpr (requires { hook.c2r_only; })
            if (hook.c2r_only) continue;  // (CTA-uniform)
        // fresh twiddle pointers for the forward half: otherwise the compiler keeps the inverse
        // half's stage twiddles and split factors (same indices) live across both transforms
        // (CSE: 816 B of spills at M = 512, E = 16)
        const cplx<T>*tw2, *twp2;
        asm volatile("mov.b64 %0, %1;" : "=l"(tw2) : "l"(tw));
        asm volatile("mov.b64 %0, %1;" : "=l"(twp2) : "l"(twp));
        stockham<T, M, E, 1, -1>(v, t, tw2, x);
        mid = natural_to_pairs<T, M, E>(v, t);
        split_store<T, M, E>(v, mid, t, valid, out ? out + (valid ? row : 0) * stride : rowp,
                             row * stride, twp2, none);
        if constexpr (hook_tiled<Hook>()) hook.tile_end();
    }
    hook.finish();
}

template <class T, int M, int E>
constexpr size_t row_smem_bytes(int rows) {
    return static_cast<size_t>(row_smem_elems<M, E>()) * rows * sizeof(cplx<T>);
}

// ---- direct DFT passes for non-power-of-two or tiny extents (test shapes) ----------------------
// O(L) per output with an exact (n*k mod L) twiddle index into a per-L FP64-derived table.

template <class T>
__global__ void k_col_direct(const cplx<T>* __restrict__ src, cplx<T>* __restrict__ dst, int L,
                             long long row_stride, long long plane_stride, int ncols, int B,
                             const cplx<T>* __restrict__ wl, int dir, const int* gate) {
    if (gated(gate)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* s = reinterpret_cast<cplx<T>*>(smem_raw);
    const long long base = static_cast<long long>(blockIdx.y) * plane_stride + blockIdx.x * B;
    for (int e = threadIdx.x; e < L * B; e += blockDim.x) {
        const int i = e / B, b = e % B;
        s[e] = (blockIdx.x * B + b < ncols) ? src[base + i * row_stride + b] : mkc<T>(T(0), T(0));
    }
    __syncthreads();
    for (int e = threadIdx.x; e < L * B; e += blockDim.x) {
        const int k = e / B, b = e % B;
        if (blockIdx.x * B + b >= ncols) continue;
        T ax = 0, ay = 0;
        long long q = 0;
        for (int n = 0; n < L; ++n) {
            const cplx<T> w = wl[q];
            const cplx<T> xv = s[n * B + b];
            const cplx<T> p = dir < 0 ? cmul(xv, w) : cmulc(xv, w);
            ax += p.x;
            ay += p.y;
            q += k;
            if (q >= L) q -= L;
        }
        dst[base + static_cast<long long>(k) * row_stride + b] = mkc<T>(ax, ay);
    }
}

template <class T>
__global__ void k_row_r2c_direct(const T* __restrict__ in, long long in_stride,
                                 cplx<T>* __restrict__ out, long long out_stride, int n2,
                                 const cplx<T>* __restrict__ wl, const int* gate) {
    if (gated(gate)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* s = reinterpret_cast<T*>(smem_raw);
    const long long row = blockIdx.x;
    for (int n = threadIdx.x; n < n2; n += blockDim.x) s[n] = in[row * in_stride + n];
    __syncthreads();
    for (int k = threadIdx.x; k <= n2 / 2; k += blockDim.x) {
        T ax = 0, ay = 0;
        long long q = 0;
        for (int n = 0; n < n2; ++n) {
            const cplx<T> w = wl[q];
            ax += s[n] * w.x;
            ay += s[n] * w.y;
            q += k;
            if (q >= n2) q -= n2;
        }
        out[row * out_stride + k] = mkc<T>(ax, ay);
    }
}

template <class T>
__global__ void k_row_c2r_direct(const cplx<T>* __restrict__ in, long long in_stride,
                                 T* __restrict__ out, long long out_stride, int n2,
                                 const cplx<T>* __restrict__ wl, T scale, const int* gate) {
    if (gated(gate)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cplx<T>* s = reinterpret_cast<cplx<T>*>(smem_raw);
    const long long row = blockIdx.x;
    const int h = n2 / 2 + 1;
    for (int k = threadIdx.x; k < h; k += blockDim.x) s[k] = in[row * in_stride + k];
    __syncthreads();
    const int kmax = (n2 - 1) / 2; // k with a distinct mirror partner
    for (int n = threadIdx.x; n < n2; n += blockDim.x) {
        T acc = s[0].x;
        long long q = n;
        for (int k = 1; k <= kmax; ++k) {
            const cplx<T> w = wl[q];  // exp(-2 pi i n k / n2)
            const cplx<T> p = cmulc(s[k], w);
            acc += T(2) * p.x;
            q += n;
            if (q >= n2) q -= n2;
        }
        if ((n2 & 1) == 0) acc += (n & 1) ? -s[n2 / 2].x : s[n2 / 2].x;
        out[row * out_stride + n] = acc * scale;
    }
}

} // namespace ffcz_gpu
