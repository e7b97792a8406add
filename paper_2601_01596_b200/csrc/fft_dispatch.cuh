// Launch-time dispatch from runtime extents to the templated pass kernels.  Included by the
// per-precision instantiation units (fft_f32.cu, fft_f64.cu).
#pragma once

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "fft_mixed.cuh"
#include "fft_plan.cuh"
#include "fft_large.cuh"

namespace ffcz_gpu {

namespace detail {

inline int pow2_floor(long long v) {
    int p = 1;
    while ((long long)p * 2 <= v) p *= 2;
    return p;
}
inline int pow2_ceil(long long v) {
    int p = 1;
    while (p < v) p *= 2;
    return p;
}

// Per-CTA complex-element budget of the exchange tile: B*L (columns) or rows*M (rows).
// 4096 FP64 / 8192 FP32 elements = 64 KiB (+1/E padding) -> three CTAs per SM.
// Measured on B200 at 512^3 FP64 (tools/passbench.py, profiles/r01_passbench.md):
//  * row passes: 1024 elements per CTA (4 rows of 256) -> 90% of HBM; bigger CTAs serialise
//    load and compute phases;
//  * column pass along the middle axis (row stride P): 2048 (B = 4 columns, 2 CTAs/SM) -> 70%;
//  * column pass along the first axis (row stride n1*P, >2 MB): 4096 (B = 8: 128-B row
//    segments keep DRAM pages / TLB entries shared by concurrent CTAs) -> 50%; 64-B segments
//    drop it to 43%, 32-B to 26%.
// FFCZ_TILE_BUDGET{64,32}_{ROW,MID,FIRST} override them (tuning runs).
enum class TileRole { kRow = 0, kMid = 1, kFirst = 2 };
template <class T> long long tile_budget(TileRole role) {
    static const long long v[3] = {
        [] {
            const char* e = std::getenv(sizeof(T) == 8 ? "FFCZ_TILE_BUDGET64_ROW" : "FFCZ_TILE_BUDGET32_ROW");
            return e ? std::max(16LL, std::atoll(e)) : (sizeof(T) == 8 ? 1024LL : 2048LL);
        }(),
        [] {
            const char* e = std::getenv(sizeof(T) == 8 ? "FFCZ_TILE_BUDGET64_MID" : "FFCZ_TILE_BUDGET32_MID");
            return e ? std::max(16LL, std::atoll(e)) : (sizeof(T) == 8 ? 2048LL : 4096LL);
        }(),
        [] {
            const char* e = std::getenv(sizeof(T) == 8 ? "FFCZ_TILE_BUDGET64_FIRST" : "FFCZ_TILE_BUDGET32_FIRST");
            return e ? std::max(16LL, std::atoll(e)) : (sizeof(T) == 8 ? 4096LL : 8192LL);
        }()};
    return v[static_cast<int>(role)];
}

// FFCZ_COL_TMA=0 selects the register-direct column pass (A/B runs); default: TMA-staged.
inline bool col_tma_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_COL_TMA");
        return !(e && e[0] == '0');
    }();
    return on;
}

// FFCZ_COL_C2=1 enables the 2-CTA cluster column pass.  Off by default: correct (parity suite)
// but measured slower than the single-CTA passes it replaces — 0.50 of HBM vs 0.67-0.75 at
// 1024^3 and 0.50 vs 0.69 on 2048-point lines (two cluster barriers per tile and no overlap of
// the DSMEM exchange with the next tile's load); kept for the deeper-pipelined version.
inline bool c2_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_COL_C2");
        return e && e[0] == '1';
    }();
    return on;
}

// FFCZ_COL_TMA1: 0 = never use the single-landing column pass, 1 = wherever it fits,
// unset = only where double buffering would fall below 128-B row segments.
inline int tma1_mode() {
    static const int m = [] {
        const char* e = std::getenv("FFCZ_COL_TMA1");
        return e ? (e[0] == '0' ? 0 : 1) : 2;
    }();
    return m;
}

// FFCZ_TMA1_E8=1: plain FP64 single-landing column passes of >= 1024 points at E = 8 / 1024
// threads instead of E = 16 / 512 (A/B)
inline bool tma1_e8() {
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_TMA1_E8");
        return e && e[0] == '1';
    }();
    return on;
}

// FFCZ_TMA1_HALF=1: plain FP64 single-landing column passes of >= 1024 points as two 256-thread
// CTAs per SM on 4-column tiles (A/B)
inline bool tma1_half() {
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_TMA1_HALF");
        return e && e[0] == '1';
    }();
    return on;
}

// raises a kernel's dynamic shared-memory limit once (a driver call per launch otherwise)
template <class K>
void set_smem(K kernel, size_t bytes) {
    if (bytes <= 48 * 1024) return;
    static std::mutex mu;
    static std::map<const void*, size_t> done;
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = done[reinterpret_cast<const void*>(kernel)];
    if (cur >= bytes) return;
    FFCZ_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(bytes)));
    cur = bytes;
}

// Persistent grid: resident-CTA capacity of the device for this kernel configuration.
template <class K>
long long resident_ctas(K kernel, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, size_t>, long long> cache;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), threads, smem);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int dev = 0, sms = 0, nb = 0;
    FFCZ_CUDA_CHECK(cudaGetDevice(&dev));
    FFCZ_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FFCZ_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem));
    return cache[key] = static_cast<long long>(std::max(1, nb)) * sms;
}

template <class K>
unsigned persistent_grid(K kernel, int threads, size_t smem, long long ntiles) {
    return static_cast<unsigned>(std::max<long long>(
        1, std::min<long long>(ntiles, resident_ctas(kernel, threads, smem))));
}

inline unsigned grid1(long long n, int threads) {
    long long b = (n + threads - 1) / threads;
    return static_cast<unsigned>(std::max<long long>(1, std::min<long long>(b, 148LL * 32)));
}

template <class T, int L, class Hook>
void col_radix(int dir, const cplx<T>* src, cplx<T>* dst, long long row_stride,
               long long plane_stride, long long nplanes, int ncols, Twiddles<T>& tw,
               const int* gate, Hook hook, cudaStream_t st) {
    // FP32 passes that carry hooks (the mixed policy's check / clip, FP64 S / F bookkeeping)
    // run at E = 16: at E = 32 the line's 64 registers plus the hooks' FP64 temporaries spill
    constexpr int E = (sizeof(T) == 4 && !std::is_same_v<Hook, HookNone> && L >= 512 &&
                       pick_E<T>(L) > 16)
                          ? 16
                          : pick_E<T>(L);
    constexpr int TT = L / E;
    constexpr int MAXT = max_threads<T, E>();
    const TileRole role = row_stride > plane_stride && nplanes > 1 ? TileRole::kFirst : TileRole::kMid;
    int B = static_cast<int>(std::min<long long>(tile_budget<T>(role) / L, MAXT / TT));
    B = std::min(B, 128);
    B = std::min(B, pow2_ceil(ncols));
    B = std::max(B, (32 + TT - 1) / TT);  // whole warps (full-mask block reductions in hooks)
    const size_t smem = col_smem_bytes<T, L, E>(B);
    const long long ntiles = static_cast<long long>((ncols + B - 1) / B) * nplanes;
    if (col_tma_enabled()) {
        // TMA-staged double-buffered pass: B columns per tile bounded by 1 CTA/SM of smem; a
        // single-lane per-component Delta rides along as a side tile
        const double* side = nullptr;
        if constexpr (hook_delta<Hook>())
            if (hook.fb.re && hook.fb.im == hook.fb.re) side = hook.fb.re;
        int Bt = static_cast<int>(std::min<long long>(MAXT / TT, 128));
        while (Bt > 1 && col_tma_smem_bytes<T, L, E>(Bt, side) > 220 * 1024) Bt /= 2;
        if (const char* e = std::getenv("FFCZ_COL_TMA_B")) Bt = std::max(1, std::atoi(e));
        Bt = std::min(Bt, pow2_ceil(ncols));
        if constexpr (L >= 1024 && sizeof(T) == 8) {
            // 2-CTA cluster (k_col_c2): each CTA lands half the rows, so tiles reach 256-B (L =
            // 1024) / 128-B (L = 2048) rows (opt-in, see c2_enabled).
            constexpr int E2 = 16, TT2 = (L / 2) / E2, NT2 = 512;
            int B2 = std::min(NT2 / TT2, 128);
            while (B2 > 1 && col_c2_smem_bytes<T, L, E2>(B2) > 220 * 1024) B2 /= 2;
            B2 = std::min(B2, pow2_ceil(ncols));
            CUtensorMap map2;
            if (!side && c2_enabled() && TT2 * B2 >= 32 && B2 * sizeof(cplx<T>) >= 128 &&
                encode_col_map(&map2, src, sizeof(T), ncols, L, row_stride, nplanes, plane_stride,
                               B2, (L / 2) < 256 ? (L / 2) : 256, true)) {
                auto kt = dir < 0 ? k_col_c2<T, L, E2, -1, Hook, NT2> : k_col_c2<T, L, E2, +1, Hook, NT2>;
                const size_t sm2 = col_c2_smem_bytes<T, L, E2>(B2);
                set_smem(kt, sm2);
                const long long nt = static_cast<long long>((ncols + B2 - 1) / B2) * nplanes;
                cudaLaunchConfig_t cfg = {};
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = 2;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.blockDim = dim3(TT2 * B2);
                cfg.dynamicSmemBytes = sm2;
                cfg.stream = st;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                static std::mutex mu;
                static std::map<std::pair<const void*, size_t>, int> clusters;
                int ncl = 0;
                {
                    std::lock_guard<std::mutex> lk(mu);
                    auto key = std::make_pair(reinterpret_cast<const void*>(kt), sm2 * 1024 + B2);
                    auto it = clusters.find(key);
                    if (it == clusters.end()) {
                        cfg.gridDim = dim3(2 * 148);
                        FFCZ_CUDA_CHECK(cudaOccupancyMaxActiveClusters(&ncl, kt, &cfg));
                        clusters[key] = ncl;
                    } else {
                        ncl = it->second;
                    }
                }
                const long long pairs = std::max<long long>(1, std::min<long long>(nt, ncl));
                cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
                FFCZ_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kt, map2, dst, row_stride, plane_stride,
                                                   ncols, B2, nt, tw.stage_table(L / 2, E2),
                                                   tw.post_table(L / 2), gate, hook));
                return;
            }
        }
        if constexpr (L >= 512) {
            // single landing buffer + scalar exchange (k_col_tma1) where it gives wider row
            // segments than double buffering: always when double buffering falls below 128 B,
            // and on the outer axis (row stride > plane stride) whenever it is wider — outer-axis
            // passes measured 0.38-0.48 of HBM at 64-B rows, 0.53-0.69 at 128 B, 0.87 at 256 B.
            // FP64 L = 512 runs it at E = 16 (same stage count as E = 8, half the threads per
            // column) so a 16-column (256-B) tile fits 512 threads.  FFCZ_COL_TMA1=0 disables,
            // =1 forces it where it fits.
            // FP32 runs it at E = 16 with 1024 threads (E = 32 at 512 threads spills: 0.70 ->
            // 0.47 of HBM on the 1024^3 middle axis), so its outer-axis tiles reach 128-B rows
            // (16 float2) like FP64's 8 double2: 1024^3 outer axis 0.41 (double-buffered, 64-B
            // rows) -> 0.45 of HBM (E = 32 at 512 threads: 0.47; profiles/r02_passbench_f32.jsonl)
            constexpr int E1 = sizeof(T) == 4 ? 16 : ((L == 512) ? 16 : E);
            constexpr int TT1 = L / E1;
            constexpr int NT1 = sizeof(T) == 4 ? 1024 : 512;
            const int mode = tma1_mode();
            int B1 = std::min(NT1 / TT1, 128);
            while (B1 > 1 && col_tma1_smem_bytes<T, L, E1>(B1) > 220 * 1024) B1 /= 2;
            B1 = std::min(B1, pow2_ceil(ncols));
            // (FP32 at L = 512 keeps double buffering: 128-B rows already, 0.80 of HBM at 512^3
            // vs 0.37 in this variant)
            const bool outer = role == TileRole::kFirst && (sizeof(T) == 8 || L >= 1024);
            // (FP32: outer axis only; its middle axis keeps double buffering)
            const bool want = !side && mode != 0 && TT1 * B1 >= 32 &&
                              (mode == 1 || (B1 > Bt && (sizeof(T) == 8
                                                              ? (Bt * sizeof(cplx<T>) < 128 || outer)
                                                              : outer)));
            if constexpr (sizeof(T) == 8 && L >= 1024 && std::is_same_v<Hook, HookNone>) {
                // plain FP64 passes as two 256-thread CTAs per SM on half-width tiles
                // (FFCZ_TMA1_HALF, A/B): consecutive CTAs take adjacent 64-B column halves, two
                // independent tile pipelines per SM instead of one
                constexpr int EH = 16, TTH = L / EH, NTH = 256;
                const int BH = std::min(NTH / TTH, pow2_ceil(ncols));
                CUtensorMap maph;
                if (want && tma1_half() && BH >= 1 && TTH * BH >= 32 &&
                    col_tma1_smem_bytes<T, L, EH>(BH) <= 110 * 1024 &&
                    encode_col_map(&maph, src, sizeof(T), ncols, L, row_stride, nplanes,
                                   plane_stride, BH, L < 256 ? L : 256, true)) {
                    auto kt = dir < 0 ? k_col_tma1<T, L, EH, -1, Hook, NTH>
                                      : k_col_tma1<T, L, EH, +1, Hook, NTH>;
                    const size_t smh = col_tma1_smem_bytes<T, L, EH>(BH);
                    set_smem(kt, smh);
                    const long long nt = static_cast<long long>((ncols + BH - 1) / BH) * nplanes;
                    const unsigned grid = persistent_grid(kt, TTH * BH, smh, nt);
                    kt<<<grid, TTH * BH, smh, st>>>(maph, dst, row_stride, plane_stride, ncols, BH,
                                                    nt, tw.stage_table(L, EH), gate, hook);
                    FFCZ_LAUNCH_CHECK();
                    return;
                }
            }
            if constexpr (sizeof(T) == 8 && L >= 1024 && std::is_same_v<Hook, HookNone>) {
                // plain FP64 passes at E = 8 with 1024 threads (FFCZ_TMA1_E8): 64 registers, 32
                // warps per SM instead of 16 (the E = 16 pass issues on 28 % of cycles: latency-
                // bound, profiles/r02_ncu_full_outer_tma1_1024.csv); one more exchange per line
                constexpr int E8 = 8, TT8 = L / E8, NT8 = 1024;
                int B8 = std::min(NT8 / TT8, 128);
                while (B8 > 1 && col_tma1_smem_bytes<T, L, E8>(B8) > 220 * 1024) B8 /= 2;
                B8 = std::min(B8, pow2_ceil(ncols));
                CUtensorMap map8;
                if (want && tma1_e8() && TT8 * B8 >= 32 && B8 >= B1 &&
                    encode_col_map(&map8, src, sizeof(T), ncols, L, row_stride, nplanes,
                                   plane_stride, B8, L < 256 ? L : 256, true)) {
                    auto kt = dir < 0 ? k_col_tma1<T, L, E8, -1, Hook, NT8>
                                      : k_col_tma1<T, L, E8, +1, Hook, NT8>;
                    const size_t sm8 = col_tma1_smem_bytes<T, L, E8>(B8);
                    set_smem(kt, sm8);
                    const long long nt = static_cast<long long>((ncols + B8 - 1) / B8) * nplanes;
                    const unsigned grid = persistent_grid(kt, TT8 * B8, sm8, nt);
                    kt<<<grid, TT8 * B8, sm8, st>>>(map8, dst, row_stride, plane_stride, ncols, B8,
                                                    nt, tw.stage_table(L, E8), gate, hook);
                    FFCZ_LAUNCH_CHECK();
                    return;
                }
            }
            CUtensorMap map1;
            if (want && encode_col_map(&map1, src, sizeof(T), ncols, L, row_stride, nplanes,
                                       plane_stride, B1, L < 256 ? L : 256, true)) {
                auto kt = dir < 0 ? k_col_tma1<T, L, E1, -1, Hook, NT1>
                                  : k_col_tma1<T, L, E1, +1, Hook, NT1>;
                const size_t sm1 = col_tma1_smem_bytes<T, L, E1>(B1);
                set_smem(kt, sm1);
                const long long nt = static_cast<long long>((ncols + B1 - 1) / B1) * nplanes;
                const unsigned grid = persistent_grid(kt, TT1 * B1, sm1, nt);
                kt<<<grid, TT1 * B1, sm1, st>>>(map1, dst, row_stride, plane_stride, ncols, B1, nt,
                                                tw.stage_table(L, E1), gate, hook);
                FFCZ_LAUNCH_CHECK();
                return;
            }
        }
        const size_t tsmem = col_tma_smem_bytes<T, L, E>(Bt, side);
        CUtensorMap map, side_map;
        bool ok = TT * Bt >= 32 && Bt * sizeof(cplx<T>) >= 32 && tsmem <= 227 * 1024 &&
                  encode_col_map(&map, src, sizeof(T), ncols, L, row_stride, nplanes,
                                 plane_stride, Bt, L < 256 ? L : 256, true);
        if (ok && side)
            ok = encode_col_map(&side_map, side, 8, ncols, L, row_stride, nplanes, plane_stride,
                                Bt, L < 256 ? L : 256, false);
        if (ok) {
            if (!side) side_map = map;
            auto kt = dir < 0 ? k_col_tma<T, L, E, -1, Hook> : k_col_tma<T, L, E, +1, Hook>;
            set_smem(kt, tsmem);
            const long long nt = static_cast<long long>((ncols + Bt - 1) / Bt) * nplanes;
            const unsigned grid = persistent_grid(kt, TT * Bt, tsmem, nt);
            kt<<<grid, TT * Bt, tsmem, st>>>(map, side_map, side != nullptr, dst, row_stride,
                                             plane_stride, ncols, Bt, nt, tw.stage_table(L, E),
                                             gate, hook);
            FFCZ_LAUNCH_CHECK();
            return;
        }
    }
    auto k = dir < 0 ? k_col<T, L, E, -1, Hook> : k_col<T, L, E, +1, Hook>;
    set_smem(k, smem);
    const unsigned grid = persistent_grid(k, TT * B, smem, ntiles);
    k<<<grid, TT * B, smem, st>>>(src, dst, row_stride, plane_stride, ncols, B, ntiles,
                                   tw.stage_table(L, E), gate, hook);
    FFCZ_LAUNCH_CHECK();
}

template <class T, int M> struct RowCfg {
    // FP64 M = 512 (1024-sample rows) ties at three stages for E = 8 and E = 16; E = 16 gives 32
    // threads per row, i.e. the warp-shuffle paired split / merge (k_row_*_sh) instead of the
    // shared-memory round trip (FFCZ_ROW512_E8 at build time restores E = 8)
#ifdef FFCZ_ROW512_E8
    static constexpr int E = pick_E<T>(M);
#else
    static constexpr int E = (sizeof(T) == 8 && M == 512) ? 16 : pick_E<T>(M);
#endif
    static constexpr int TT = M / E;
    static constexpr int MAXT = max_threads<T, E>();
};

// E of a row pass carrying `Hook`: FP32 C2R passes with real-output hooks (the mixed policy's
// s-clip: FP64 S bookkeeping on FP32 values) run at E = 16 — at E = 32 the 64 registers of line
// data plus the hook's FP64 temporaries spill (3.2 ms vs 1.4 ms for the plain pass at 1024^3)
template <class T, int M, class Hook>
constexpr int row_E() {
    if constexpr (sizeof(T) == 4 && !std::is_same_v<Hook, RealHookNone> &&
                  !std::is_same_v<Hook, HookNone> && RowCfg<T, M>::E > 16 && M / 16 <= 32)
        return 16;
    else
        return RowCfg<T, M>::E;
}

template <class T, int M, int E = RowCfg<T, M>::E>
int rows_per_cta(long long nrows) {
    constexpr int TT = M / E;
    long long r = std::min<long long>(tile_budget<T>(TileRole::kRow) / M, max_threads<T, E>() / TT);
    r = std::min<long long>(r, pow2_ceil(nrows));
    // whole warps only: the paired split/merge and the block reductions use full-mask shuffles
    r = std::max<long long>(r, (32 + TT - 1) / TT);
    return static_cast<int>(std::max<long long>(1, r));
}

template <class T, int M, class Hook = HookNone>
void row_r2c_radix(const T* in, long long in_stride, cplx<T>* out, long long out_stride,
                   long long nrows, Twiddles<T>& tw, const int* gate, cudaStream_t st,
                   Hook hook = Hook{}) {
    constexpr int E = RowCfg<T, M>::E, TT = RowCfg<T, M>::TT;
    const int R = rows_per_cta<T, M>(nrows);
    const size_t smem = row_smem_bytes<T, M, E>(R);
    auto k = TT <= 32 ? k_row_r2c_sh<T, M, E, Hook> : k_row_r2c<T, M, E, Hook>;
    set_smem(k, smem);
    k<<<persistent_grid(k, TT * R, smem, (nrows + R - 1) / R), TT * R, smem, st>>>(
        in, in_stride, out, out_stride, nrows, tw.stage_table(M, E), tw.post_table(M), gate,
        hook);
    FFCZ_LAUNCH_CHECK();
}

template <class T, int M, class Hook = RealHookNone>
void row_c2r_radix(const cplx<T>* in, long long in_stride, T* out, long long out_stride,
                   long long nrows, T scale, Twiddles<T>& tw, const int* gate, cudaStream_t st,
                   Hook hook = Hook{}) {
    constexpr int E = row_E<T, M, Hook>(), TT = M / E;
    const int R = rows_per_cta<T, M, E>(nrows);
    size_t smem = row_smem_bytes<T, M, E>(R);
    if constexpr (hook_prefetch<Hook>())  // two input fields' rows + the mbarrier (k_row_c2r_sh)
        if (TT <= 32) smem += 2 * static_cast<size_t>(2 * M) * R * Hook::prefetch_scalar_bytes() + 16;
    auto k = TT <= 32 ? k_row_c2r_sh<T, M, E, Hook> : k_row_c2r<T, M, E, Hook>;
    set_smem(k, smem);
    k<<<persistent_grid(k, TT * R, smem, (nrows + R - 1) / R), TT * R, smem, st>>>(
        in, in_stride, out, out_stride, nrows, tw.stage_table(M, E), tw.post_table(M), scale,
        gate, hook);
    FFCZ_LAUNCH_CHECK();
}

template <class T, int M, class Hook>
void row_fused_radix(cplx<T>* data, long long stride, long long nrows, long long real_stride,
                     T scale, Twiddles<T>& tw, const int* gate, Hook hook, cudaStream_t st,
                     cplx<T>* out) {
    constexpr int E = RowCfg<T, M>::E, TT = RowCfg<T, M>::TT;
    const int R = rows_per_cta<T, M>(nrows);
    size_t smem = row_smem_bytes<T, M, E>(R);
    if constexpr (hook_prefetch<Hook>())  // two input fields' rows + the mbarrier
        if (TT <= 32) smem += 2 * static_cast<size_t>(2 * M) * R * Hook::prefetch_scalar_bytes() + 16;
    auto k = TT <= 32 ? k_row_c2r_r2c_sh<T, M, E, Hook> : k_row_c2r_r2c<T, M, E, Hook>;
    set_smem(k, smem);
    k<<<persistent_grid(k, TT * R, smem, (nrows + R - 1) / R), TT * R, smem, st>>>(
        data, stride, nrows, real_stride, tw.stage_table(M, E), tw.post_table(M), scale, gate,
        hook, out);
    FFCZ_LAUNCH_CHECK();
}

// Mixed-radix passes (fft_mixed.cuh) take every extent that is not on the power-of-two path when
// the two ping-pong buffers of one line fit; FFCZ_MIXED=0 keeps the O(L) direct passes (A/B).
inline bool mixed_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_MIXED");
        return !(e && e[0] == '0');
    }();
    return on;
}
constexpr size_t kMixedSmemMax = 220 * 1024;  // (the padded 1000-point tiles keep 4 columns)
inline bool mixed_pipe_enabled() {  // FFCZ_MIXED_PIPE=0: the one-tile-per-CTA column pass (A/B)
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_MIXED_PIPE");
        return !(e && e[0] == '0');
    }();
    return on;
}
inline size_t mixed_smem_target() {  // FFCZ_MIXED_SMEM=<KB> for tile-size sweeps
    static const size_t t = [] {
        const char* e = std::getenv("FFCZ_MIXED_SMEM");
        return e ? static_cast<size_t>(std::atoi(e)) * 1024 : size_t(64 * 1024);
    }();
    return t;
}
// lines per CTA: as many as fit the target (at least one line within the maximum), at most 16
template <class T>
inline int mixed_lines(long long L, long long nlines, bool pad = true) {
    const size_t per = 2 * sizeof(cplx<T>) *
                       static_cast<size_t>(pad ? mixed::padded(static_cast<int>(L)) : L);
    if (per > kMixedSmemMax) return 0;
    long long b = std::max<long long>(1, static_cast<long long>(mixed_smem_target() / per));
    b = std::min<long long>({b, 16, std::max<long long>(1, nlines)});
    return static_cast<int>(b);
}

template <class T, int L, class Hook, int E1, int NT1>
void col_rt_radix_e(const cplx<T>* src, cplx<T>* dst, long long row_stride,
                    long long plane_stride, long long nplanes, int ncols, Twiddles<T>& tw,
                    const int* gate, Hook hook, cudaStream_t st) {
    // k_col_tma1's tile: B columns of 128-B+ rows within one SM's smem, plus the marks' landing
    // tile (>= 16 columns: TMA boxes are 16-B multiples)
    constexpr int TT1 = L / E1;
    int B1 = std::min(NT1 / TT1, 128);
    B1 = std::min(B1, pow2_ceil(ncols));
    B1 = std::max(B1, (32 + TT1 - 1) / TT1);  // whole warps (the hook's block reduction)
    auto mbw = [](int b) { return std::max(b, 16); };
    while (B1 > 1 && TT1 * (B1 / 2) >= 32 && col_rt_smem_bytes<T, L, E1>(B1, mbw(B1)) > 220 * 1024)
        B1 /= 2;
    const int MB = mbw(B1);
    CUtensorMap map1, mmap;
    if (col_rt_smem_bytes<T, L, E1>(B1, MB) > 220 * 1024 ||
        !encode_col_map(&map1, src, sizeof(T), ncols, L, row_stride, nplanes, plane_stride, B1,
                        L < 256 ? L : 256, true) ||
        !encode_col_map(&mmap, hook.moved, 1, ncols, L, row_stride, nplanes, plane_stride, MB,
                        L < 256 ? L : 256, false))
        throw Error(kUnsupported, "round-trip column pass: no TMA tile for this axis");
    auto kt = k_col_tma1_rt<T, L, E1, Hook, NT1>;
    const size_t sm1 = col_rt_smem_bytes<T, L, E1>(B1, MB);
    set_smem(kt, sm1);
    const long long nt = static_cast<long long>((ncols + B1 - 1) / B1) * nplanes;
    const unsigned grid = persistent_grid(kt, TT1 * B1, sm1, nt);
    kt<<<grid, TT1 * B1, sm1, st>>>(map1, mmap, dst, row_stride, plane_stride, ncols, B1, MB, nt,
                                    tw.stage_table(L, E1), gate, hook);
    FFCZ_LAUNCH_CHECK();
}

// FFCZ_RT_E8=1: the round trip of >= 1024-point lines at E = 8 / 1024 threads (64 registers,
// 32 warps per SM) instead of E = 16 / 512 (A/B)
inline bool rt_e8() {
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_RT_E8");
        return e && e[0] == '1';
    }();
    return on;
}

template <class T, int L, class Hook>
void col_rt_radix(const cplx<T>* src, cplx<T>* dst, long long row_stride, long long plane_stride,
                  long long nplanes, int ncols, Twiddles<T>& tw, const int* gate, Hook hook,
                  cudaStream_t st) {
    if constexpr (L >= 1024) {
        if (rt_e8()) {
            col_rt_radix_e<T, L, Hook, 8, 1024>(src, dst, row_stride, plane_stride, nplanes, ncols,
                                                tw, gate, hook, st);
            return;
        }
    }
    col_rt_radix_e<T, L, Hook, 16, 512>(src, dst, row_stride, plane_stride, nplanes, ncols, tw,
                                        gate, hook, st);
}

template <class T, int L>
void col_frebuild_radix(const cplx<T>* src, const cplx<T>* delta, cplx<T>* F,
                        const unsigned char* moved, long long row_stride, long long plane_stride,
                        long long nplanes, int ncols, Twiddles<T>& tw, cudaStream_t st) {
    constexpr int E1 = 16, TT1 = L / E1, NT1 = 512;
    int B1 = std::min(NT1 / TT1, 128);
    B1 = std::min(B1, pow2_ceil(ncols));
    B1 = std::max(B1, (32 + TT1 - 1) / TT1);
    auto mbw = [](int b) { return std::max(b, 16); };
    while (B1 > 1 && TT1 * (B1 / 2) >= 32 && col_rt_smem_bytes<T, L, E1>(B1, mbw(B1)) > 220 * 1024)
        B1 /= 2;
    const int MB = mbw(B1);
    const int LB = L < 256 ? L : 256;
    CUtensorMap map1, mmap, dmap;
    if (col_rt_smem_bytes<T, L, E1>(B1, MB) > 220 * 1024 ||
        !encode_col_map(&map1, src, sizeof(T), ncols, L, row_stride, nplanes, plane_stride, B1, LB,
                        true) ||
        !encode_col_map(&mmap, moved, 1, ncols, L, row_stride, nplanes, plane_stride, MB, LB,
                        false) ||
        !encode_col_map(&dmap, delta, sizeof(T), ncols, L, row_stride, nplanes, plane_stride, B1,
                        LB, true))
        throw Error(kUnsupported, "F rebuild pass: no TMA tile for this axis");
    auto kt = k_col_tma1_frebuild<T, L, E1, NT1>;
    const size_t sm1 = col_rt_smem_bytes<T, L, E1>(B1, MB);
    set_smem(kt, sm1);
    const long long nt = static_cast<long long>((ncols + B1 - 1) / B1) * nplanes;
    const unsigned grid = persistent_grid(kt, TT1 * B1, sm1, nt);
    kt<<<grid, TT1 * B1, sm1, st>>>(map1, mmap, dmap, F, row_stride, plane_stride, ncols, B1, MB,
                                    nt, tw.stage_table(L, E1));
    FFCZ_LAUNCH_CHECK();
}

} // namespace detail

// Round-trip column pass (k_col_tma1_rt): power-of-two lines of 16..4096 points.
template <class T, class Hook>
void launch_col_rt(long long L, const cplx<T>* src, cplx<T>* dst, long long row_stride,
                   long long plane_stride, long long nplanes, int ncols, Twiddles<T>& tw,
                   const int* gate, Hook hook, cudaStream_t st) {
    switch (L) {
#define X(n)                                                                                   \
    case n:                                                                                    \
        detail::col_rt_radix<T, n, Hook>(src, dst, row_stride, plane_stride, nplanes, ncols,   \
                                         tw, gate, hook, st);                                  \
        return;
        X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096)
#undef X
    default:
        throw Error(kUnsupported, "round-trip column pass needs a power-of-two extent in [16, 4096]");
    }
}

// The gate's F rebuild on the completing axis (k_col_tma1_frebuild): lines of 16..4096 points.
template <class T>
void launch_col_frebuild(long long L, const cplx<T>* src, const cplx<T>* delta, cplx<T>* F,
                         const unsigned char* moved, long long row_stride, long long plane_stride,
                         long long nplanes, int ncols, Twiddles<T>& tw, cudaStream_t st) {
    switch (L) {
#define X(n)                                                                                    \
    case n:                                                                                     \
        detail::col_frebuild_radix<T, n>(src, delta, F, moved, row_stride, plane_stride, nplanes, \
                                         ncols, tw, st);                                        \
        return;
        X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096)
#undef X
    default:
        throw Error(kUnsupported, "F rebuild pass needs a power-of-two extent in [16, 4096]");
    }
}

#define FFCZ_POW2_CASES(X) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096)

template <class T, class Hook>
void launch_col(long long L, int dir, const cplx<T>* src, cplx<T>* dst, long long row_stride,
                long long plane_stride, long long nplanes, int ncols, Twiddles<T>& tw,
                const int* gate, Hook hook, cudaStream_t st) {
    if (radix_col_ok(L)) {
        switch (L) {
#define X(n)                                                                                   \
    case n:                                                                                    \
        detail::col_radix<T, n, Hook>(dir, src, dst, row_stride, plane_stride, nplanes, ncols, \
                                      tw, gate, hook, st);                                     \
        return;
            FFCZ_POW2_CASES(X)
#undef X
        }
    }
    if constexpr (!std::is_same_v<Hook, HookNone>) {
        throw Error(kUnsupported, "fused column pass needs a power-of-two extent in [16, 4096]");
    } else {
        if (detail::mixed_pipe_enabled() && detail::mixed_enabled()) {
            // 3 rotating tile buffers, B columns each (at most 16), within ~96 KB per CTA
            const size_t per =
                3 * sizeof(cplx<T>) * static_cast<size_t>(mixed::padded(static_cast<int>(L)));
            if (per <= detail::kMixedSmemMax) {
                static const long long kb = [] {
                    const char* e = std::getenv("FFCZ_MIXED_PIPE_KB");
                    return e ? std::atoll(e) : 96LL;
                }();
                long long Bm = std::max<long long>(1, static_cast<long long>(kb * 1024 / per));
                // at least 4 columns (64-B runs for FP64) while they fit: L = 1000 FP64 measured
                // 0.29 / 0.20 of HBM at 2 columns, 0.31 / 0.28 at 4 (r01_passbench_mixed_1000)
                Bm = std::max<long long>(
                    Bm, std::min<long long>(4, static_cast<long long>(detail::kMixedSmemMax / per)));
                Bm = std::min<long long>({Bm, 16, static_cast<long long>(ncols)});
                const size_t smem = per * Bm;
                const long long ntiles = nplanes * ((ncols + Bm - 1) / Bm);
                auto k = k_col_mixed_pipe<T>;
                detail::set_smem(k, smem);
                const unsigned grid = detail::persistent_grid(k, 256, smem, ntiles);
                k<<<grid, 256, smem, st>>>(src, dst, make_mixed_plan(L), row_stride, plane_stride,
                                           ncols, static_cast<int>(Bm), ntiles, tw.table_for(L),
                                           dir, gate);
                FFCZ_LAUNCH_CHECK();
                return;
            }
        }
        if (const int Bm = detail::mixed_enabled() ? detail::mixed_lines<T>(L, ncols) : 0) {
            const size_t smem = 2 * sizeof(cplx<T>) * mixed::padded(static_cast<int>(L)) * Bm;
            detail::set_smem(k_col_mixed<T>, smem);
            dim3 grid((ncols + Bm - 1) / Bm, static_cast<unsigned>(nplanes));
            k_col_mixed<T><<<grid, 256, smem, st>>>(src, dst, make_mixed_plan(L), row_stride,
                                                     plane_stride, ncols, Bm, tw.table_for(L),
                                                     dir, gate);
            FFCZ_LAUNCH_CHECK();
            return;
        }
        // direct O(L) pass: tile L x B columns in smem
        const size_t per_col = sizeof(cplx<T>) * L;
        if (per_col > 96 * 1024) {  // longer than shared memory holds: global-memory passes
            LineAddr a;
            a.compact = false;
            a.row_stride = row_stride;
            a.plane_stride = plane_stride;
            a.ncols = ncols;
            a.nl = static_cast<long long>(ncols) * nplanes;
            large_lines<T>(L, dir, src, a, dst, a, a.nl, tw, gate, st);
            return;
        }
        int B = static_cast<int>(std::max<long long>(1, std::min<long long>(48 * 1024 / per_col, 32)));
        B = std::min(B, detail::pow2_ceil(ncols));
        const size_t smem = per_col * B;
        detail::set_smem(k_col_direct<T>, smem);
        dim3 grid((ncols + B - 1) / B, static_cast<unsigned>(nplanes));
        k_col_direct<T><<<grid, 256, smem, st>>>(src, dst, static_cast<int>(L), row_stride,
                                                  plane_stride, ncols, B, tw.table_for(L), dir,
                                                  gate);
        FFCZ_LAUNCH_CHECK();
    }
}

template <class T>
void launch_row_r2c(long long n2, const T* in, long long in_stride, cplx<T>* out,
                    long long out_stride, long long nrows, Twiddles<T>& tw, const int* gate,
                    cudaStream_t st) {
    if (radix_row_ok(n2)) {
        switch (n2 / 2) {
#define X(n)                                                                                   \
    case n:                                                                                    \
        detail::row_r2c_radix<T, n>(in, in_stride, out, out_stride, nrows, tw, gate, st);      \
        return;
            FFCZ_POW2_CASES(X)
#undef X
        }
    }
    const long long Lm = (n2 % 2 == 0) ? n2 / 2 : n2;  // packed real row: n2/2 points
    if (const int R = detail::mixed_enabled() ? detail::mixed_lines<T>(Lm + 1, nrows, false) : 0) {
        const size_t smem = 2 * sizeof(cplx<T>) * (Lm + 1) * R;
        detail::set_smem(k_row_r2c_mixed<T>, smem);
        k_row_r2c_mixed<T><<<static_cast<unsigned>((nrows + R - 1) / R), 256, smem, st>>>(
            in, in_stride, out, out_stride, nrows, static_cast<int>(n2), R, make_mixed_plan(Lm),
            tw.table_for(n2), gate);
        FFCZ_LAUNCH_CHECK();
        return;
    }
    const size_t smem = sizeof(T) * n2;
    if (smem > 96 * 1024) {  // longer than shared memory holds: global-memory passes
        large_row_r2c<T>(n2, in, in_stride, out, out_stride, nrows, tw, gate, st);
        return;
    }
    detail::set_smem(k_row_r2c_direct<T>, smem);
    k_row_r2c_direct<T><<<static_cast<unsigned>(nrows), 256, smem, st>>>(
        in, in_stride, out, out_stride, static_cast<int>(n2), tw.table_for(n2), gate);
    FFCZ_LAUNCH_CHECK();
}

// eps0 fused into the first R2C (k_row_r2c_eps0_sh); false when the row length has no
// warp-paired FP64 variant (the caller then runs k_eps0 + R2C)
template <class TI>
bool launch_row_r2c_eps0(long long n2, const TI* orig, const TI* dec, double2* out,
                         long long out_stride, long long nrows, Twiddles<double>& tw, SpatialB sb,
                         double fscale, double slack, Ctl* ctl, cudaStream_t st, const double* S) {
    if (!radix_row_ok(n2)) return false;
    bool done = false;
    switch (n2 / 2) {
#define X(n)                                                                                   \
    case n:                                                                                    \
        if constexpr (detail::RowCfg<double, n>::TT <= 32 && n >= 32) {                        \
            constexpr int E = detail::RowCfg<double, n>::E, TT = detail::RowCfg<double, n>::TT; \
            const int R = detail::rows_per_cta<double, n>(nrows);                              \
            const size_t smem = row_smem_bytes<double, n, E>(R);                               \
            auto k = k_row_r2c_eps0_sh<TI, n, E, SpatialB, Ctl>;                               \
            detail::set_smem(k, smem);                                                         \
            k<<<detail::persistent_grid(k, TT * R, smem, (nrows + R - 1) / R), TT * R, smem,   \
                st>>>(orig, dec, n2, out, out_stride, nrows, tw.stage_table(n, E),             \
                      tw.post_table(n), sb, fscale, slack, ctl, S);                            \
            FFCZ_LAUNCH_CHECK();                                                               \
            done = true;                                                                       \
        }                                                                                      \
        break;
        FFCZ_POW2_CASES(X)
#undef X
    }
    return done;
}

template <class T, class Hook>
void launch_row_r2c_hook(long long n2, const T* in, long long in_stride, cplx<T>* out,
                         long long out_stride, long long nrows, Twiddles<T>& tw, const int* gate,
                         Hook hook, cudaStream_t st) {
    if (radix_row_ok(n2)) {
        switch (n2 / 2) {
#define X(n)                                                                                   \
    case n:                                                                                    \
        detail::row_r2c_radix<T, n, Hook>(in, in_stride, out, out_stride, nrows, tw, gate, st, \
                                          hook);                                               \
        return;
            FFCZ_POW2_CASES(X)
#undef X
        }
    }
    throw Error(kUnsupported, "R2C with a hook needs a power-of-two last axis in [32, 8192]");
}

template <class T>
void launch_row_c2r(long long n2, const cplx<T>* in, long long in_stride, T* out,
                    long long out_stride, long long nrows, T scale, Twiddles<T>& tw,
                    const int* gate, cudaStream_t st) {
    if (radix_row_ok(n2)) {
        switch (n2 / 2) {
#define X(n)                                                                                   \
    case n:                                                                                    \
        detail::row_c2r_radix<T, n>(in, in_stride, out, out_stride, nrows, scale, tw, gate, st); \
        return;
            FFCZ_POW2_CASES(X)
#undef X
        }
    }
    const long long Lm = (n2 % 2 == 0) ? n2 / 2 : n2;
    if (const int R = detail::mixed_enabled() ? detail::mixed_lines<T>(Lm + 1, nrows, false) : 0) {
        const size_t smem = 2 * sizeof(cplx<T>) * (Lm + 1) * R;
        detail::set_smem(k_row_c2r_mixed<T>, smem);
        k_row_c2r_mixed<T><<<static_cast<unsigned>((nrows + R - 1) / R), 256, smem, st>>>(
            in, in_stride, out, out_stride, nrows, static_cast<int>(n2), R, make_mixed_plan(Lm),
            tw.table_for(n2), scale, gate);
        FFCZ_LAUNCH_CHECK();
        return;
    }
    const size_t smem = sizeof(cplx<T>) * (n2 / 2 + 1);
    if (smem > 96 * 1024) {  // longer than shared memory holds: global-memory passes
        large_row_c2r<T>(n2, in, in_stride, out, out_stride, nrows, scale, tw, gate, st);
        return;
    }
    detail::set_smem(k_row_c2r_direct<T>, smem);
    k_row_c2r_direct<T><<<static_cast<unsigned>(nrows), 256, smem, st>>>(
        in, in_stride, out, out_stride, static_cast<int>(n2), tw.table_for(n2), scale, gate);
    FFCZ_LAUNCH_CHECK();
}

template <class T, class Hook>
void launch_row_c2r_hook(long long n2, const cplx<T>* in, long long in_stride, T* out,
                         long long out_stride, long long nrows, T scale, Twiddles<T>& tw,
                         const int* gate, Hook hook, cudaStream_t st) {
    if (radix_row_ok(n2)) {
        switch (n2 / 2) {
#define X(n)                                                                                   \
    case n:                                                                                    \
        detail::row_c2r_radix<T, n, Hook>(in, in_stride, out, out_stride, nrows, scale, tw,    \
                                          gate, st, hook);                                     \
        return;
            FFCZ_POW2_CASES(X)
#undef X
        }
    }
    throw Error(kUnsupported, "C2R with a fused epilogue needs a power-of-two last axis in [32, 8192]");
}

template <class T, class Hook>
void launch_row_fused(long long n2, cplx<T>* data, long long stride, long long nrows,
                      long long real_stride, T scale, Twiddles<T>& tw, const int* gate, Hook hook,
                      cudaStream_t st, cplx<T>* out) {
    if (radix_row_ok(n2)) {
        switch (n2 / 2) {
#define X(n)                                                                                   \
    case n:                                                                                    \
        detail::row_fused_radix<T, n, Hook>(data, stride, nrows, real_stride, scale, tw, gate, \
                                            hook, st, out);                                    \
        return;
            FFCZ_POW2_CASES(X)
#undef X
        }
    }
    throw Error(kUnsupported, "fused row pass needs a power-of-two last axis in [32, 8192]");
}

template <class T>
void FftPlan<T>::r2c(const T* x, cplx<T>* half, const int* gate, cudaStream_t st) const {
    launch_row_r2c<T>(g.n2, x, g.n2, half, g.P, g.rows, *tw, gate, st);
    col<HookNone>(1, -1, half, half, gate, HookNone{}, st);
    col<HookNone>(0, -1, half, half, gate, HookNone{}, st);
}

template <class T>
void FftPlan<T>::c2r(const cplx<T>* half, cplx<T>* work, T* x, T scale, const int* gate,
                     cudaStream_t st) const {
    const cplx<T>* src = half;
    if (g.d[0] > 1) {
        col<HookNone>(0, +1, src, work, gate, HookNone{}, st);
        src = work;
    }
    if (g.d[1] > 1) {
        col<HookNone>(1, +1, src, work, gate, HookNone{}, st);
        src = work;
    }
    launch_row_c2r<T>(g.n2, src, g.P, x, g.n2, g.rows, scale, *tw, gate, st);
}

template <class T>
bool FftPlan<T>::fused_ok() const {
    if (!radix_row_ok(g.n2)) return false;
    for (int a = 0; a < 2; ++a)
        if (g.d[a] > 1 && !radix_col_ok(g.d[a])) return false;
    return g.ndim >= 2;
}

} // namespace ffcz_gpu
