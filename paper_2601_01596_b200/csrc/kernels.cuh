// Projection-loop hooks, control and FP64-gate kernels (sm_100a).
//
// Each device function cites the reference function whose arithmetic it restates; every
// comparison / clamp / accumulation is the same IEEE-754 double operation in the same order as
// the reference so that, given the same spectrum values, decisions and flags are identical.
#pragma once

#include "common.cuh"

namespace ffcz_gpu {

constexpr double kMaxIndex = 2147483520.0;  // pipeline.cpp:57 (overflow escapes)
// 2^e as a double (|e| < 1022) by its bit pattern: x * pow2i(e) == ldexp(x, e) bit for bit
// (both are the correctly rounded x 2^e), without ldexp's range-check sequence
__device__ __forceinline__ double pow2i(int e) {
    return __longlong_as_double(static_cast<long long>(1023 + e) << 52);
}

// ---- bounds ------------------------------------------------------------------------------------

// Spatial bound E(n) (bounds.hpp:11-18): per-point array or one global value.
struct SpatialB {
    const double* v;
    double g;
    __device__ __forceinline__ double at(long long n) const { return v ? v[n] : g; }
};

// Frequency bound Delta (bounds.hpp:20-31) restricted to the half spectrum, stored in the
// pitched half layout (offset = row*P + k2).  Hermitian consistency (bounds.cpp:50-54) makes the
// half restriction lossless.
struct FreqB {
    const double* re;
    const double* im;
    double g;
    __device__ __forceinline__ double re_at(long long off) const { return re ? re[off] : g; }
    __device__ __forceinline__ double im_at(long long off) const { return im ? im[off] : g; }
    // both lanes with one load when they share storage (rho-mode bounds: Re lane == Im lane)
    __device__ __forceinline__ double2 at2(long long off) const {
        if (!re) return make_double2(g, g);
        const double r = re[off];
        return make_double2(r, im == re ? r : im[off]);
    }
};

// a / b correctly rounded, given rb = RN(1/b) (one true division per kernel for a global bound):
// q0 = RN(a rb) is within an ulp of a / b, the remainder a - b q0 is exact under FMA, and one
// correction step RN(q0 + r rb) is the correctly rounded quotient (Markstein's final-step
// theorem; finite a, normal b and quotient, as the gate's values are) — bit for bit a / b,
// without the division's Newton sequence and range checks per element
__device__ __forceinline__ double div_rn(double a, double b, double rb) {
    const double q0 = a * rb;
    const double r = fma(-q0, b, a);
    return fma(r, rb, q0);
}

// std::clamp(v, -b, b) (projection.cpp:14-16)
template <class T>
__device__ __forceinline__ T clamp_abs(T v, T b) {
    return v < -b ? -b : (b < v ? b : v);
}

// ---- loop control block ------------------------------------------------------------------------

struct Ctl {
    unsigned long long peak_bits;  // max(|Re|,|Im|) of the current spectrum (as non-negative double)
    unsigned long long exc_bits;   // max(excess, 0)
    unsigned long long passes;
    unsigned long long max_iters;
    int done;
    int converged;
    double residual_f;
    unsigned long long bad1, bad2;       // first index failing the correct()/loop preconditions
    unsigned long long res_s_bits;       // residual_s
    unsigned long long act_s, act_f;     // active counts (act_f over the FULL spectrum)
    int dirty;                           // escape repair: a component violated this round
    int pad0;
    unsigned long long vs_bits, vf_bits; // verify: max spatial / frequency excess (> 0 only)
    unsigned long long count_a, count_b; // scratch totals of compactions
    // mixed policy
    int phase;                           // 0: FP32 phase, 1: FP64 phase
    int switch_now;
    unsigned long long passes32;
    double tau;
    int s_any;    // a spatial clip moved some sample (S is not identically zero)
    int dirty_s;  // escape repair: a spatial component was repaired this round
    double ex32_prev;  // mixed policy: max excess at the previous FP32 check
};

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* p, double v) {
    atomicMax(p, dbits(v));
}

// Block-wide max of two non-negative doubles, then one atomic per CTA.
__device__ __forceinline__ void block_max2_atomic(double a, double b, unsigned long long* pa,
                                                  unsigned long long* pb) {
    __shared__ double sa[32], sb[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sa[w] = a;
        sb[w] = b;
    }
    __syncthreads();
    if (w == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        a = l < nw ? sa[l] : 0.0;
        b = l < nw ? sb[l] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if (l == 0) {
            if (pa && a > 0.0) atomic_max_nonneg(pa, a);
            if (pb && b > 0.0) atomic_max_nonneg(pb, b);
        }
    }
}

// ---- loop hooks ----------------------------------------------------------------------------------

// check_convergence (projection.cpp:29-52) in one pass: peak = max(|Re|,|Im|) and
// max_excess = max(max(|Re|-Dre, |Im|-Dim), 0).  "some excess > 1e-11*peak" <=> max_excess > tol,
// and when violated the reference's max over violators equals the global max.
struct HookFReduce {
    FreqB fb;
    double fscale;  // working = original * (1 - 2^-m) (bounds.cpp:74-85); 1.0 for working input
    Ctl* ctl;
    double peak = 0.0, ex = 0.0;
    static constexpr bool kDelta = true;  // post_d takes Delta(off) from the caller (TMA side tile)
    template <class C> __device__ __forceinline__ void pre_d(C&, long long, int, double2) {}
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    template <class C>
    __device__ __forceinline__ void post_d(C& v, long long, int, double2 d) {
        const double ar = fabs(static_cast<double>(v.x)), ai = fabs(static_cast<double>(v.y));
        peak = fmax(peak, fmax(ar, ai));
        const double e = fmax(ar - d.x * fscale, ai - d.y * fscale);
        if (e > ex) ex = e;
    }
    template <class C>
    __device__ __forceinline__ void post(C& v, long long off, int c) { post_d(v, off, c, fb.at2(off)); }
    __device__ __forceinline__ void finish() { block_max2_atomic(peak, ex, &ctl->peak_bits, &ctl->exc_bits); }
};

// project_onto_fcube + F accumulation (projection.cpp:54-66, 117-119): clamp Re and Im
// independently; F += clipped - delta (read-modify-write only where the clamp moved the value).
// With `ctl` set (fused loop), the first clip pass (passes == 1 after the decision) writes F
// densely instead of read-modify-write: F is zero before it, so F = 0 + displacement exactly, and
// the loop needs no separate zero fill of F.
template <class T>
struct HookFClip {
    FreqB fb;
    double fscale;
    double2* F;
    const Ctl* ctl = nullptr;
    // rebuild mode (fused loop): after the first clip pass, F is not read-modify-written; the
    // pass only marks `moved[off] = 1` where a clamp moved a component, and the gate rebuilds
    // F = mask(delta_final - FFT(eps0 + S)) once (HookFRebuild) — the loop's invariant
    // eps = eps0 + S + IFFT(F) (projection.cpp:117-124) makes that the same sum.
    unsigned char* moved = nullptr;
    bool first = false;
    __device__ __forceinline__ void begin() {  // without ctl, `first` is the caller's value
        if (ctl) first = *reinterpret_cast<const volatile unsigned long long*>(&ctl->passes) == 1;
    }
    static constexpr bool kDelta = true;
    template <class C> __device__ __forceinline__ void post_d(C&, long long, int, double2) {}
    template <class C>
    __device__ __forceinline__ void pre(C& v, long long off, int c) { pre_d(v, off, c, fb.at2(off)); }
    template <class C>
    __device__ __forceinline__ void pre_d(C& v, long long off, int, double2 d) {
        const double re = v.x, im = v.y;
        const double dre = d.x * fscale, dim = d.y * fscale;
        const double cre = clamp_abs(re, dre), cim = clamp_abs(im, dim);
        const double xre = cre - re, xim = cim - im;
        if (moved) {
            if (first) F[off] = make_double2(0.0 + xre, 0.0 + xim);
            if (xre != 0.0 || xim != 0.0) moved[off] = 1;
        } else if (first) {
            F[off] = make_double2(0.0 + xre, 0.0 + xim);
        } else if (xre != 0.0 || xim != 0.0) {
            // read through the non-coherent path: element `off` is read once, by this thread,
            // before its own store, so the compiler may hoist the loads of the whole register
            // set above the pass's stores (no exposed latency per clipped element)
            double2 f = __ldg(&F[off]);
            f.x += xre;
            f.y += xim;
            F[off] = f;
        }
        v.x = static_cast<T>(cre);
        v.y = static_cast<T>(cim);
    }
    template <class C> __device__ __forceinline__ void post(C&, long long, int) {}
    __device__ __forceinline__ void finish() {}
};

// check_convergence (HookFReduce) and project_onto_fcube (HookFClip, rebuild mode) on the same
// spectrum values, between the forward and the inverse transform of the completing axis
// (k_col_tma1_rt): the loop's K3a + K3b as one HBM round trip from the forward chain's buffer
// into the inverse chain's (`old` = the component's mark, landed with the tile).  The clip is speculative: when the decision after the pass (k_decide)
// ends the loop at this check, the reference does not clip (projection.cpp:104-116), so the
// clipped output is dropped and the recovery launch (recover = 1, same kernel: the forward values
// are re-formed bit for bit) stores the spectrum and clears the marks only that clip set.
// Marks: 0 never moved, 1 moved by a committed clip, 2 first moved by the latest clip.  A clip
// that moves a component writes old ? 1 : 2 — every clip before the latest one is committed,
// since the loop went on past it; recovery turns a 2 the last clip set back into 0.
// F is written densely by the first clip (passes == 0 before its decision), as HookFClip does.
struct HookRT {
    FreqB fb;
    double fscale;
    Ctl* ctl;
    double2* F;
    unsigned char* moved;
    int recover = 0;
    // (const members only: the kernel keeps the first flag and the reduction in registers, so
    // the hook object never needs a local-memory copy)
    __device__ __forceinline__ bool fwd_only() const { return recover != 0; }
    __device__ __forceinline__ bool is_first() const {
        return *reinterpret_cast<const volatile unsigned long long*>(&ctl->passes) == 0;
    }
    template <class C>
    __device__ __forceinline__ void mid(C& v, long long off, double2 d, unsigned old, bool first,
                                        double& peak, double& ex) const {
        const double re = v.x, im = v.y;
        const double dre = d.x * fscale, dim = d.y * fscale;
        const double cre = clamp_abs(re, dre), cim = clamp_abs(im, dim);
        const double xre = cre - re, xim = cim - im;
        const bool mv = xre != 0.0 || xim != 0.0;
        if (recover) {
            if (mv && old == 2) moved[off] = 0;
            return;
        }
        const double ar = fabs(re), ai = fabs(im);
        peak = fmax(peak, fmax(ar, ai));
        const double e = fmax(ar - dre, ai - dim);
        if (e > ex) ex = e;
        if (first) F[off] = make_double2(0.0 + xre, 0.0 + xim);
        if (mv) moved[off] = old ? 1 : 2;
        v.x = cre;
        v.y = cim;
    }
    __device__ __forceinline__ void finish(double peak, double ex) const {
        if (!recover) block_max2_atomic(peak, ex, &ctl->peak_bits, &ctl->exc_bits);
    }
};

// ---- fused slab transpose (slab.py peer path) ---------------------------------------------------
// n / d for n < 2^32 by multiply-high (Granlund-Montgomery round-up method): the scatter decodes
// element offsets at every store, where a hardware-less 32-bit division would cost ~20 ops.
struct FastDiv {
    unsigned d = 1, m = 1;
    int l = 0;
    __host__ static FastDiv make(unsigned d) {
        FastDiv f;
        f.d = d;
        while ((1ull << f.l) < d) ++f.l;
        f.m = static_cast<unsigned>((((1ull << 32) * ((1ull << f.l) - d)) / d) + 1);
        return f;
    }
    __device__ __forceinline__ unsigned div(unsigned n) const {
        return static_cast<unsigned>((static_cast<unsigned long long>(__umulhi(n, m)) + n) >> l);
    }
};

// The all-to-all of slab.py (_transpose_ab / _transpose_ba) as the store of the pass that
// produces the data: element `off` of this rank's (d0, d1, P) buffer goes straight into the
// receive buffer of the rank that owns it in the other layout (CUDA IPC mappings; NVLink peer
// stores across GPUs).  Forward (A (c0, n1, P) -> B (n0, c1, P)): (i0, i1, k) -> rank i1 / c1,
// row (r c0 + i0) c1 + i1 mod c1.  Backward (B -> A): (i0, i1l, k) -> rank i0 / c0, row
// (i0 mod c0) n1 + r c1 + i1l.  Offsets of one slab fit 32 bits (checked on the host).
struct PeerScatter {
    double2* const* peers;  // W receive buffers, this rank's own at [r]
    FastDiv row;            // P
    // powers of two (the slab's hooked passes need power-of-two axes, so n1, c1 and c0 are):
    int d1_sh;              // d1 of this buffer (forward: n1; backward: c1)
    int part_sh;            // forward: c1; backward: c0
    int width_sh;           // forward: c1; backward: n1
    unsigned base;          // forward: r c0; backward: r c1
    int fwd;
    __device__ __forceinline__ void store(double2 v, long long off) const {
        const unsigned o = static_cast<unsigned>(off);
        const unsigned q = row.div(o), k = o - q * row.d;
        const unsigned a = q >> d1_sh, b = q & ((1u << d1_sh) - 1u);
        const unsigned x = fwd ? b : a;  // the exchanged index
        const unsigned s = x >> part_sh, xl = x & ((1u << part_sh) - 1u);
        const unsigned drow = fwd ? ((base + a) << width_sh) + xl : (xl << width_sh) + base + b;
        double2* dst = reinterpret_cast<double2*>(
            __ldg(reinterpret_cast<const unsigned long long*>(peers) + s));
        dst[static_cast<size_t>(drow) * row.d + k] = v;
    }
};

// plain pass whose outputs are scattered (FFCZ_SLAB_FWD_LOCAL_PEER: forward axis 1 of A)
struct HookScatter {
    static constexpr bool kNoStore = true;
    PeerScatter ps;
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    template <class C> __device__ __forceinline__ void post(C& v, long long off, int) {
        ps.store(make_double2(v.x, v.y), off);
    }
    // the peer stores are performed system-wide before the pass ends (the orchestrator's barrier
    // then orders them with the receiving rank's next pass)
    __device__ __forceinline__ void finish() { __threadfence_system(); }
};

// project_onto_fcube + inverse axis 0 (HookFClip) whose outputs are scattered back to the natural
// slabs (FFCZ_SLAB_COL0_CLIP_INV_PEER)
template <class T>
struct HookFClipScatter : HookFClip<T> {
    static constexpr bool kNoStore = true;
    PeerScatter ps;
    template <class C> __device__ __forceinline__ void post_d(C& v, long long off, int, double2) {
        ps.store(make_double2(v.x, v.y), off);
    }
    template <class C> __device__ __forceinline__ void post(C& v, long long off, int) {
        ps.store(make_double2(v.x, v.y), off);
    }
    __device__ __forceinline__ void finish() { __threadfence_system(); }
};

// project_onto_scube + S accumulation (projection.cpp:68-79, 121-124) on the real outputs of a
// C2R row pass; writes the clipped epsilon (the reference's `eps = sc.clipped`).
// Same first-pass dense write of S as HookFClip (S is zero before the first s-clip).
template <class T>
struct HookSClip {
    SpatialB sb;
    double fscale;
    double* S;
    T* eps;
    const Ctl* ctl = nullptr;
    bool first = false;
    int any = 0;  // a clip moved some sample of this CTA (reported as ctl->s_any)
    // fused row pass only: stop after the C2R half (re-forming the last iteration's epsilon after
    // the loop, with S == nullptr: no accumulation)
    int c2r_only = 0;
    __device__ __forceinline__ void begin() {  // without ctl, `first` is the caller's value
        if (ctl) first = *reinterpret_cast<const volatile unsigned long long*>(&ctl->passes) == 1;
    }
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    __device__ __forceinline__ T one(T x, long long n) {
        const double xd = x;
        const double e = sb.at(n) * fscale;
        const double c = clamp_abs(xd, e);
        const double d = c - xd;
        if (S) {
            if (first) S[n] = 0.0 + d;
            else if (d != 0.0) S[n] = __ldg(&S[n]) + d;  // see HookFClip
        }
        any |= d != 0.0;
        return static_cast<T>(c);
    }
    __device__ __forceinline__ void post_real(T& x0, T& x1, long long n) {
        x0 = one(x0, n);
        x1 = one(x1, n + 1);
        if (eps) reinterpret_cast<typename cvec<T>::type*>(eps)[n >> 1] = mkc<T>(x0, x1);
    }
    __device__ __forceinline__ void finish() {
        if (__syncthreads_or(any) && threadIdx.x == 0 && ctl)
            const_cast<Ctl*>(ctl)->s_any = 1;
    }
};

// Rebuild of the accumulated frequency edits at the end of a rebuild-mode loop: the pass
// transforms eps0 + S forward; F = delta_final - that, where any clip ever moved the component,
// else exactly 0 (the reference's F is exactly 0 where it never clipped, editset.cpp:43-66).
struct HookFRebuild {
    static constexpr bool kNoStore = true;
    const double2* delta;
    double2* F;
    const unsigned char* moved;
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    template <class C>
    __device__ __forceinline__ void post(C& v, long long off, int) {
        // both loads unconditional and through the non-coherent path, so the compiler can issue
        // the tile's loads ahead of its F stores (a plain load of `moved` after each F store
        // serialised them: 10.3 ms for 26 GB at 1024^3)
        const unsigned char mv = __ldg(&moved[off]);
        const double2 d = __ldg(&delta[off]);
        F[off] = mv ? make_double2(d.x - v.x, d.y - v.y) : make_double2(0.0, 0.0);
    }
    __device__ __forceinline__ void finish() {}
};

// eps0 + S (the forward input of the F rebuild), eps0 = dec - orig as k_eps0 forms it
template <class TI>
__global__ void k_eps0_plus_s(const TI* __restrict__ orig, const TI* __restrict__ dec,
                              const double* __restrict__ S, double* out, long long N);

// ---- batched frames (BASELINE config 3): one projection loop over a stack of 2-D frames --------
// Every frame keeps its own control block, bounds and decision (each frame is an independent
// correct(), pipeline.cpp:26-178); the passes run over the whole stack and skip the tiles of
// frames that have converged, so a frame's state freezes exactly where its own loop stops.
// Tiled hooks (kTiled) get tile_skip / tile_begin / tile_end around every tile (CTA-uniform);
// `unit` is the tile's plane (column passes along axis 1: plane = frame) or its first row (row
// passes: frame = row / rows_per_frame).
struct FrameCtl {
    unsigned long long peak_bits, exc_bits, passes, max_iters;
    int done, converged;
    double residual_f;
};

struct FrameBatch {
    FrameCtl* fc;
    const double* E;          // spatial bound per frame
    const double* D;          // frequency bound per frame
    double fscale;            // 1 - 2^-m (working bounds)
    long long rows_per_frame; // n1
    __device__ __forceinline__ long long frame_of(long long unit, bool rows) const {
        return rows ? unit / rows_per_frame : unit;
    }
    __device__ __forceinline__ bool done(long long f) const {
        return *reinterpret_cast<const volatile int*>(&fc[f].done) != 0;
    }
    __device__ __forceinline__ bool first(long long f) const {
        return *reinterpret_cast<const volatile unsigned long long*>(&fc[f].passes) == 1;
    }
};

template <bool kRows>
struct HookSkipB {  // plain pass that only skips converged frames
    static constexpr bool kTiled = true;
    FrameBatch fb;
    __device__ __forceinline__ bool tile_skip(long long u) const { return fb.done(fb.frame_of(u, kRows)); }
    __device__ __forceinline__ void tile_begin(long long) {}
    __device__ __forceinline__ void tile_end() {}
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    template <class C> __device__ __forceinline__ void post(C&, long long, int) {}
    template <class T> __device__ __forceinline__ void post_real(T&, T&, long long) {}
    __device__ __forceinline__ void finish() {}
};

// check_convergence per frame (projection.cpp:29-52), flushed per tile to the frame's block
struct HookFReduceB {
    static constexpr bool kTiled = true;
    FrameBatch fb;
    long long frame = 0;
    double d = 0.0, peak = 0.0, ex = 0.0;
    __device__ __forceinline__ bool tile_skip(long long u) const { return fb.done(u); }
    __device__ __forceinline__ void tile_begin(long long u) {
        frame = u;
        d = fb.D[u] * fb.fscale;
        peak = 0.0;
        ex = 0.0;
    }
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    template <class C>
    __device__ __forceinline__ void post(C& v, long long, int) {
        const double ar = fabs(static_cast<double>(v.x)), ai = fabs(static_cast<double>(v.y));
        peak = fmax(peak, fmax(ar, ai));
        const double e = fmax(ar - d, ai - d);
        if (e > ex) ex = e;
    }
    __device__ __forceinline__ void tile_end() {
        block_max2_atomic(peak, ex, &fb.fc[frame].peak_bits, &fb.fc[frame].exc_bits);
    }
    __device__ __forceinline__ void finish() {}
};

// project_onto_fcube per frame (projection.cpp:54-66): F dense on the frame's first clip, clip
// map afterwards (HookFClip rebuild mode)
template <class T>
struct HookFClipB {
    static constexpr bool kTiled = true;
    FrameBatch fb;
    double2* F;
    unsigned char* moved;
    double d = 0.0;
    bool first = false;
    __device__ __forceinline__ bool tile_skip(long long u) const { return fb.done(u); }
    __device__ __forceinline__ void tile_begin(long long u) {
        d = fb.D[u] * fb.fscale;
        first = fb.first(u);
    }
    template <class C>
    __device__ __forceinline__ void pre(C& v, long long off, int) {
        const double re = v.x, im = v.y;
        const double cre = clamp_abs(re, d), cim = clamp_abs(im, d);
        const double xre = cre - re, xim = cim - im;
        if (first) F[off] = make_double2(0.0 + xre, 0.0 + xim);
        if (xre != 0.0 || xim != 0.0) moved[off] = 1;
        v.x = static_cast<T>(cre);
        v.y = static_cast<T>(cim);
    }
    template <class C> __device__ __forceinline__ void post(C&, long long, int) {}
    __device__ __forceinline__ void tile_end() {}
    __device__ __forceinline__ void finish() {}
};

// project_onto_scube per frame (projection.cpp:68-79) on the C2R outputs
template <class T>
struct HookSClipB {
    static constexpr bool kTiled = true;
    FrameBatch fb;
    double* S;
    double e = 0.0;
    bool first = false;
    __device__ __forceinline__ bool tile_skip(long long u) const { return fb.done(fb.frame_of(u, true)); }
    __device__ __forceinline__ void tile_begin(long long u) {
        const long long f = fb.frame_of(u, true);
        e = fb.E[f] * fb.fscale;
        first = fb.first(f);
    }
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    __device__ __forceinline__ T one(T x, long long n) const {
        const double xd = x;
        const double c = clamp_abs(xd, e);
        const double dd = c - xd;
        if (first) S[n] = 0.0 + dd;
        else if (dd != 0.0) S[n] = __ldg(&S[n]) + dd;
        return static_cast<T>(c);
    }
    __device__ __forceinline__ void post_real(T& x0, T& x1, long long n) {
        x0 = one(x0, n);
        x1 = one(x1, n + 1);
    }
    __device__ __forceinline__ void tile_end() {}
    __device__ __forceinline__ void finish() {}
};

// loop decision per frame (projection.cpp:106-116); the last frame to finish sets ctl->done
__global__ void k_decide_frames(FrameCtl* fc, long long nframes, Ctl* ctl);
__global__ void k_frames_init(FrameCtl* fc, long long nframes, unsigned long long max_iters);
// compute_error + preconditions of every frame (pipeline.cpp:31-42; first failing index)
template <class TI>
__global__ void k_eps0_frames(const TI* __restrict__ orig, const TI* __restrict__ dec, double* eps,
                              long long N, long long frameN, const double* __restrict__ E,
                              double fscale, double slack, Ctl* ctl);

// ---- FP64 gate hooks (fused into the round / verify passes) -----------------------------------------

__device__ __forceinline__ void set_bit_g(unsigned* words, long long i) {
    atomicOr(&words[i >> 5], 1u << (i & 31));
}

template <class TI> struct Pair2;
template <> struct Pair2<float> { using type = float2; };
template <> struct Pair2<double> { using type = double2; };

template <class TI>
__device__ __forceinline__ double2 load_pair(const TI* p, long long n) {
    const typename Pair2<TI>::type v = *reinterpret_cast<const typename Pair2<TI>::type*>(p + n);
    return make_double2(static_cast<double>(v.x), static_cast<double>(v.y));
}

// apply_edits + verify_bounds, spatial side (archive.cpp:262-287): corrected = dec + spat_cur +
// Re(IFFT(freq_cur)) is written out, eps = corrected - orig goes on to the R2C half.
template <class TI>
struct HookVerifyS {
    const TI* orig;
    const TI* dec;
    const double* spat_cur;
    double* corrected;
    SpatialB sb;
    Ctl* ctl;
    double m = 0.0;
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    __device__ __forceinline__ void post_real(double& x0, double& x1, long long n) {
        const double2 o = load_pair(orig, n), d = load_pair(dec, n);
        const double2 sc = *reinterpret_cast<const double2*>(spat_cur + n);
        const double c0 = d.x + sc.x + x0, c1 = d.y + sc.y + x1;
        if (corrected) *reinterpret_cast<double2*>(corrected + n) = make_double2(c0, c1);
        x0 = c0 - o.x;
        x1 = c1 - o.y;
        const double ex0 = fabs(x0) - sb.at(n), ex1 = fabs(x1) - sb.at(n + 1);
        if (ex0 > 0.0 && ex0 > m) m = ex0;
        if (ex1 > 0.0 && ex1 > m) m = ex1;
    }
    __device__ __forceinline__ void finish() { block_max2_atomic(m, 0.0, &ctl->vs_bits, nullptr); }
};

// One escape-repair round fused with a speculative apply_edits + verify_bounds (archive.cpp:262-287)
// on the same inverse transform: when the round turns out clean (no component repaired, so
// spat_cur and freq_cur are final), the decoder view dec + spat_cur + Re(IFFT(freq_cur)) is the
// one this pass already has, and the separate verify inverse (3 passes) is skipped.  Writes
// eps_tilde (handed on to the R2C; the pinned components get spat_cur + (final_eps - eps_tilde),
// pipeline.cpp:154-160), plus `corrected` and eps_v = corrected - orig.  The two
// epsilons are formed exactly as the reference forms them (eps0 + s + f vs (dec + s + f) - orig).
template <class TI>
struct HookRepairVerifyS {
    const TI* orig;
    const TI* dec;
    double* spat_cur;
    const double* final_eps;
    SpatialB sb;
    unsigned* esc_words;
    double* corrected;
    double* eps_v;
    Ctl* ctl;
    bool sc_zero = false;  // spat_cur is identically zero (no spatial edits): skip its load
    // spat_cur is nonzero only where a spatial flag or escape bit is set (quantised edits,
    // overflow escapes, repairs — each sets its esc bit): with the flag bitmap given, spat_cur
    // is loaded only for those samples (one cached bitmap word per 32 samples instead of 8 B
    // per sample: at 1024^3 config 4 the round's C2R moves 26 GB instead of 34)
    const unsigned* keep_words = nullptr;
    // decoder-view repair: check and repair the decoder's own view v = (dec + S + fpart) - orig
    // instead of eps_tilde = (dec - orig) + S + fpart (same value up to rounding) and hand v to
    // the round's forward transform, so a clean round IS verify_bounds (no separate verify
    // transform, no eps_v store).  Off = the reference's order (pipeline.cpp:134-160).
    bool dview = false;
    int dirty = 0;
    double m = 0.0;
    // orig / dec rows prefetched into shared memory by the row kernel (hook_prefetch)
    static constexpr bool kPrefetch = true;
    const TI* po = nullptr;
    const TI* pd = nullptr;
    long long pbase = 0;
    __host__ __device__ static constexpr unsigned prefetch_scalar_bytes() { return sizeof(TI); }
    __device__ __forceinline__ const void* prefetch_src(int k, long long n0) const {
        return (k ? dec : orig) + n0;
    }
    __device__ __forceinline__ void use_prefetch(const void* o, const void* d, long long n0) {
        po = static_cast<const TI*>(o);
        pd = static_cast<const TI*>(d);
        pbase = n0;
    }
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    __device__ __forceinline__ void post_real(double& x0, double& x1, long long n) {
        const double2 o = po ? load_pair(po, n - pbase) : load_pair(orig, n);
        const double2 d = pd ? load_pair(pd, n - pbase) : load_pair(dec, n);
        double2 sc = make_double2(0.0, 0.0);
        if (!sc_zero) {
            bool any = true;
            if (keep_words) {  // n is even: both samples' bits sit in one word
                // (this sample's esc bits change only by this thread, in an earlier round)
                const unsigned w = __ldg(keep_words + (n >> 5)) | esc_words[n >> 5];
                any = (w >> (n & 31)) & 3u;
            }
            if (any) sc = *reinterpret_cast<const double2*>(spat_cur + n);
        }
        const double e0 = d.x - o.x, e1 = d.y - o.y;
        const double c0 = d.x + sc.x + x0, c1 = d.y + sc.y + x1;
        const double v0 = c0 - o.x, v1 = c1 - o.y;
        if (corrected) *reinterpret_cast<double2*>(corrected + n) = make_double2(c0, c1);
        if (!dview) *reinterpret_cast<double2*>(eps_v + n) = make_double2(v0, v1);
        const double E0 = sb.at(n), E1 = sb.at(n + 1);
        const double ex0 = fabs(v0) - E0, ex1 = fabs(v1) - E1;
        if (ex0 > 0.0 && ex0 > m) m = ex0;
        if (ex1 > 0.0 && ex1 > m) m = ex1;
        const double t0 = dview ? v0 : e0 + sc.x + x0, t1 = dview ? v1 : e1 + sc.y + x1;
        bool w = false;
        if (fabs(t0) > E0) {
            sc.x = sc.x + (final_eps[n] - t0);
            set_bit_g(esc_words, n);
            w = true;
        }
        if (fabs(t1) > E1) {
            sc.y = sc.y + (final_eps[n + 1] - t1);
            set_bit_g(esc_words, n + 1);
            w = true;
        }
        if (w) {
            *reinterpret_cast<double2*>(spat_cur + n) = sc;
            dirty = 1;
        }
        x0 = t0;
        x1 = t1;
    }
    __device__ __forceinline__ void finish() {
        if (__syncthreads_or(dirty) && threadIdx.x == 0) {
            ctl->dirty = 1;
            ctl->dirty_s = 1;
        }
        block_max2_atomic(m, 0.0, &ctl->vs_bits, nullptr);
    }
};

// Frequency check of an escape-repair round (pipeline.cpp:140-147): marks violating components
// of delta_tilde (against the ORIGINAL Delta) in a bitmap over storage offsets; the repair itself
// is done sparsely afterwards (k_repair_freq_sparse) because conjugate partners live in other
// columns.
struct HookMarkViol {
    FreqB fb;
    unsigned* viol_words;
    Ctl* ctl;
    int any = 0;
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    static constexpr bool kDelta = true;
    template <class C> __device__ __forceinline__ void pre_d(C&, long long, int, double2) {}
    template <class C>
    __device__ __forceinline__ void post(C& v, long long off, int c) { post_d(v, off, c, fb.at2(off)); }
    template <class C>
    __device__ __forceinline__ void post_d(C& v, long long off, int, double2 d) {
        if (fabs(v.x) > d.x || fabs(v.y) > d.y) {
            set_bit_g(viol_words, off);
            any = 1;
        }
    }
    __device__ __forceinline__ void finish() {
        if (__syncthreads_or(any) && threadIdx.x == 0) ctl->dirty = 1;
    }
};

// verify_bounds, frequency side (archive.cpp:288-294): max positive excess; output not stored.
struct HookVerifyF {
    static constexpr bool kNoStore = true;
    FreqB fb;
    Ctl* ctl;
    double m = 0.0;
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    static constexpr bool kDelta = true;
    template <class C> __device__ __forceinline__ void pre_d(C&, long long, int, double2) {}
    template <class C>
    __device__ __forceinline__ void post(C& v, long long off, int c) { post_d(v, off, c, fb.at2(off)); }
    template <class C>
    __device__ __forceinline__ void post_d(C& v, long long, int, double2 d) {
        const double ex = fmax(fabs(v.x) - d.x, fabs(v.y) - d.y);
        if (ex > 0.0 && ex > m) m = ex;
    }
    __device__ __forceinline__ void finish() { block_max2_atomic(m, 0.0, &ctl->vf_bits, nullptr); }
};

// ---- batched frames: the FP64 gate over the whole stack ---------------------------------------------
// Per-frame gate state (pipeline.cpp:46-176 for each frame); `active` masks select the frames a
// pass works on (tiles of other frames are skipped, so their buffers are untouched).
struct FrameGate {
    unsigned long long act_s, act_f;   // active counts (act_f over the full spectrum)
    unsigned long long vs_bits, vf_bits;
    int dirty, dirty_s;
    int pad[2];
};

struct FrameMask {
    const int* active;                 // per frame: process (1) / skip (0)
    long long rows_per_frame;          // n1
    __device__ __forceinline__ long long frame_of(long long u, bool rows) const {
        return rows ? u / rows_per_frame : u;
    }
    __device__ __forceinline__ bool skip(long long f) const { return active[f] == 0; }
};

template <bool kRows>
struct HookMaskB {  // plain pass over the active frames
    static constexpr bool kTiled = true;
    FrameMask fm;
    __device__ __forceinline__ bool tile_skip(long long u) const { return fm.skip(fm.frame_of(u, kRows)); }
    __device__ __forceinline__ void tile_begin(long long) {}
    __device__ __forceinline__ void tile_end() {}
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    template <class C> __device__ __forceinline__ void post(C&, long long, int) {}
    template <class T> __device__ __forceinline__ void post_real(T&, T&, long long) {}
    __device__ __forceinline__ void finish() {}
};

// F rebuild (HookFRebuild) for the frames that need it
struct HookFRebuildB {
    static constexpr bool kTiled = true;
    static constexpr bool kNoStore = true;
    FrameMask fm;
    const double2* delta;
    double2* F;
    const unsigned char* moved;
    __device__ __forceinline__ bool tile_skip(long long u) const { return fm.skip(u); }
    __device__ __forceinline__ void tile_begin(long long) {}
    __device__ __forceinline__ void tile_end() {}
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    template <class C>
    __device__ __forceinline__ void post(C& v, long long off, int) {
        const unsigned char mv = __ldg(&moved[off]);  // hoistable loads (HookFRebuild)
        const double2 d = __ldg(&delta[off]);
        F[off] = mv ? make_double2(d.x - v.x, d.y - v.y) : make_double2(0.0, 0.0);
    }
    __device__ __forceinline__ void finish() {}
};

// escape-repair round + speculative decoder view (HookRepairVerifyS) per frame
template <class TI>
struct HookRepairVerifySB {
    static constexpr bool kTiled = true;
    FrameMask fm;
    const double* E;     // per frame
    FrameGate* fg;
    const TI* orig;
    const TI* dec;
    double* spat_cur;
    const double* final_eps;
    unsigned* esc_words;
    double* corrected;
    double* eps_v;
    bool dview = false;  // HookRepairVerifyS::dview
    long long frame = 0;
    double e = 0.0, m = 0.0;
    int dirty = 0;
    __device__ __forceinline__ bool tile_skip(long long u) const { return fm.skip(fm.frame_of(u, true)); }
    __device__ __forceinline__ void tile_begin(long long u) {
        frame = fm.frame_of(u, true);
        e = E[frame];
        m = 0.0;
        dirty = 0;
    }
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    __device__ __forceinline__ void post_real(double& x0, double& x1, long long n) {
        const double2 o = load_pair(orig, n), d = load_pair(dec, n);
        double2 sc = *reinterpret_cast<const double2*>(spat_cur + n);
        const double e0 = d.x - o.x, e1 = d.y - o.y;
        const double c0 = d.x + sc.x + x0, c1 = d.y + sc.y + x1;
        const double v0 = c0 - o.x, v1 = c1 - o.y;
        if (corrected) *reinterpret_cast<double2*>(corrected + n) = make_double2(c0, c1);
        if (!dview) *reinterpret_cast<double2*>(eps_v + n) = make_double2(v0, v1);
        const double ex0 = fabs(v0) - e, ex1 = fabs(v1) - e;
        if (ex0 > 0.0 && ex0 > m) m = ex0;
        if (ex1 > 0.0 && ex1 > m) m = ex1;
        const double t0 = dview ? v0 : e0 + sc.x + x0, t1 = dview ? v1 : e1 + sc.y + x1;
        bool w = false;
        if (fabs(t0) > e) {
            sc.x = sc.x + (final_eps[n] - t0);
            set_bit_g(esc_words, n);
            w = true;
        }
        if (fabs(t1) > e) {
            sc.y = sc.y + (final_eps[n + 1] - t1);
            set_bit_g(esc_words, n + 1);
            w = true;
        }
        if (w) {
            *reinterpret_cast<double2*>(spat_cur + n) = sc;
            dirty = 1;
        }
        x0 = t0;
        x1 = t1;
    }
    __device__ __forceinline__ void tile_end() {
        if (__syncthreads_or(dirty) && threadIdx.x == 0) {
            fg[frame].dirty = 1;
            fg[frame].dirty_s = 1;
        }
        block_max2_atomic(m, 0.0, &fg[frame].vs_bits, nullptr);
    }
    __device__ __forceinline__ void finish() {}
};

// apply_edits + verify_bounds spatial side (HookVerifyS) per frame
template <class TI>
struct HookVerifySB {
    static constexpr bool kTiled = true;
    FrameMask fm;
    const double* E;
    FrameGate* fg;
    const TI* orig;
    const TI* dec;
    const double* spat_cur;
    double* corrected;
    long long frame = 0;
    double e = 0.0, m = 0.0;
    __device__ __forceinline__ bool tile_skip(long long u) const { return fm.skip(fm.frame_of(u, true)); }
    __device__ __forceinline__ void tile_begin(long long u) {
        frame = fm.frame_of(u, true);
        e = E[frame];
        m = 0.0;
    }
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    __device__ __forceinline__ void post_real(double& x0, double& x1, long long n) {
        const double2 o = load_pair(orig, n), d = load_pair(dec, n);
        const double2 sc = *reinterpret_cast<const double2*>(spat_cur + n);
        const double c0 = d.x + sc.x + x0, c1 = d.y + sc.y + x1;
        if (corrected) *reinterpret_cast<double2*>(corrected + n) = make_double2(c0, c1);
        x0 = c0 - o.x;
        x1 = c1 - o.y;
        const double ex0 = fabs(x0) - e, ex1 = fabs(x1) - e;
        if (ex0 > 0.0 && ex0 > m) m = ex0;
        if (ex1 > 0.0 && ex1 > m) m = ex1;
    }
    __device__ __forceinline__ void tile_end() { block_max2_atomic(m, 0.0, &fg[frame].vs_bits, nullptr); }
    __device__ __forceinline__ void finish() {}
};

// violation marking (HookMarkViol) per frame
struct HookMarkViolB {
    static constexpr bool kTiled = true;
    FrameMask fm;
    const double* D;
    FrameGate* fg;
    unsigned* viol_words;
    long long frame = 0;
    double d = 0.0;
    int any = 0;
    __device__ __forceinline__ bool tile_skip(long long u) const { return fm.skip(u); }
    __device__ __forceinline__ void tile_begin(long long u) {
        frame = u;
        d = D[u];
        any = 0;
    }
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    template <class C>
    __device__ __forceinline__ void post(C& v, long long off, int) {
        if (fabs(v.x) > d || fabs(v.y) > d) {
            set_bit_g(viol_words, off);
            any = 1;
        }
    }
    __device__ __forceinline__ void tile_end() {
        if (__syncthreads_or(any) && threadIdx.x == 0) fg[frame].dirty = 1;
    }
    __device__ __forceinline__ void finish() {}
};

// verify_bounds frequency side (HookVerifyF) per frame, output not stored
struct HookVerifyFB {
    static constexpr bool kTiled = true;
    static constexpr bool kNoStore = true;
    FrameMask fm;
    const double* D;
    FrameGate* fg;
    long long frame = 0;
    double d = 0.0, m = 0.0;
    __device__ __forceinline__ bool tile_skip(long long u) const { return fm.skip(u); }
    __device__ __forceinline__ void tile_begin(long long u) {
        frame = u;
        d = D[u];
        m = 0.0;
    }
    template <class C> __device__ __forceinline__ void pre(C&, long long, int) {}
    template <class C>
    __device__ __forceinline__ void post(C& v, long long, int) {
        const double ex = fmax(fabs(v.x) - d, fabs(v.y) - d);
        if (ex > 0.0 && ex > m) m = ex;
    }
    __device__ __forceinline__ void tile_end() { block_max2_atomic(m, 0.0, &fg[frame].vf_bits, nullptr); }
    __device__ __forceinline__ void finish() {}
};

// ---- elementwise kernels (unfused path / generic shapes) -------------------------------------------

struct HalfGeom {
    long long rows;  // prod(dims[:-1])
    int H;           // n2/2 + 1
    int P;           // pitch
    long long n2;
    double invH;     // 1.0 / H
    // storage offset of half-grid index h = row*H + k2 (no 64-bit integer division)
    __device__ __forceinline__ long long offset_of(long long h) const {
        long long q = static_cast<long long>(static_cast<double>(h) * invH);
        long long r = h - q * H;
        if (r < 0) { --q; r += H; } else if (r >= H) { ++q; r -= H; }
        return q * P + r;
    }
};

// check_convergence over the half spectrum (projection.cpp:29-52)
__global__ void k_freduce(const double2* __restrict__ spec, HalfGeom g, FreqB fb, double fscale,
                          Ctl* ctl, const int* gate);
// project_onto_fcube + F += displacement (projection.cpp:54-66, 117-119)
__global__ void k_fclip(double2* spec, HalfGeom g, FreqB fb, double fscale, double2* F,
                        const int* gate);
// project_onto_scube + S += displacement; eps = clipped (projection.cpp:68-79, 121-124)
__global__ void k_sclip(const double* __restrict__ x, double* eps, long long N, SpatialB sb,
                        double fscale, double* S, const int* gate);
// compute_error + both preconditions (projection.cpp:20-27,88-94; pipeline.cpp:31-37)
template <class TI>
__global__ void k_eps0(const TI* __restrict__ orig, const TI* __restrict__ dec, double* eps,
                       long long N, SpatialB sb, double fscale, double slack, int check_original,
                       Ctl* ctl);
__global__ void k_cast_to_double(const float* __restrict__ in, double* out, long long N);
__global__ void k_cast_to_float(const double* __restrict__ in, float* out, long long N);
// mixed policy: FP32-phase decision (switch to FP64 when excess <= tau * peak)
__global__ void k_decide32(Ctl* ctl);
// loop decision (projection.cpp:106-116,125)
__global__ void k_decide(Ctl* ctl);
__global__ void k_ctl_init(Ctl* ctl, unsigned long long max_iters);
__global__ void k_export_ctl(const Ctl* __restrict__ ctl, Ctl* host);
// report: residual_s (projection.cpp:129-133)
__global__ void k_residual_s(const double* __restrict__ eps, long long N, SpatialB sb,
                             double fscale, Ctl* ctl);
__global__ void k_count_spatial(const double* __restrict__ S, long long N, Ctl* ctl);
__global__ void k_count_freq(const double2* __restrict__ F, HalfGeom g, Ctl* ctl);

// bounds: full -> half restriction of per-component arrays
__global__ void k_gather_half(const double* __restrict__ full, double* half, HalfGeom g);
// half <-> full spectrum expansion (expand_edits' conjugate mirror, archive.cpp:251-258)
__global__ void k_expand_full(const double2* __restrict__ half, double2* full, int ndim,
                              long long d0, long long d1, long long d2, int P);

// ---- FP64 gate (pipeline.cpp:46-176) ---------------------------------------------------------------

// compact_edits + overflow escapes + quantize->dequantize (editset.cpp:43-66,76-104;
// pipeline.cpp:57-106).  Writes the decoder-view dense array, the keep / escape bitmaps.
__global__ void k_gate_spatial(const double* __restrict__ S, long long N, SpatialB sb, int m,
                               double* spat_cur, unsigned* keep_words, unsigned* esc_words,
                               Ctl* ctl);
__global__ void k_gate_codes_freq(const double2* __restrict__ F, HalfGeom g, FreqB fb, int m,
                                  double2* freq_cur, unsigned* keep_words, unsigned* esc_words,
                                  int* codes, unsigned long long* tile_status,
                                  unsigned* tile_ticket, long long ntiles, Ctl* ctl);
constexpr long long kGateCodesTile = 4096;  // k_gate_codes_freq: half entries per tile
__global__ void k_gate_freq(const double2* __restrict__ F, HalfGeom g, FreqB fb, int m,
                            double2* freq_cur, unsigned* keep_words, unsigned* esc_words,
                            Ctl* ctl);
// bitmap compaction helpers
__global__ void k_popc_blocks(const unsigned* __restrict__ words, long long nwords,
                              unsigned long long* block_counts);
__global__ void k_scan_blocks(unsigned long long* counts, long long nblocks,
                              unsigned long long* total);
__global__ void k_compact(const unsigned* __restrict__ words, long long nwords,
                          const unsigned long long* __restrict__ block_offsets,
                          unsigned long long* out_idx);
// int32 codes of the kept edits, in flag order (editset.cpp:86-119)
__global__ void k_codes_spatial(const unsigned long long* __restrict__ idx, long long n,
                                const double* __restrict__ S, SpatialB sb, int m, int* codes);
__global__ void k_codes_freq(const unsigned long long* __restrict__ idx, long long n,
                             const double2* __restrict__ F, HalfGeom g, FreqB fb, int m,
                             int* codes);
// the same codes straight from the keep bitmap + k_popc_blocks/k_scan_blocks offsets (1024
// words per CTA, 1024 threads): no index list round trip
__global__ void __launch_bounds__(1024) k_codes_spatial_bits(const unsigned* __restrict__ keep_words, long long nwords,
                                     const unsigned long long* __restrict__ block_offsets,
                                     const double* __restrict__ S, SpatialB sb, int m, int* codes);
__global__ void __launch_bounds__(1024) k_codes_freq_bits(const unsigned* __restrict__ keep_words, long long nwords,
                                  const unsigned long long* __restrict__ block_offsets,
                                  const double2* __restrict__ F, HalfGeom g, FreqB fb, int m,
                                  int* codes);
// escape repair (pipeline.cpp:114-163)
template <class TI>
__global__ void k_repair_spatial(const TI* __restrict__ orig, const TI* __restrict__ dec,
                                 const double* __restrict__ fpart, const double* __restrict__ final_eps,
                                 long long N, SpatialB sb, double* spat_cur, double* eps_tilde,
                                 unsigned* esc_words, Ctl* ctl);
__global__ void k_repair_freq(const double2* __restrict__ delta_star,
                              const double2* __restrict__ delta_tilde, HalfGeom g, int ndim,
                              long long d0, long long d1, FreqB fb, double2* freq_cur,
                              unsigned* esc_words, Ctl* ctl);
// apply_edits + verify_bounds (archive.cpp:262-297)
template <class TI>
__global__ void k_verify_spatial(const TI* __restrict__ orig, const TI* __restrict__ dec,
                                 const double* __restrict__ spat_cur,
                                 const double* __restrict__ fpart, long long N, SpatialB sb,
                                 double* corrected, double* eps_v, Ctl* ctl);
__global__ void k_verify_freq(const double2* __restrict__ delta, HalfGeom g, FreqB fb, Ctl* ctl);
// sparse frequency repair from the violation bitmap of HookMarkViol (pipeline.cpp:140-153)
__global__ void k_repair_freq_sparse(const unsigned* __restrict__ viol_words, long long nwords,
                                     const double2* __restrict__ delta_star,
                                     const double2* __restrict__ delta_tilde, HalfGeom g,
                                     long long d0, long long d1, double2* freq_cur,
                                     unsigned* esc_words);
// device image of ffcz_cuda_escape (include/ffcz_cuda.h): int32 frequency, u64 index, re, im
struct EscapeRec {
    int frequency;
    int pad;
    unsigned long long index;
    double re, im;
};
static_assert(sizeof(EscapeRec) == 32, "EscapeRec layout");
// decoder side (expand_edits / apply_edits, archive.cpp:227-273)
__global__ void k_dequant_spatial_bits(const unsigned* __restrict__ keep_words, long long nwords,
                                       const unsigned long long* __restrict__ block_offsets,
                                       const int* __restrict__ codes, SpatialB sb, int m,
                                       double* spat);
__global__ void __launch_bounds__(1024) k_dequant_freq_bits(const unsigned* __restrict__ keep_words, long long nwords,
                                    const unsigned long long* __restrict__ block_offsets,
                                    const int* __restrict__ codes, HalfGeom g, FreqB fb, int m,
                                    double2* freq);
__global__ void k_scatter_escapes(const EscapeRec* __restrict__ recs, long long n, double* spat,
                                  double2* freq, HalfGeom g);
template <class TI>
__global__ void k_apply_sum(const TI* __restrict__ dec, const double* __restrict__ spat,
                            const double* __restrict__ fpart, double* out, long long N);
__global__ void k_escape_records_s(const unsigned long long* __restrict__ idx, long long n,
                                   const double* __restrict__ spat_cur, EscapeRec* out);
__global__ void k_escape_records_f(const unsigned long long* __restrict__ idx, long long n,
                                   const double2* __restrict__ freq_cur, HalfGeom g, EscapeRec* out);
__global__ void k_gather_escapes_s(const unsigned long long* __restrict__ idx, long long n,
                                   const double* __restrict__ spat_cur, double* out_re);
__global__ void k_gather_escapes_f(const unsigned long long* __restrict__ idx, long long n,
                                   const double2* __restrict__ freq_cur, HalfGeom g, double2* out);

// inverse_dft helpers: Hermitian / anti-Hermitian parts of a FULL spectrum on the half grid
__global__ void k_split_hermitian(const double2* __restrict__ full, double2* Hh, double2* Ah,
                                  HalfGeom g, long long d0, long long d1);
__global__ void k_maxabs(const double* __restrict__ x, long long N, unsigned long long* out);

// gate kernels over the stack with per-frame bounds (frame = n / frameN, row / n1)
__global__ void k_gate_spatial_frames(const double* __restrict__ S, long long N, long long frameN,
                                      const double* __restrict__ E, int m, double* spat_cur,
                                      unsigned* keep_words, unsigned* esc_words, FrameGate* fg);
__global__ void k_gate_freq_frames(const double2* __restrict__ F, HalfGeom g, long long n1,
                                   const double* __restrict__ D, int m, double2* freq_cur,
                                   unsigned* keep_words, unsigned* esc_words, FrameGate* fg);
__global__ void k_codes_spatial_frames(const unsigned* __restrict__ keep_words, long long nwords,
                                       const unsigned long long* __restrict__ block_offsets,
                                       const double* __restrict__ S, long long frameN,
                                       const double* __restrict__ E, int m, int* codes);
__global__ void __launch_bounds__(1024) k_codes_freq_frames(const unsigned* __restrict__ keep_words, long long nwords,
                                    const unsigned long long* __restrict__ block_offsets,
                                    const double2* __restrict__ F, HalfGeom g, long long n1,
                                    const double* __restrict__ D, int m, int* codes);
// per-frame popcount of a bitmap whose frames are whole words
__global__ void k_frame_popc(const unsigned* __restrict__ words, long long words_per_frame,
                             long long nframes, unsigned long long* counts);
// sparse frequency repair inside each frame (mirror within the frame's 2-D grid)
__global__ void k_repair_freq_sparse_frames(const unsigned* __restrict__ viol_words,
                                            long long nwords, const double2* __restrict__ delta_star,
                                            const double2* __restrict__ delta_tilde, HalfGeom g,
                                            long long n1, double2* freq_cur, unsigned* esc_words);

__global__ void k_frame_gate_reset(FrameGate* fg, long long nframes);

} // namespace ffcz_gpu
