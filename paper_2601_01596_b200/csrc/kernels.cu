// Elementwise / reduction / gate kernels of the FFCz B200 engine.  See kernels.cuh for the
// reference function each one restates.
#include "kernels.cuh"

namespace ffcz_gpu {

namespace {

__device__ __forceinline__ int plane_weight(int k2, long long n2) {
    // number of FULL-spectrum entries a half entry stands for (weight 1 on the self-mirror planes)
    return (k2 == 0 || 2LL * k2 == n2) ? 1 : 2;
}

// block-wide sum, one atomic per CTA (per-warp atomics on one address serialise in L2)
__device__ __forceinline__ void block_sum_atomic(unsigned long long v, unsigned long long* dst) {
    __shared__ unsigned long long sacc[32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sacc[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        const int nw = (blockDim.x + 31) >> 5;
        v = threadIdx.x < nw ? sacc[threadIdx.x] : 0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0 && v) atomicAdd(dst, v);
    }
}

__device__ __forceinline__ void set_bit(unsigned* words, long long i) {
    atomicOr(&words[i >> 5], 1u << (i & 31));
}

// Grid-stride walk over the logical half grid h = row*H + k2 without a 64-bit division per
// element (one division per thread, then carry arithmetic).
struct HalfWalk {
    long long i, row, total, stride, dq;
    int k2, H, dr;
    __device__ __forceinline__ explicit HalfWalk(const HalfGeom& g) {
        H = g.H;
        total = g.rows * g.H;
        i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
        stride = static_cast<long long>(gridDim.x) * blockDim.x;
        row = i / H;
        k2 = static_cast<int>(i - row * H);
        dq = stride / H;
        dr = static_cast<int>(stride - dq * H);
    }
    __device__ __forceinline__ bool ok() const { return i < total; }
    // the whole block's window is still inside the grid (for ballot-based kernels)
    __device__ __forceinline__ bool block_ok() const { return i - threadIdx.x < total; }
    __device__ __forceinline__ void next() {
        i += stride;
        row += dq;
        k2 += dr;
        if (k2 >= H) {
            k2 -= H;
            ++row;
        }
    }
};

} // namespace

__global__ void k_freduce(const double2* __restrict__ spec, HalfGeom g, FreqB fb, double fscale,
                          Ctl* ctl, const int* gate) {
    if (gated(gate)) return;
    HookFReduce h{fb, fscale, ctl};
    for (HalfWalk w(g); w.ok(); w.next()) {
        const long long i = w.i, row = w.row;
        const int k2 = w.k2;
        const long long off = row * g.P + k2;
        double2 v = spec[off];
        h.post(v, off, k2);
    }
    h.finish();
}

__global__ void k_fclip(double2* spec, HalfGeom g, FreqB fb, double fscale, double2* F,
                        const int* gate) {
    if (gated(gate)) return;
    HookFClip<double> h{fb, fscale, F};
    for (HalfWalk w(g); w.ok(); w.next()) {
        const long long i = w.i, row = w.row;
        const int k2 = w.k2;
        const long long off = row * g.P + k2;
        double2 v = spec[off];
        h.pre(v, off, k2);
        spec[off] = v;
    }
}

__global__ void k_sclip(const double* __restrict__ x, double* eps, long long N, SpatialB sb,
                        double fscale, double* S, const int* gate) {
    if (gated(gate)) return;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < N;
         n += (long long)gridDim.x * blockDim.x) {
        const double xd = x[n];
        const double e = sb.at(n) * fscale;
        const double c = clamp_abs(xd, e);
        const double d = c - xd;
        if (d != 0.0) S[n] += d;
        eps[n] = c;
    }
}

template <class TI>
__global__ void k_eps0(const TI* __restrict__ orig, const TI* __restrict__ dec, double* eps,
                       long long N, SpatialB sb, double fscale, double slack, int check_original,
                       Ctl* ctl) {
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < N;
         n += (long long)gridDim.x * blockDim.x) {
        const double e = static_cast<double>(dec[n]) - static_cast<double>(orig[n]);
        eps[n] = e;
        const double E = sb.at(n);
        if (check_original && fabs(e) > E * (1.0 + 0x1p-20))
            atomicMin(&ctl->bad1, static_cast<unsigned long long>(n));
        const double Ew = E * fscale;
        if (fabs(e) > Ew * (1.0 + slack)) atomicMin(&ctl->bad2, static_cast<unsigned long long>(n));
    }
}
template __global__ void k_eps0<float>(const float*, const float*, double*, long long, SpatialB,
                                       double, double, int, Ctl*);
template __global__ void k_eps0<double>(const double*, const double*, double*, long long,
                                        SpatialB, double, double, int, Ctl*);

template <class TI>
__global__ void k_eps0_plus_s(const TI* __restrict__ orig, const TI* __restrict__ dec,
                              const double* __restrict__ S, double* out, long long N) {
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < N;
         n += (long long)gridDim.x * blockDim.x)
        out[n] = (static_cast<double>(dec[n]) - static_cast<double>(orig[n])) + S[n];
}
template __global__ void k_eps0_plus_s<float>(const float*, const float*, const double*, double*,
                                              long long);
template __global__ void k_eps0_plus_s<double>(const double*, const double*, const double*,
                                               double*, long long);

__global__ void k_frames_init(FrameCtl* fc, long long nframes, unsigned long long max_iters) {
    for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < nframes;
         f += (long long)gridDim.x * blockDim.x) {
        FrameCtl c{};
        c.max_iters = max_iters;
        fc[f] = c;
    }
}

__global__ void k_decide_frames(FrameCtl* fc, long long nframes, Ctl* ctl) {
    for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < nframes;
         f += (long long)gridDim.x * blockDim.x) {
        FrameCtl& c = fc[f];
        if (c.done) continue;
        const double peak = bitsd(c.peak_bits);
        const double ex = bitsd(c.exc_bits);
        bool fin = false;
        if (!(ex > 1e-11 * peak)) {           // projection.cpp:40, 106-111
            c.converged = 1;
            c.residual_f = 0.0;
            fin = true;
        } else if (c.passes >= c.max_iters) { // :112-116
            c.converged = 0;
            c.residual_f = ex;
            fin = true;
        } else {
            c.passes += 1;
        }
        c.peak_bits = 0;
        c.exc_bits = 0;
        if (fin) {
            c.done = 1;
            if (atomicAdd(&ctl->count_b, 1ull) + 1 == static_cast<unsigned long long>(nframes))
                ctl->done = 1;
        }
    }
}

template <class TI>
__global__ void k_eps0_frames(const TI* __restrict__ orig, const TI* __restrict__ dec, double* eps,
                              long long N, long long frameN, const double* __restrict__ E,
                              double fscale, double slack, Ctl* ctl) {
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < N;
         n += (long long)gridDim.x * blockDim.x) {
        const double e = static_cast<double>(dec[n]) - static_cast<double>(orig[n]);
        eps[n] = e;
        const double Eb = E[n / frameN];
        if (fabs(e) > Eb * (1.0 + 0x1p-20)) atomicMin(&ctl->bad1, static_cast<unsigned long long>(n));
        if (fabs(e) > Eb * fscale * (1.0 + slack))
            atomicMin(&ctl->bad2, static_cast<unsigned long long>(n));
    }
}
template __global__ void k_eps0_frames<float>(const float*, const float*, double*, long long,
                                              long long, const double*, double, double, Ctl*);
template __global__ void k_eps0_frames<double>(const double*, const double*, double*, long long,
                                               long long, const double*, double, double, Ctl*);

__global__ void k_cast_to_float(const double* __restrict__ in, float* out, long long N) {
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < N;
         n += (long long)gridDim.x * blockDim.x)
        out[n] = static_cast<float>(in[n]);
}

// Mixed policy, FP32 phase: the phase never declares convergence (its
// round-off is far above the reference's 1e-11 * peak); it hands over to the FP64 phase once
// max_excess <= tau * peak or at the iteration cap, and clips otherwise.
__global__ void k_decide32(Ctl* ctl) {
    if (ctl->switch_now) return;
    const double peak = bitsd(ctl->peak_bits);
    const double ex = bitsd(ctl->exc_bits);
    // (also when the FP32 excess stopped shrinking: FP32 round-off floor reached before tau —
    // a tau below it otherwise keeps the FP32 phase running to max_iters)
    const bool stalled = ctl->passes32 >= 1 && !(ex < ctl->ex32_prev);
    if (!(ex > ctl->tau * peak) || ctl->passes >= ctl->max_iters || stalled) {
        ctl->switch_now = 1;
        ctl->phase = 1;
    } else {
        ctl->ex32_prev = ex;
        ctl->passes += 1;
        ctl->passes32 += 1;
    }
    ctl->peak_bits = 0;
    ctl->exc_bits = 0;
}

__global__ void k_cast_to_double(const float* __restrict__ in, double* out, long long N) {
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < N;
         n += (long long)gridDim.x * blockDim.x)
        out[n] = in[n];
}

__global__ void k_decide(Ctl* ctl) {
    if (ctl->done) return;
    const double peak = bitsd(ctl->peak_bits);
    const double ex = bitsd(ctl->exc_bits);
    const double tol = 1e-11 * peak;  // projection.cpp:40
    if (!(ex > tol)) {
        ctl->converged = 1;
        ctl->residual_f = 0.0;
        ctl->done = 1;
    } else if (ctl->passes >= ctl->max_iters) {
        ctl->converged = 0;
        ctl->residual_f = ex;
        ctl->done = 1;
    } else {
        ctl->passes += 1;
    }
    ctl->peak_bits = 0;
    ctl->exc_bits = 0;
}

// Loop-control readback through mapped pinned memory: a one-warp kernel stores the control block
// straight into the host mirror, so a poll never queues behind a large D2H on the copy engines.
__global__ void k_export_ctl(const Ctl* __restrict__ ctl, Ctl* host) {
    static_assert(sizeof(Ctl) % 8 == 0, "Ctl layout");
    const volatile unsigned long long* s = reinterpret_cast<const volatile unsigned long long*>(ctl);
    volatile unsigned long long* d = reinterpret_cast<volatile unsigned long long*>(host);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(Ctl) / 8); i += blockDim.x) d[i] = s[i];
    __threadfence_system();
}

__global__ void k_ctl_init(Ctl* ctl, unsigned long long max_iters) {
    Ctl c{};
    c.max_iters = max_iters;
    c.bad1 = ~0ull;
    c.bad2 = ~0ull;
    *ctl = c;
}

__global__ void k_residual_s(const double* __restrict__ eps, long long N, SpatialB sb,
                             double fscale, Ctl* ctl) {
    double m = 0.0;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < N;
         n += (long long)gridDim.x * blockDim.x) {
        const double ex = fabs(eps[n]) - sb.at(n) * fscale;
        if (ex > m) m = ex;
    }
    block_max2_atomic(m, 0.0, &ctl->res_s_bits, nullptr);
}

__global__ void k_count_spatial(const double* __restrict__ S, long long N, Ctl* ctl) {
    unsigned long long c = 0;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < N;
         n += (long long)gridDim.x * blockDim.x)
        c += S[n] != 0.0;
    block_sum_atomic(c, &ctl->act_s);
}

__global__ void k_count_freq(const double2* __restrict__ F, HalfGeom g, Ctl* ctl) {
    unsigned long long c = 0;
    for (HalfWalk w(g); w.ok(); w.next()) {
        const long long i = w.i, row = w.row;
        const int k2 = w.k2;
        const double2 v = F[row * g.P + k2];
        if (v.x != 0.0 || v.y != 0.0) c += plane_weight(k2, g.n2);
    }
    block_sum_atomic(c, &ctl->act_f);
}

__global__ void k_gather_half(const double* __restrict__ full, double* half, HalfGeom g) {
    for (HalfWalk w(g); w.ok(); w.next()) {
        const long long i = w.i, row = w.row;
        const int k2 = w.k2;
        half[row * g.P + k2] = full[row * g.n2 + k2];
    }
}

__global__ void k_expand_full(const double2* __restrict__ half, double2* full, int ndim,
                              long long d0, long long d1, long long d2, int P) {
    // dims padded to 3-D: (d0, d1, d2) with d2 the last axis
    const long long total = d0 * d1 * d2;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < total;
         k += (long long)gridDim.x * blockDim.x) {
        const long long k2 = k % d2;
        const long long r = k / d2;
        const long long k1 = r % d1, k0 = r / d1;
        if (2 * k2 <= d2) {
            full[k] = half[r * P + k2];
        } else {
            const long long m0 = k0 ? d0 - k0 : 0, m1 = k1 ? d1 - k1 : 0;
            double2 v = half[(m0 * d1 + m1) * P + (d2 - k2)];
            v.y = -v.y;
            full[k] = v;
        }
    }
    (void)ndim;
}

// ---- FP64 gate ---------------------------------------------------------------------------------

// The spatial gate processes U grid-stride windows per trip with all loads issued first (U
// independent loads in flight per thread: 662 -> 484 us at 512^3; the same unroll made the
// frequency gate slower, 693 -> 800 us, so it keeps one window per trip).
constexpr int kGateU = 4;

__global__ void k_gate_spatial(const double* __restrict__ S, long long N, SpatialB sb, int m,
                               double* spat_cur, unsigned* keep_words, unsigned* esc_words,
                               Ctl* ctl) {
    unsigned long long nz_acc = 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const double rstep = 1.0 / (sb.g * pow2i(1 - m));
    for (long long base = blockIdx.x * (long long)blockDim.x; base < N; base += kGateU * stride) {
        double v[kGateU], E[kGateU];
#pragma unroll
        for (int u = 0; u < kGateU; ++u) {
            const long long n = base + u * stride + threadIdx.x;
            v[u] = n < N ? S[n] : 0.0;
            E[u] = n < N ? sb.at(n) : 1.0;
        }
#pragma unroll
        for (int u = 0; u < kGateU; ++u) {
            const long long n = base + u * stride + threadIdx.x;
            if (base + u * stride >= N) break;                   // warp-uniform
            bool keep = false, ovf = false;
            if (n < N) {
                const bool nz = v[u] != 0.0;
                const double step = ((E[u]) * pow2i(1 - m));       // editset.cpp:31-33
                // v / step (global E: by the hoisted reciprocal, the same bits)
                const double qv = sb.v ? v[u] / step : div_rn(v[u], step, rstep);
                ovf = nz && (fabs(qv) > kMaxIndex);               // pipeline.cpp:63-64
                keep = nz && !ovf;
                double cur = 0.0;
                if (keep) {
                    const long long q = llround(qv);              // editset.cpp:76-84
                    cur = static_cast<double>(static_cast<int>(q)) * step;  // editset.cpp:102
                } else if (ovf) {
                    cur = v[u];
                }
                spat_cur[n] = cur;
            }
            const unsigned bk = __ballot_sync(0xffffffffu, keep);
            const unsigned be = __ballot_sync(0xffffffffu, ovf);
            if ((threadIdx.x & 31) == 0 && n < N) {
                keep_words[n >> 5] = bk;
                esc_words[n >> 5] = be;
            }
            if ((threadIdx.x & 31) == 0) nz_acc += __popc(bk) + __popc(be);
        }
    }
    block_sum_atomic(nz_acc, &ctl->act_s);
}

__global__ void k_gate_freq(const double2* __restrict__ F, HalfGeom g, FreqB fb, int m,
                            double2* freq_cur, unsigned* keep_words, unsigned* esc_words,
                            Ctl* ctl) {
    unsigned long long nz_acc = 0;
    const long long total = g.rows * g.H;
    const double rD = 1.0 / fb.g;  // (global Delta: the reciprocal of div_rn)
    for (HalfWalk hw(g); hw.block_ok(); hw.next()) {
        const long long h = hw.i;
        bool keep = false, ovf = false;
        int w = 0;
        if (h < total) {
            const long long row = hw.row;
            const int k2 = hw.k2;
            const long long off = row * g.P + k2;
            const double2 v = F[off];
            const bool nz = v.x != 0.0 || v.y != 0.0;
            const double2 db = fb.at2(off);
            const double sre = ((db.x) * pow2i(1 - m));   // editset.cpp:35-41
            const double sim = ((db.y) * pow2i(1 - m));
            // v / step == (v / Delta) 2^(m-1) bit for bit (step = Delta 2^(1-m); scaling by a
            // power of two commutes with rounding): one division per lane instead of two
            const double qx = ((fb.re ? v.x / db.x : div_rn(v.x, db.x, rD)) * pow2i(m - 1)),
                         qy = ((fb.re ? v.y / db.y : div_rn(v.y, db.y, rD)) * pow2i(m - 1));
            ovf = nz && (fabs(qx) > kMaxIndex || fabs(qy) > kMaxIndex);  // :68-69
            keep = nz && !ovf;
            double2 cur = make_double2(0.0, 0.0);
            if (keep) {
                cur.x = static_cast<double>(static_cast<int>(llround(qx))) * sre;
                cur.y = static_cast<double>(static_cast<int>(llround(qy))) * sim;
            } else if (ovf) {
                cur = v;
            }
            freq_cur[off] = cur;
            if (nz) w = plane_weight(k2, g.n2);
        }
        const unsigned bk = __ballot_sync(0xffffffffu, keep);
        const unsigned be = __ballot_sync(0xffffffffu, ovf);
        if ((threadIdx.x & 31) == 0 && h < total) {
            keep_words[h >> 5] = bk;
            esc_words[h >> 5] = be;
        }
        nz_acc += w;
    }
    block_sum_atomic(nz_acc, &ctl->act_f);
}

// k_gate_freq + k_codes_freq_bits in ONE pass (single-pass compaction with decoupled look-back):
// each CTA takes the next tile of kGcTile half entries by ticket (so every predecessor tile is
// already resident), quantises, writes flags / freq_cur, ranks its kept entries in ascending h,
// publishes its count, looks back for its exclusive offset, and stores the int32 code pairs —
// F and Delta are read once instead of twice.  Same values as the two-pass kernels.
constexpr int kGcItems = 16, kGcThreads = 256, kGcTile = kGcItems * kGcThreads;
constexpr unsigned long long kGcAgg = 1ull << 62, kGcIncl = 2ull << 62, kGcMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(kGcThreads) k_gate_codes_freq(
    const double2* __restrict__ F, HalfGeom g, FreqB fb, int m, double2* freq_cur,
    unsigned* keep_words, unsigned* esc_words, int* codes, unsigned long long* tile_status,
    unsigned* tile_ticket, long long ntiles, Ctl* ctl) {
    __shared__ long long s_tile;
    __shared__ unsigned s_cnt[kGcItems][kGcThreads / 32];
    __shared__ unsigned long long s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ticket, 1u);
    __syncthreads();
    const long long t = s_tile;
    const long long total = g.rows * g.H;
    const long long base = t * kGcTile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned kmask[kGcItems];
    int2 code[kGcItems];
    unsigned long long nz_acc = 0;
#pragma unroll
    for (int u = 0; u < kGcItems; ++u) {
        const long long h = base + u * kGcThreads + threadIdx.x;
        bool keep = false, ovf = false;
        code[u] = make_int2(0, 0);
        if (h < total) {
            long long q = static_cast<long long>(static_cast<double>(h) * g.invH);
            long long r = h - q * g.H;
            if (r < 0) { --q; r += g.H; } else if (r >= g.H) { ++q; r -= g.H; }
            const long long off = q * g.P + r;
            const double2 v = F[off];
            const bool nz = v.x != 0.0 || v.y != 0.0;
            const double2 db = fb.at2(off);
            const double sre = ((db.x) * pow2i(1 - m));   // editset.cpp:35-41
            const double sim = ((db.y) * pow2i(1 - m));
            ovf = nz && (fabs(v.x) / sre > kMaxIndex || fabs(v.y) / sim > kMaxIndex);  // :68-69
            keep = nz && !ovf;
            double2 cur = make_double2(0.0, 0.0);
            if (keep) {
                code[u] = make_int2(static_cast<int>(llround(v.x / sre)),
                                    static_cast<int>(llround(v.y / sim)));
                cur.x = static_cast<double>(code[u].x) * sre;
                cur.y = static_cast<double>(code[u].y) * sim;
            } else if (ovf) {
                cur = v;
            }
            freq_cur[off] = cur;
            if (nz) nz_acc += plane_weight(static_cast<int>(r), g.n2);
        }
        const unsigned bk = __ballot_sync(0xffffffffu, keep);
        const unsigned be = __ballot_sync(0xffffffffu, ovf);
        if (lane == 0 && h < total) {
            keep_words[h >> 5] = bk;
            esc_words[h >> 5] = be;
            s_cnt[u][warp] = __popc(bk);
        } else if (lane == 0) {
            s_cnt[u][warp] = 0;
        }
        kmask[u] = bk;
    }
    __syncthreads();
    // tile-local exclusive offsets in ascending h: (item u, warp w) in u-major order
    if (threadIdx.x == 0) {
        unsigned acc = 0;
        for (int u = 0; u < kGcItems; ++u)
            for (int w = 0; w < kGcThreads / 32; ++w) {
                const unsigned c = s_cnt[u][w];
                s_cnt[u][w] = acc;
                acc += c;
            }
        s_prefix = acc;  // the tile's aggregate, until the look-back below replaces it
        atomicExch(&tile_status[t], (t == 0 ? kGcIncl : kGcAgg) | acc);
    }
    __syncthreads();
    if (warp == 0) {
        // warp-parallel look-back over 32 predecessors at a time (decoupled look-back)
        const unsigned long long agg = s_prefix;
        unsigned long long excl = 0;
        long long hi = t - 1;
        while (hi >= 0) {
            const long long i = hi - lane;
            unsigned long long st = kGcIncl;  // lanes past tile 0: an inclusive zero
            if (i >= 0) {
                do {
                    st = *reinterpret_cast<volatile unsigned long long*>(&tile_status[i]);
                } while ((st >> 62) == 0);
            }
            const unsigned incl = __ballot_sync(0xffffffffu, (st >> 62) == 2);
            // nearest inclusive predecessor: the lowest lane with one; sum lanes up to it
            const int stop = incl ? __ffs(incl) - 1 : 31;
            unsigned long long v = lane <= stop ? (st & kGcMask) : 0;
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            excl += v;
            if (incl) break;
            hi -= 32;
        }
        if (lane == 0) {
            if (t > 0) {
                __threadfence();
                atomicExch(&tile_status[t], kGcIncl | (excl + agg));
            }
            if (t == ntiles - 1) ctl->count_b = excl + agg;
            s_prefix = excl;
        }
    }
    __syncthreads();
    const unsigned long long p0 = s_prefix;
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int u = 0; u < kGcItems; ++u)
        if (kmask[u] >> lane & 1u)
            reinterpret_cast<int2*>(codes)[p0 + s_cnt[u][warp] + __popc(kmask[u] & lt)] = code[u];
    block_sum_atomic(nz_acc, &ctl->act_f);
}

__global__ void k_popc_blocks(const unsigned* __restrict__ words, long long nwords,
                              unsigned long long* block_counts) {
    __shared__ unsigned long long s[32];
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    unsigned long long c = i < nwords ? __popc(words[i]) : 0;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
        block_counts[blockIdx.x] = t;
    }
}

// single-CTA exclusive scan (in place) with running carry; *total = sum
__global__ void k_scan_blocks(unsigned long long* counts, long long nblocks,
                              unsigned long long* total) {
    __shared__ unsigned long long s[1024];
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (long long base = 0; base < nblocks; base += blockDim.x) {
        const long long i = base + threadIdx.x;
        const unsigned long long v = i < nblocks ? counts[i] : 0;
        s[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < (int)blockDim.x; o <<= 1) {
            const unsigned long long a = threadIdx.x >= (unsigned)o ? s[threadIdx.x - o] : 0;
            __syncthreads();
            s[threadIdx.x] += a;
            __syncthreads();
        }
        if (i < nblocks) counts[i] = carry + s[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += s[threadIdx.x];
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void k_compact(const unsigned* __restrict__ words, long long nwords,
                          const unsigned long long* __restrict__ block_offsets,
                          unsigned long long* out_idx) {
    __shared__ unsigned s[1024];
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const unsigned w = i < nwords ? words[i] : 0u;
    const unsigned c = __popc(w);
    s[threadIdx.x] = c;
    __syncthreads();
    for (int o = 1; o < (int)blockDim.x; o <<= 1) {
        const unsigned a = threadIdx.x >= (unsigned)o ? s[threadIdx.x - o] : 0u;
        __syncthreads();
        s[threadIdx.x] += a;
        __syncthreads();
    }
    unsigned long long pos = block_offsets[blockIdx.x] + s[threadIdx.x] - c;
    unsigned rem = w;
    while (rem) {
        const int b = __ffs(rem) - 1;
        rem &= rem - 1;
        out_idx[pos++] = static_cast<unsigned long long>(i) * 32 + b;
    }
}

__global__ void k_codes_spatial(const unsigned long long* __restrict__ idx, long long n,
                                const double* __restrict__ S, SpatialB sb, int m, int* codes) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long k = idx[i];
        const double step = ((sb.at(k)) * pow2i(1 - m));
        codes[i] = static_cast<int>(llround(S[k] / step));
    }
}

__global__ void k_codes_freq(const unsigned long long* __restrict__ idx, long long n,
                             const double2* __restrict__ F, HalfGeom g, FreqB fb, int m,
                             int* codes) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long off = g.offset_of(static_cast<long long>(idx[i]));
        const double2 v = F[off];
        const double sre = ((fb.re_at(off)) * pow2i(1 - m));
        const double sim = ((fb.im_at(off)) * pow2i(1 - m));
        codes[2 * i] = static_cast<int>(llround(v.x / sre));
        codes[2 * i + 1] = static_cast<int>(llround(v.y / sim));
    }
}

// Codes straight from the keep bitmap (no index list): CTA b owns words [1024 b, 1024 b + 1024)
// = the block of k_popc_blocks, whose exclusive offsets k_scan_blocks left in block_offsets.  A
// CTA-wide scan of the per-word popcounts gives every word's output position; warp j then walks
// words 32 j .. 32 j + 31 with lane l on element 32 w + l, so the F / S / bound loads are
// coalesced and codes land in ascending index order (editset.cpp:86-119).
namespace {
template <class Emit>
__device__ __forceinline__ void codes_from_bits(const unsigned* __restrict__ words, long long nwords,
                                                const unsigned long long* __restrict__ block_offsets,
                                                Emit&& emit) {
    __shared__ unsigned s[1024];
    __shared__ unsigned sw[1024];
    const long long wbase = blockIdx.x * 1024LL;
    const long long wi = wbase + threadIdx.x;
    const unsigned w = wi < nwords ? words[wi] : 0u;
    const unsigned c = __popc(w);
    sw[threadIdx.x] = w;
    // block-wide inclusive scan of popcounts: warp scans + scan of warp totals
    unsigned v = c;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned a = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += a;
    }
    __shared__ unsigned wsum[32];
    if (lane == 31) wsum[warp] = v;
    __syncthreads();
    if (warp == 0) {
        unsigned t = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned a = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += a;
        }
        wsum[lane] = t;
    }
    __syncthreads();
    s[threadIdx.x] = v - c + (warp ? wsum[warp - 1] : 0u);  // exclusive prefix of this word
    __syncthreads();
    const unsigned long long boff = block_offsets[blockIdx.x];
    const unsigned lt = (1u << lane) - 1u;
    if constexpr (requires { emit.batched; }) {
        // four words per step: the emitter issues all four elements' loads before any store
        for (int k0 = 0; k0 < 32; k0 += 4) {
            long long nn[4];
            unsigned long long pp[4];
            bool act[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int wl = warp * 32 + k0 + u;
                const long long wg = wbase + wl;
                const unsigned word = wg < nwords ? sw[wl] : 0u;
                act[u] = (word >> lane) & 1u;
                nn[u] = wg * 32 + lane;
                pp[u] = boff + s[wl] + __popc(word & lt);
            }
            emit(nn, pp, act);
        }
    } else {
        for (int k = 0; k < 32; ++k) {
            const int wl = warp * 32 + k;
            const long long wg = wbase + wl;
            if (wg >= nwords) break;
            const unsigned word = sw[wl];
            if (!word) continue;
            if (word >> lane & 1u) emit(wg * 32 + lane, boff + s[wl] + __popc(word & lt));
        }
    }
}

// batched emitters of the two code kernels (loads of four elements first, then the stores)
struct EmitCodesS {
    static constexpr bool batched = true;
    const double* __restrict__ S;
    SpatialB sb;
    int m;
    int* codes;
    __device__ __forceinline__ void operator()(const long long (&n)[4],
                                               const unsigned long long (&pos)[4],
                                               const bool (&act)[4]) const {
        double v[4], e[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            v[u] = act[u] ? S[n[u]] : 0.0;
            e[u] = act[u] ? sb.at(n[u]) : 1.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (act[u]) {
                const double step = (e[u]) * pow2i(1 - m);
                codes[pos[u]] = static_cast<int>(
                    llround(sb.v ? v[u] / step : div_rn(v[u], step, 1.0 / (sb.g * pow2i(1 - m)))));
            }
    }
};

struct EmitCodesF {
    static constexpr bool batched = true;
    const double2* __restrict__ F;
    HalfGeom g;
    FreqB fb;
    int m;
    int* codes;
    __device__ __forceinline__ void operator()(const long long (&h)[4],
                                               const unsigned long long (&pos)[4],
                                               const bool (&act)[4]) const {
        double2 v[4], d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long off = act[u] ? g.offset_of(h[u]) : 0;
            v[u] = act[u] ? F[off] : make_double2(0.0, 0.0);
            d[u] = act[u] ? fb.at2(off) : make_double2(1.0, 1.0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (act[u])
                reinterpret_cast<int2*>(codes)[pos[u]] =
                    fb.re ? make_int2(static_cast<int>(llround(((v[u].x / d[u].x) * pow2i(m - 1)))),
                                      static_cast<int>(llround(((v[u].y / d[u].y) * pow2i(m - 1)))))
                          : make_int2(static_cast<int>(llround(div_rn(v[u].x, fb.g, 1.0 / fb.g) * pow2i(m - 1))),
                                      static_cast<int>(llround(div_rn(v[u].y, fb.g, 1.0 / fb.g) * pow2i(m - 1))));
    }
};
} // namespace

__global__ void __launch_bounds__(1024) k_codes_spatial_bits(const unsigned* __restrict__ keep_words, long long nwords,
                                     const unsigned long long* __restrict__ block_offsets,
                                     const double* __restrict__ S, SpatialB sb, int m, int* codes) {
    codes_from_bits(keep_words, nwords, block_offsets, EmitCodesS{S, sb, m, codes});
}

__global__ void __launch_bounds__(1024) k_codes_freq_bits(const unsigned* __restrict__ keep_words, long long nwords,
                                  const unsigned long long* __restrict__ block_offsets,
                                  const double2* __restrict__ F, HalfGeom g, FreqB fb, int m,
                                  int* codes) {
    codes_from_bits(keep_words, nwords, block_offsets, EmitCodesF{F, g, fb, m, codes});
}

// dequantize_edits (editset.cpp:106-133) scattered to the flagged positions (expand_edits,
// archive.cpp:227-260): dense arrays must be zero on entry
__global__ void k_dequant_spatial_bits(const unsigned* __restrict__ keep_words, long long nwords,
                                       const unsigned long long* __restrict__ block_offsets,
                                       const int* __restrict__ codes, SpatialB sb, int m,
                                       double* spat) {
    codes_from_bits(keep_words, nwords, block_offsets, [&](long long n, unsigned long long pos) {
        spat[n] = static_cast<double>(codes[pos]) * ((sb.at(n)) * pow2i(1 - m));
    });
}

__global__ void __launch_bounds__(1024) k_dequant_freq_bits(const unsigned* __restrict__ keep_words, long long nwords,
                                    const unsigned long long* __restrict__ block_offsets,
                                    const int* __restrict__ codes, HalfGeom g, FreqB fb, int m,
                                    double2* freq) {
    codes_from_bits(keep_words, nwords, block_offsets, [&](long long h, unsigned long long pos) {
        const long long off = g.offset_of(h);
        const double2 d = fb.at2(off);
        const int2 c = reinterpret_cast<const int2*>(codes)[pos];
        freq[off] = make_double2(static_cast<double>(c.x) * ((d.x) * pow2i(1 - m)),
                                 static_cast<double>(c.y) * ((d.y) * pow2i(1 - m)));
    });
}

__global__ void k_scatter_escapes(const EscapeRec* __restrict__ recs, long long n, double* spat,
                                  double2* freq, HalfGeom g) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const EscapeRec e = recs[i];
        if (e.frequency) freq[g.offset_of(static_cast<long long>(e.index))] = make_double2(e.re, e.im);
        else spat[e.index] = e.re;
    }
}

// apply_edits (archive.cpp:262-273): decompressed + spatial + Re(IFFT(frequency))
template <class TI>
__global__ void k_apply_sum(const TI* __restrict__ dec, const double* __restrict__ spat,
                            const double* __restrict__ fpart, double* out, long long N) {
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < N;
         n += (long long)gridDim.x * blockDim.x)
        out[n] = static_cast<double>(dec[n]) + spat[n] + fpart[n];
}
template __global__ void k_apply_sum<float>(const float*, const double*, const double*, double*,
                                            long long);
template __global__ void k_apply_sum<double>(const double*, const double*, const double*, double*,
                                             long long);

template <class TI>
__global__ void k_repair_spatial(const TI* __restrict__ orig, const TI* __restrict__ dec,
                                 const double* __restrict__ fpart, const double* __restrict__ final_eps,
                                 long long N, SpatialB sb, double* spat_cur, double* eps_tilde,
                                 unsigned* esc_words, Ctl* ctl) {
    bool dirty = false;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < N;
         n += (long long)gridDim.x * blockDim.x) {
        const double e0 = static_cast<double>(dec[n]) - static_cast<double>(orig[n]);
        const double sc = spat_cur[n];
        const double et = e0 + sc + fpart[n];                       // pipeline.cpp:134-136
        eps_tilde[n] = et;
        if (fabs(et) > sb.at(n)) {                                  // pipeline.cpp:154-160
            dirty = true;
            spat_cur[n] = sc + (final_eps[n] - et);
            set_bit(esc_words, n);
        }
    }
    if (__any_sync(0xffffffffu, dirty) && (threadIdx.x & 31) == 0) ctl->dirty = 1;
}
template __global__ void k_repair_spatial<float>(const float*, const float*, const double*,
                                                 const double*, long long, SpatialB, double*,
                                                 double*, unsigned*, Ctl*);
template __global__ void k_repair_spatial<double>(const double*, const double*, const double*,
                                                  const double*, long long, SpatialB, double*,
                                                  double*, unsigned*, Ctl*);

__global__ void k_repair_freq(const double2* __restrict__ delta_star,
                              const double2* __restrict__ delta_tilde, HalfGeom g, int ndim,
                              long long d0, long long d1, FreqB fb, double2* freq_cur,
                              unsigned* esc_words, Ctl* ctl) {
    // pipeline.cpp:140-153; half rows are (k0, k1) of a 3-D grid padded as (d0, d1)
    bool dirty = false;
    for (HalfWalk w(g); w.ok(); w.next()) {
        const long long h = w.i, row = w.row;
        const int k2 = w.k2;
        auto violates = [&](long long r) {
            const long long off = r * g.P + k2;
            const double2 d = delta_tilde[off];
            return fabs(d.x) > fb.re_at(off) || fabs(d.y) > fb.im_at(off);
        };
        auto repaired = [&](long long r) {
            const long long off = r * g.P + k2;
            const double2 c = freq_cur[off], s = delta_star[off], t = delta_tilde[off];
            return make_double2(c.x + (s.x - t.x), c.y + (s.y - t.y));
        };
        const bool plane = (k2 == 0) || (2LL * k2 == g.n2);
        long long mrow = row;
        if (plane) {
            const long long k1 = row % d1, k0 = row / d1;
            mrow = (k0 ? d0 - k0 : 0) * d1 + (k1 ? d1 - k1 : 0);
        }
        if (mrow == row) {
            if (violates(row)) {
                dirty = true;
                freq_cur[row * g.P + k2] = repaired(row);
                set_bit(esc_words, h);
            }
        } else if (row < mrow) {
            // the pair (h, hm) is owned by its smaller index; the larger index wins when both
            // violate, because the reference visits it last (pipeline.cpp:141-152)
            const long long hm = mrow * g.H + k2;
            const bool va = violates(row), vb = violates(mrow);
            if (va || vb) {
                dirty = true;
                double2 r = vb ? repaired(mrow) : repaired(row);
                double2 rc = make_double2(r.x, -r.y);
                if (vb) {
                    freq_cur[mrow * g.P + k2] = r;
                    freq_cur[row * g.P + k2] = rc;
                } else {
                    freq_cur[row * g.P + k2] = r;
                    freq_cur[mrow * g.P + k2] = rc;
                }
                set_bit(esc_words, h);
                set_bit(esc_words, hm);
            }
        }
    }
    (void)ndim;
    if (__any_sync(0xffffffffu, dirty) && (threadIdx.x & 31) == 0) ctl->dirty = 1;
}

template <class TI>
__global__ void k_verify_spatial(const TI* __restrict__ orig, const TI* __restrict__ dec,
                                 const double* __restrict__ spat_cur,
                                 const double* __restrict__ fpart, long long N, SpatialB sb,
                                 double* corrected, double* eps_v, Ctl* ctl) {
    double m = 0.0;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < N;
         n += (long long)gridDim.x * blockDim.x) {
        const double c = static_cast<double>(dec[n]) + spat_cur[n] + fpart[n];  // archive.cpp:271
        if (corrected) corrected[n] = c;
        const double e = c - static_cast<double>(orig[n]);                      // archive.cpp:284
        eps_v[n] = e;
        const double ex = fabs(e) - sb.at(n);
        if (ex > 0.0 && ex > m) m = ex;                                         // :285-286
    }
    block_max2_atomic(m, 0.0, &ctl->vs_bits, nullptr);
}
template __global__ void k_verify_spatial<float>(const float*, const float*, const double*,
                                                 const double*, long long, SpatialB, double*,
                                                 double*, Ctl*);
template __global__ void k_verify_spatial<double>(const double*, const double*, const double*,
                                                  const double*, long long, SpatialB, double*,
                                                  double*, Ctl*);

__global__ void k_verify_freq(const double2* __restrict__ delta, HalfGeom g, FreqB fb, Ctl* ctl) {
    double m = 0.0;
    for (HalfWalk w(g); w.ok(); w.next()) {
        const long long off = w.row * g.P + w.k2;
        const double2 d = delta[off];
        const double ex = fmax(fabs(d.x) - fb.re_at(off), fabs(d.y) - fb.im_at(off));  // :290-292
        if (ex > 0.0 && ex > m) m = ex;
    }
    block_max2_atomic(m, 0.0, &ctl->vf_bits, nullptr);
}

__global__ void k_gather_escapes_s(const unsigned long long* __restrict__ idx, long long n,
                                   const double* __restrict__ spat_cur, double* out_re) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out_re[i] = spat_cur[idx[i]];
}

__global__ void k_gather_escapes_f(const unsigned long long* __restrict__ idx, long long n,
                                   const double2* __restrict__ freq_cur, HalfGeom g, double2* out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        out[i] = freq_cur[g.offset_of(static_cast<long long>(idx[i]))];
    }
}

__global__ void k_split_hermitian(const double2* __restrict__ full, double2* Hh, double2* Ah,
                                  HalfGeom g, long long d0, long long d1) {
    // Re(ifft X) = C2R(H), Im(ifft X) = C2R(A) with H = (X + conj X_m)/2, A = (X - conj X_m)/(2i)
    for (HalfWalk w(g); w.ok(); w.next()) {
        const long long i = w.i, row = w.row;
        const int k2 = w.k2;
        const long long k1 = row % d1, k0 = row / d1;
        const long long mrow = (k0 ? d0 - k0 : 0) * d1 + (k1 ? d1 - k1 : 0);
        const long long mk2 = k2 ? g.n2 - k2 : 0;
        const double2 x = full[row * g.n2 + k2];
        const double2 xm = full[mrow * g.n2 + mk2];
        Hh[row * g.P + k2] = make_double2(0.5 * (x.x + xm.x), 0.5 * (x.y - xm.y));
        const double dx = x.x - xm.x, dy = x.y + xm.y;
        Ah[row * g.P + k2] = make_double2(0.5 * dy, -0.5 * dx);
    }
}

__global__ void k_maxabs(const double* __restrict__ x, long long N, unsigned long long* out) {
    double m = 0.0;
    for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < N;
         n += (long long)gridDim.x * blockDim.x)
        m = fmax(m, fabs(x[n]));
    block_max2_atomic(m, 0.0, out, nullptr);
}

__global__ void k_repair_freq_sparse(const unsigned* __restrict__ viol_words, long long nwords,
                                     const double2* __restrict__ delta_star,
                                     const double2* __restrict__ delta_tilde, HalfGeom g,
                                     long long d0, long long d1, double2* freq_cur,
                                     unsigned* esc_words) {
    for (long long wi = blockIdx.x * (long long)blockDim.x + threadIdx.x; wi < nwords;
         wi += (long long)gridDim.x * blockDim.x) {
        unsigned bits = viol_words[wi];
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const long long off = wi * 32 + b;
            const long long row = off / g.P;
            const int k2 = static_cast<int>(off - row * g.P);
            auto repaired = [&](long long o) {
                const double2 c = freq_cur[o], s = delta_star[o], t = delta_tilde[o];
                return make_double2(c.x + (s.x - t.x), c.y + (s.y - t.y));
            };
            const bool plane = (k2 == 0) || (2LL * k2 == g.n2);
            long long mrow = row;
            if (plane) {
                const long long k1 = row % d1, k0 = row / d1;
                mrow = (k0 ? d0 - k0 : 0) * d1 + (k1 ? d1 - k1 : 0);
            }
            if (mrow == row) {
                freq_cur[off] = repaired(off);
                set_bit(esc_words, row * g.H + k2);
                continue;
            }
            // conjugate pair inside the half grid: the reference visits indices in ascending
            // order, so the larger index's repair wins when both violate (pipeline.cpp:141-152)
            const long long moff = mrow * g.P + k2;
            const bool mviol = (viol_words[moff >> 5] >> (moff & 31)) & 1u;
            if (row > mrow && mviol) continue;  // the smaller partner handles the pair
            const long long lo = row < mrow ? off : moff, hi = row < mrow ? moff : off;
            const bool hi_viol = row < mrow ? mviol : true;
            double2 r = hi_viol ? repaired(hi) : repaired(lo);
            const double2 rc = make_double2(r.x, -r.y);
            if (hi_viol) {
                freq_cur[hi] = r;
                freq_cur[lo] = rc;
            } else {
                freq_cur[lo] = r;
                freq_cur[hi] = rc;
            }
            set_bit(esc_words, row * g.H + k2);
            set_bit(esc_words, mrow * g.H + k2);
        }
    }
}

__global__ void k_escape_records_s(const unsigned long long* __restrict__ idx, long long n,
                                   const double* __restrict__ spat_cur, EscapeRec* out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long k = idx[i];
        out[i] = EscapeRec{0, 0, k, spat_cur[k], 0.0};
    }
}

__global__ void k_escape_records_f(const unsigned long long* __restrict__ idx, long long n,
                                   const double2* __restrict__ freq_cur, HalfGeom g, EscapeRec* out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long h = idx[i];
        const double2 v = freq_cur[g.offset_of(static_cast<long long>(h))];
        out[i] = EscapeRec{1, 0, h, v.x, v.y};
    }
}

// ---- batched frames: gate kernels over the stack -------------------------------------------------

// warp-aggregated per-frame count (a warp's 32 consecutive indices never straddle a frame: frame
// sizes are multiples of 32)
__device__ __forceinline__ void frame_count_add(unsigned long long* dst, unsigned v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, static_cast<unsigned long long>(v));
}

__global__ void k_gate_spatial_frames(const double* __restrict__ S, long long N, long long frameN,
                                      const double* __restrict__ E, int m, double* spat_cur,
                                      unsigned* keep_words, unsigned* esc_words, FrameGate* fg) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long base = blockIdx.x * (long long)blockDim.x; base < N; base += stride) {
        const long long n = base + threadIdx.x;
        bool keep = false, ovf = false;
        const long long f = (base + (threadIdx.x & ~31)) / frameN;
        if (n < N) {
            const double v = S[n];
            const bool nz = v != 0.0;
            const double step = ((E[f]) * pow2i(1 - m));           // editset.cpp:31-33
            ovf = nz && (fabs(v) / step > kMaxIndex);            // pipeline.cpp:63-64
            keep = nz && !ovf;
            double cur = 0.0;
            if (keep) cur = static_cast<double>(static_cast<int>(llround(v / step))) * step;
            else if (ovf) cur = v;
            spat_cur[n] = cur;
        }
        const unsigned bk = __ballot_sync(0xffffffffu, keep);
        const unsigned be = __ballot_sync(0xffffffffu, ovf);
        if ((threadIdx.x & 31) == 0 && n < N) {
            keep_words[n >> 5] = bk;
            esc_words[n >> 5] = be;
        }
        if (n - (threadIdx.x & 31) < N)
            frame_count_add(&fg[f].act_s, (threadIdx.x & 31) ? 0u : __popc(bk) + __popc(be));
    }
}

__global__ void k_gate_freq_frames(const double2* __restrict__ F, HalfGeom g, long long n1,
                                   const double* __restrict__ D, int m, double2* freq_cur,
                                   unsigned* keep_words, unsigned* esc_words, FrameGate* fg) {
    const long long total = g.rows * g.H;
    for (HalfWalk hw(g); hw.block_ok(); hw.next()) {
        const long long h = hw.i;
        bool keep = false, ovf = false;
        unsigned wt = 0;
        const long long frame = hw.row / n1;
        if (h < total) {
            const int k2 = hw.k2;
            const long long off = hw.row * g.P + k2;
            const double2 v = F[off];
            const bool nz = v.x != 0.0 || v.y != 0.0;
            const double st = ((D[frame]) * pow2i(1 - m));          // editset.cpp:35-41
            ovf = nz && (fabs(v.x) / st > kMaxIndex || fabs(v.y) / st > kMaxIndex);
            keep = nz && !ovf;
            double2 cur = make_double2(0.0, 0.0);
            if (keep) {
                cur.x = static_cast<double>(static_cast<int>(llround(v.x / st))) * st;
                cur.y = static_cast<double>(static_cast<int>(llround(v.y / st))) * st;
            } else if (ovf) {
                cur = v;
            }
            freq_cur[off] = cur;
            if (nz) wt = plane_weight(k2, g.n2);
        }
        const unsigned bk = __ballot_sync(0xffffffffu, keep);
        const unsigned be = __ballot_sync(0xffffffffu, ovf);
        if ((threadIdx.x & 31) == 0 && h < total) {
            keep_words[h >> 5] = bk;
            esc_words[h >> 5] = be;
        }
        // the warp's 32 consecutive h share a frame (n1 * H is a multiple of 32)
        const long long wframe = __shfl_sync(0xffffffffu, frame, 0);
        if (h - (threadIdx.x & 31) < total) frame_count_add(&fg[wframe].act_f, wt);
    }
}

__global__ void k_codes_spatial_frames(const unsigned* __restrict__ keep_words, long long nwords,
                                       const unsigned long long* __restrict__ block_offsets,
                                       const double* __restrict__ S, long long frameN,
                                       const double* __restrict__ E, int m, int* codes) {
    codes_from_bits(keep_words, nwords, block_offsets, [&](long long n, unsigned long long pos) {
        const double step = ((E[n / frameN]) * pow2i(1 - m));
        codes[pos] = static_cast<int>(llround(S[n] / step));
    });
}

__global__ void __launch_bounds__(1024) k_codes_freq_frames(const unsigned* __restrict__ keep_words, long long nwords,
                                    const unsigned long long* __restrict__ block_offsets,
                                    const double2* __restrict__ F, HalfGeom g, long long n1,
                                    const double* __restrict__ D, int m, int* codes) {
    codes_from_bits(keep_words, nwords, block_offsets, [&](long long h, unsigned long long pos) {
        const long long off = g.offset_of(h);
        const double2 v = F[off];
        const double st = ((D[(off / g.P) / n1]) * pow2i(1 - m));
        reinterpret_cast<int2*>(codes)[pos] = make_int2(static_cast<int>(llround(v.x / st)),
                                                        static_cast<int>(llround(v.y / st)));
    });
}

__global__ void k_frame_popc(const unsigned* __restrict__ words, long long words_per_frame,
                             long long nframes, unsigned long long* counts) {
    for (long long f = blockIdx.x; f < nframes; f += gridDim.x) {
        unsigned long long c = 0;
        const unsigned* w = words + f * words_per_frame;
        for (long long i = threadIdx.x; i < words_per_frame; i += blockDim.x) c += __popc(w[i]);
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        __shared__ unsigned long long sc[32];
        if ((threadIdx.x & 31) == 0) sc[threadIdx.x >> 5] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int k = 0; k < (blockDim.x + 31) / 32; ++k) t += sc[k];
            counts[f] = t;
        }
        __syncthreads();
    }
}

// k_repair_freq_sparse with the conjugate mirror taken inside each frame's n1 x n2 grid
__global__ void k_repair_freq_sparse_frames(const unsigned* __restrict__ viol_words,
                                            long long nwords, const double2* __restrict__ delta_star,
                                            const double2* __restrict__ delta_tilde, HalfGeom g,
                                            long long n1, double2* freq_cur, unsigned* esc_words) {
    for (long long wi = blockIdx.x * (long long)blockDim.x + threadIdx.x; wi < nwords;
         wi += (long long)gridDim.x * blockDim.x) {
        unsigned bits = viol_words[wi];
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const long long off = wi * 32 + b;
            const long long row = off / g.P;
            const int k2 = static_cast<int>(off - row * g.P);
            auto repaired = [&](long long o) {
                const double2 c = freq_cur[o], s = delta_star[o], t = delta_tilde[o];
                return make_double2(c.x + (s.x - t.x), c.y + (s.y - t.y));
            };
            const bool plane = (k2 == 0) || (2LL * k2 == g.n2);
            long long mrow = row;
            if (plane) {
                const long long fr = row / n1, k1 = row - fr * n1;
                mrow = fr * n1 + (k1 ? n1 - k1 : 0);
            }
            if (mrow == row) {
                freq_cur[off] = repaired(off);
                set_bit(esc_words, row * g.H + k2);
                continue;
            }
            const long long moff = mrow * g.P + k2;
            const bool mviol = (viol_words[moff >> 5] >> (moff & 31)) & 1u;
            if (row > mrow && mviol) continue;  // the smaller partner handles the pair
            const long long lo = row < mrow ? off : moff, hi = row < mrow ? moff : off;
            const bool hi_viol = row < mrow ? mviol : true;
            double2 r = hi_viol ? repaired(hi) : repaired(lo);
            const double2 rc = make_double2(r.x, -r.y);
            if (hi_viol) {
                freq_cur[hi] = r;
                freq_cur[lo] = rc;
            } else {
                freq_cur[lo] = r;
                freq_cur[hi] = rc;
            }
            set_bit(esc_words, row * g.H + k2);
            set_bit(esc_words, mrow * g.H + k2);
        }
    }
}

__global__ void k_frame_gate_reset(FrameGate* fg, long long nframes) {
    for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < nframes;
         f += (long long)gridDim.x * blockDim.x) {
        fg[f].vs_bits = 0;
        fg[f].vf_bits = 0;
        fg[f].dirty = 0;
        fg[f].dirty_s = 0;
    }
}

} // namespace ffcz_gpu
