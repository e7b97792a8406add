// Host orchestration of the FFCz correction step on one B200 + the C-ABI (include/ffcz_cuda.h).
//
// Control flow restates ffcz::correct (/root/reference/proj/core/src/pipeline.cpp:26-178) and
// ffcz::alternating_projection (/root/reference/proj/core/src/projection.cpp:81-142):
//   eps0 + preconditions -> device-resident projection loop -> FP64 gate (compaction,
//   quantisation, overflow escapes, escape repair, verify) -> optional host archive.
// The projection loop is enqueued speculatively in chunks; every loop kernel returns at once
// after the on-device decision kernel has set ctl->done, so the host never syncs per iteration.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <functional>
#include <atomic>
#include <map>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include <cuda.h>

#include "../../include/ffcz_cuda.h"
#include "archive.hpp"
#include "archive_dev.cuh"
#include "deflate.cuh"
#include "encode.cuh"
#include "fft_plan.cuh"
#include "kernels.cuh"
#include "metrics.cuh"

using namespace ffcz_gpu;

double bitsd_host(unsigned long long b);

namespace {

// Process-wide pool of pinned host blocks backing library-owned result buffers: D2H of the edit
// set and the corrected field runs at full PCIe speed and repeated calls reuse the pinned pages.
struct PinnedPool {
    std::mutex mu;
    std::multimap<size_t, void*> free_blocks;
    std::map<void*, size_t> sizes;
    void* get(size_t bytes) {
        bytes = std::max<size_t>(bytes, 64);
        std::lock_guard<std::mutex> lk(mu);
        auto it = free_blocks.lower_bound(bytes);
        if (it != free_blocks.end() && it->first <= 2 * bytes + (1 << 20)) {
            void* p = it->second;
            free_blocks.erase(it);
            return p;
        }
        void* p = nullptr;
        if (cudaMallocHost(&p, bytes) != cudaSuccess) {
            cudaGetLastError();
            p = std::malloc(bytes);  // pageable fallback (still correct, slower copies)
            if (!p) throw std::bad_alloc();
            sizes[p] = 0;
        } else {
            sizes[p] = bytes;
        }
        return p;
    }
    void put(void* p) {
        if (!p) return;
        std::lock_guard<std::mutex> lk(mu);
        auto it = sizes.find(p);
        if (it == sizes.end()) return;
        if (it->second == 0) {
            std::free(p);
            sizes.erase(it);
        } else {
            free_blocks.emplace(it->second, p);
        }
    }
};

PinnedPool& pinned() {
    static PinnedPool* pool = new PinnedPool;  // never destroyed: results may outlive contexts
    return *pool;
}

} // namespace

struct ffcz_cuda_ctx {
    int device = 0;
    cudaStream_t st = nullptr;
    bool own_stream = false;
    cudaStream_t st_copy = nullptr;  // D2H of the edit set, overlapped with repair / verify
    cudaEvent_t ev_codes = nullptr;
    std::mutex mu;
    Twiddles<double> tw64;
    Twiddles<float> tw32;
    std::map<std::string, std::pair<void*, size_t>> bufs;
    std::vector<ffcz_cuda_ctx*> lanes;  // ffcz_cuda_correct_batch: sub-contexts, one stream each
    Ctl* ctl = nullptr;
    Ctl* hctl = nullptr;   // pinned mirror (one slot per in-flight chunk)
    Ctl* hctl_dev = nullptr;  // device alias of the mapped mirror (k_export_ctl writes it)
    unsigned long long launches = 0;
    cudaEvent_t ev[8] = {};
    // per-kernel-class profiling (ffcz_cuda_profile_*)
    struct ProfRec {
        int cls;
        cudaEvent_t a, b;
        double bytes;
    };
    bool prof_on = false;
    uint32_t call_flags = 0;  // ffcz_cuda_options.flags of the call in progress (per-call switches)
    std::vector<ProfRec> prof;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    cudaEvent_t take_event() {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t e;
            FFCZ_CUDA_CHECK(cudaEventCreate(&e));
            ev_pool.push_back(e);
        }
        return ev_pool[ev_used++];
    }

    void* buf(const std::string& name, size_t bytes) {
        auto it = bufs.find(name);
        if (it != bufs.end() && it->second.second >= bytes) return it->second.first;
        if (it != bufs.end()) {
            FFCZ_CUDA_CHECK(cudaStreamSynchronize(st));
            if (st_copy) FFCZ_CUDA_CHECK(cudaStreamSynchronize(st_copy));
            cudaFree(it->second.first);
            bufs.erase(it);
        }
        void* p = nullptr;
        FFCZ_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
        bufs[name] = {p, std::max<size_t>(bytes, 256)};
        return p;
    }
    template <class T> T* b(const std::string& name, size_t count) {
        return static_cast<T*>(buf(name, count * sizeof(T)));
    }
    void sync() { FFCZ_CUDA_CHECK(cudaStreamSynchronize(st)); }
    Ctl read_ctl() {
        k_export_ctl<<<1, 32, 0, st>>>(ctl, hctl_dev);
        FFCZ_LAUNCH_CHECK();
        sync();
        return *hctl;
    }
};

namespace {

enum ProfClass { kColFwdCheck = 0, kColClipInv, kColPass, kRowR2C, kRowC2R, kRowFused,
                 kElemPre, kElemGate, kElemCompact, kElemCodes, kColRoundTrip, kNumProf };
const char* kProfNames[kNumProf] = {"col_fwd_check (K3a)", "col_clip_inv (K3b)", "col_pass",
                                    "row_r2c", "row_c2r", "row_c2r_sclip_r2c (K1)",
                                    "elem_bounds_eps0_residual", "elem_gate_quantize",
                                    "elem_compact", "elem_codes", "col_check_clip_rt (K3)"};

// RAII event pair around one launch when profiling is on
struct Prof {
    ffcz_cuda_ctx& c;
    int cls;
    double bytes;
    cudaEvent_t a = nullptr;
    Prof(ffcz_cuda_ctx& c_, int cls_, double bytes_) : c(c_), cls(cls_), bytes(bytes_) {
        if (c.prof_on) {
            a = c.take_event();
            FFCZ_CUDA_CHECK(cudaEventRecord(a, c.st));
        }
    }
    ~Prof() {
        if (a) {
            cudaEvent_t b = c.take_event();
            cudaEventRecord(b, c.st);
            c.prof.push_back({cls, a, b, bytes});
        }
    }
};

thread_local std::string g_last_error;

int fail(int status, const std::string& msg) {
    g_last_error = msg;
    return status;
}

template <class F>
int guarded(ffcz_cuda_ctx* ctx, F&& f) {
    try {
        if (!ctx) return fail(kValidation, "null context");
        std::lock_guard<std::mutex> lk(ctx->mu);
        FFCZ_CUDA_CHECK(cudaSetDevice(ctx->device));
        f();
        return kOk;
    } catch (const Error& e) {
        return fail(e.status, e.what());
    } catch (const std::bad_alloc& e) {
        return fail(kOom, e.what());
    } catch (const std::exception& e) {
        return fail(kCuda, e.what());
    }
}

inline unsigned grid_for(long long n, int threads = 256) {
    long long b = (n + threads - 1) / threads;
    return static_cast<unsigned>(std::max<long long>(1, std::min<long long>(b, 148LL * 16)));
}

constexpr int kPitchAlign = 16;

// The column axis whose pass completes the forward transform (and starts the inverse), i.e. the
// pass that carries the f-cube check / clip / mark / verify hooks.  For 3-D fields this is the
// MIDDLE axis (row stride P: a tile's rows sit inside one plane, so the hooks' F / Delta accesses
// stay TLB- and DRAM-page-local), with the outer axis transformed first.  FFCZ_COMPLETE_AXIS=0
// restores the outer axis (A/B runs).  2-D fields have only axis 1.
// FFCZ_EPS0_FUSION=1: form eps0 inside the first R2C instead of a separate eps0 pass.  Off by
// default: measured at 512^3 the fused kernel (840 us, 2.5 TB/s) is slower than the two passes
// it replaces (376 + 343 us), so the separate pass stays.
inline // Frequency gate and code compaction in one pass (k_gate_codes_freq, decoupled look-back) is
// opt-in (FFCZ_GATE_CODES=1pass): at 512^3 it measured 1.74 ms per call against 1.46 ms for the
// two-pass flags -> scan -> codes kernels it would replace (profiles/r01_summary.md).
bool gate_codes_one_pass() {
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_GATE_CODES");
        return e && std::strcmp(e, "1pass") == 0;
    }();
    return on;
}

// Gate rounds: C2R -> repair -> R2C as one fused row pass (FFCZ_GATE_ROW_FUSED=1, A/B).
bool gate_row_fused() {
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_GATE_ROW_FUSED");
        return e && e[0] == '1';
    }();
    return on;
}

// Escape repair on the decoder view (HookRepairVerifyS::dview; default on).  FFCZ_REPAIR_ORDER=
// reference restores the reference's eps_tilde check plus a separate verify transform.
// Per call: FFCZ_REPAIR_REFERENCE_ORDER in ffcz_cuda_options.flags selects the reference order.
bool decoder_view_repair(const ffcz_cuda_ctx& c) {
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_REPAIR_ORDER");
        return !(e && std::strcmp(e, "reference") == 0);
    }();
    return on && !(c.call_flags & FFCZ_REPAIR_REFERENCE_ORDER);
}

bool eps0_fusion_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_EPS0_FUSION");
        return e && e[0] == '1';
    }();
    return on;
}

// FFCZ_F_REBUILD=0: accumulate F in every clip pass (read-modify-write) instead of marking the
// moved components and rebuilding F once at the gate (HookFClip::moved, HookFRebuild).
// Per call: FFCZ_F_ACCUMULATE in ffcz_cuda_options.flags selects the accumulation.
inline bool f_rebuild_enabled(const ffcz_cuda_ctx& c) {
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_F_REBUILD");
        return !(e && e[0] == '0');
    }();
    if (c.call_flags & FFCZ_F_ACCUMULATE) return false;
    return on;
}

// FFCZ_LOOP_RT=0: the loop's check and clip as two passes (K3a, K3b) instead of one round trip
inline bool loop_rt_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_LOOP_RT");
        return !(e && e[0] == '0');
    }();
    return on;
}

// FFCZ_LOOP_K1=0: the loop's last-axis step as C2R (+ s-clip, eps written) then R2C instead of
// one fused row pass
inline bool loop_k1_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_LOOP_K1");
        return !(e && e[0] == '0');
    }();
    return on;
}

// FFCZ_LOOP_EPS_LATE=0: the fused row pass stores epsilon every iteration instead of once
inline bool loop_eps_late_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_LOOP_EPS_LATE");
        return !(e && e[0] == '0');
    }();
    return on;
}

// The column axis whose pass completes the forward transform (and carries the check / clip):
// FFCZ_COMPLETE_AXIS=0 / 1 forces the outer / middle axis; by default the outer axis with a global
// frequency bound (the round trip there and the plain passes on the middle axis: 464.6 vs 467.9
// ms at 1024^3 config 4) and the middle axis with per-component lanes (config 2 at 512^3: 41.1 vs
// 27.3 GB/s on the outer axis), profiles/r02_ab_complete_axis.txt
inline int complete_axis(bool three_d, bool global_delta) {
    static const int v = [] {
        const char* e = std::getenv("FFCZ_COMPLETE_AXIS");
        return e ? (e[0] == '0' ? 0 : 1) : -1;
    }();
    if (!three_d) return 1;
    return v >= 0 ? v : (global_delta ? 0 : 1);
}

struct Bounds {
    SpatialB sb{nullptr, 0.0};
    FreqB fb{nullptr, nullptr, 0.0};
};

// DualBounds' invariants (bounds.cpp:10-18,43-59): every per-point E and per-component Delta
// entry strictly positive and finite, and the Re / Im lanes Hermitian-consistent
// (lane[k] == lane[mirror(k)], field.cpp:41-50).  The reference enforces them when a DualBounds
// is built; a C-ABI caller hands raw arrays, so they are checked here unless the caller sets
// FFCZ_BOUNDS_VALIDATED (the C++ shim: its ffcz::DualBounds was built by those factories).
// Device arrays: one pass (bad[0] = first non-positive index, bad[1] = first asymmetric index).
__global__ void k_check_bounds(const double* __restrict__ e, const double* __restrict__ re,
                               const double* __restrict__ im, long long d0, long long d1,
                               long long d2, unsigned long long* bad) {
    const long long N = d0 * d1 * d2;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        if (e) {
            const double v = e[i];
            if (!(v > 0.0) || !isfinite(v)) atomicMin(&bad[0], (unsigned long long)i);
        }
        if (re) {
            const long long i2 = i % d2, t = i / d2, i1 = t % d1, i0 = t / d1;
            const long long m = (((d0 - i0) % d0) * d1 + (d1 - i1) % d1) * d2 + (d2 - i2) % d2;
            const double a = re[i], b = im[i];
            if (!(a > 0.0) || !isfinite(a) || !(b > 0.0) || !isfinite(b))
                atomicMin(&bad[0], (unsigned long long)(N + i));
            if (a != re[m] || b != im[m]) atomicMin(&bad[1], (unsigned long long)i);
        }
    }
}

void validate_bounds(ffcz_cuda_ctx& c, const Geometry& g, const ffcz_bounds_desc& bd, bool on_dev) {
    const bool pp = bd.spatial_per_point, pc = bd.freq_per_component;
    if (!pp && !pc) return;
    if (pp && !bd.spatial_values) throw Error(kValidation, "per-point spatial bound array is null");
    if (pc && (!bd.freq_re || !bd.freq_im))
        throw Error(kValidation, "per-component frequency bound arrays are null");
    const long long N = g.N, d0 = g.d[0], d1 = g.d[1], d2 = g.d[2];
    unsigned long long bad[2] = {~0ull, ~0ull};
    if (on_dev) {
        unsigned long long* db = c.b<unsigned long long>("bounds_bad", 2);
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(db, bad, sizeof(bad), cudaMemcpyHostToDevice, c.st));
        k_check_bounds<<<grid_for(N), 256, 0, c.st>>>(pp ? bd.spatial_values : nullptr,
                                                      pc ? bd.freq_re : nullptr,
                                                      pc ? bd.freq_im : nullptr, d0, d1, d2, db);
        FFCZ_LAUNCH_CHECK();
        ++c.launches;
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(bad, db, sizeof(bad), cudaMemcpyDeviceToHost, c.st));
        c.sync();
    } else {
        const int nt = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
        std::vector<std::array<unsigned long long, 2>> part(nt, {~0ull, ~0ull});
        auto work = [&](int t) {
            const long long lo = N * t / nt, hi = N * (t + 1) / nt;
            auto& b = part[t];
            for (long long i = lo; i < hi; ++i) {
                if (pp) {
                    const double v = bd.spatial_values[i];
                    if (!(v > 0.0) || !std::isfinite(v)) b[0] = std::min<unsigned long long>(b[0], i);
                }
                if (pc) {
                    const long long i2 = i % d2, q = i / d2, i1 = q % d1, i0 = q / d1;
                    const long long m = (((d0 - i0) % d0) * d1 + (d1 - i1) % d1) * d2 + (d2 - i2) % d2;
                    const double a = bd.freq_re[i], bb = bd.freq_im[i];
                    if (!(a > 0.0) || !std::isfinite(a) || !(bb > 0.0) || !std::isfinite(bb))
                        b[0] = std::min<unsigned long long>(b[0], N + i);
                    if (a != bd.freq_re[m] || bb != bd.freq_im[m])
                        b[1] = std::min<unsigned long long>(b[1], i);
                }
            }
        };
        std::vector<std::thread> th;
        for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
        work(0);
        for (auto& t : th) t.join();
        for (auto& p : part) {
            bad[0] = std::min(bad[0], p[0]);
            bad[1] = std::min(bad[1], p[1]);
        }
    }
    if (bad[0] != ~0ull) {
        if (bad[0] < static_cast<unsigned long long>(N))
            throw Error(kValidation, "per-point spatial bound must be strictly positive and finite");
        throw Error(kValidation, "per-component frequency bound must be strictly positive and finite");
    }
    if (bad[1] != ~0ull)
        throw Error(kValidation, "per-component frequency bounds are not Hermitian-consistent");
}

// Copies / restricts the caller's bounds onto the device (per-component arrays -> half layout).
Bounds upload_bounds(ffcz_cuda_ctx& c, const Geometry& g, const ffcz_bounds_desc& bd, bool on_dev,
                     bool validate = false) {
    if (validate) validate_bounds(c, g, bd, on_dev);
    Bounds b;
    const long long N = g.N;
    if (bd.spatial_per_point) {
        if (!bd.spatial_values) throw Error(kValidation, "per-point spatial bound array is null");
        if (on_dev) {
            b.sb.v = bd.spatial_values;
        } else {
            double* d = c.b<double>("E_pp", N);
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(d, bd.spatial_values, N * sizeof(double),
                                            cudaMemcpyHostToDevice, c.st));
            b.sb.v = d;
        }
    } else {
        if (!(bd.spatial_global > 0.0) || !std::isfinite(bd.spatial_global))
            throw Error(kValidation, "spatial bound E must be strictly positive and finite");
        b.sb.g = bd.spatial_global;
    }
    if (bd.freq_per_component) {
        if (!bd.freq_re || !bd.freq_im)
            throw Error(kValidation, "per-component frequency bound arrays are null");
        const HalfGeom hg = g.hg();
        auto restrict_lane = [&](const double* full, const char* name) {
            double* half = c.b<double>(name, g.half_elems());
            if (!on_dev) {
                // host lane: copy only the half-grid columns k2 <= n2/2 of every row, straight
                // into the pitched half layout (one strided DMA; half the bytes of the full lane)
                FFCZ_CUDA_CHECK(cudaMemcpy2DAsync(half, g.P * sizeof(double), full,
                                                  g.n2 * sizeof(double), g.H * sizeof(double),
                                                  g.rows, cudaMemcpyHostToDevice, c.st));
                return half;
            }
            const double* dfull = full;
            {
                Prof p(c, kElemPre, 16.0 * g.Nc());
                k_gather_half<<<grid_for(g.Nc()), 256, 0, c.st>>>(dfull, half, hg);
            }
            FFCZ_LAUNCH_CHECK();
            ++c.launches;
            return half;
        };
        bool same = bd.freq_re == bd.freq_im;
        if (!same && !on_dev) same = std::memcmp(bd.freq_re, bd.freq_im, N * sizeof(double)) == 0;
        b.fb.re = restrict_lane(bd.freq_re, "D_re");
        b.fb.im = same ? b.fb.re : restrict_lane(bd.freq_im, "D_im");
    } else {
        if (!(bd.freq_global > 0.0) || !std::isfinite(bd.freq_global))
            throw Error(kValidation, "frequency bound Delta must be strictly positive and finite");
        b.fb.g = bd.freq_global;
    }
    return b;
}

struct LoopResult {
    unsigned long long passes = 0;
    bool converged = false;
    double residual_f = 0.0;
    bool fused = false;
    const unsigned char* moved = nullptr;  // rebuild mode: F is complete only after pass 1
    unsigned long long passes32 = 0;       // mixed policy: passes run by the FP32 phase
    bool s_zero = false;                   // fused loop: no spatial clip ever moved a sample
};

// The POCS loop (projection.cpp:96-126) on device.  eps holds epsilon0 on entry and the final
// epsilon on exit; S (N) and F (half) are the accumulated edits.
LoopResult run_loop(ffcz_cuda_ctx& c, const Geometry& g, double* eps, const Bounds& bw,
                    double fscale, bool allow_fused, double* S, double2* F,
                    bool allow_rebuild = true, bool keep_moved = false,
                    bool have_r2c = false) {
    cudaStream_t st = c.st;
    FftPlan<double> plan{g, &c.tw64};
    const int* gate = &c.ctl->done;
    double2* spec = c.b<double2>("spec", g.half_elems());
    const double invN = 1.0 / static_cast<double>(g.N);
    const HalfGeom hg = g.hg();
    const bool fused = allow_fused && plan.fused_ok();
    if (!fused) {  // the fused hooks write S and F densely on the first clip instead
        FFCZ_CUDA_CHECK(cudaMemsetAsync(S, 0, g.N * sizeof(double), st));
        FFCZ_CUDA_CHECK(cudaMemsetAsync(F, 0, g.half_elems() * sizeof(double2), st));
    }
    const bool three_d = g.d[0] > 1;
    unsigned char* moved = nullptr;
    if (fused && (keep_moved || (allow_rebuild && f_rebuild_enabled(c)))) {
        moved = c.b<unsigned char>("f_moved", g.half_elems());
        if (!keep_moved) FFCZ_CUDA_CHECK(cudaMemsetAsync(moved, 0, g.half_elems(), st));
    }
    const int za = complete_axis(three_d, !bw.fb.re);  // the pass that completes the forward transform
    const int mid = 1 - za;                   // the other column axis (3-D only)
    double* tmp = fused ? nullptr : c.b<double>("real_tmp", g.N);
    // K3a + K3b as one round trip (HookRT): the forward chain ends in `spec`, the inverse chain
    // starts from `spec_rt`; the last check's clip is speculative and undone after the loop
    // (global Delta only: per-component lanes would add 16 dependent loads per thread to the
    // check / clip; those keep the K3a / K3b pair with its TMA side tile)
    const bool rt = fused && moved && !keep_moved && !bw.fb.re && loop_rt_enabled() &&
                    plan.rt_ok(za);
    double2* spec_rt = rt ? c.b<double2>("spec_rt", g.half_elems()) : nullptr;
    double2* inv_src = rt ? spec_rt : spec;
    // fused K1 on the radix row path (power-of-two last axis)
    const bool k1 = fused && loop_k1_enabled() && radix_row_ok(g.n2);
    // K1 without the epsilon store: the inverse chain alternates between two buffers, so the
    // last executed K1's input is intact after the loop and its C2R half re-forms the final
    // epsilon once (same kernel, same bits) instead of every iteration storing it
    const bool eps_late = rt && k1 && loop_eps_late_enabled();
    double2* spec_rt2 = eps_late ? c.b<double2>("spec_rt2", g.half_elems()) : nullptr;

    const double pass_bytes = 32.0 * g.Nc();
    const double dlanes = bw.fb.re ? (bw.fb.im == bw.fb.re ? 1.0 : 2.0) : 0.0;
    const double check_bytes = pass_bytes + 8.0 * g.Nc() * dlanes;
    const double fused_bytes = pass_bytes + 8.0 * g.N + (bw.sb.v ? 8.0 * g.N : 0.0);
    int nbody = 0;  // bodies enqueued: body k (from 0) is clip pass k + 1 unless gated
    auto body = [&]() {
        if (rt) {
            {
                // read + write of the spectrum, Delta, the 1-B marks (read; written where a clamp
                // moved: counted as N_c), F written densely by the first clip
                Prof p(c, kColRoundTrip,
                       check_bytes + 2.0 * g.Nc() + (nbody == 0 ? 16.0 * g.Nc() : 0.0));
                if (eps_late) inv_src = (nbody & 1) ? spec_rt2 : spec_rt;
                plan.col_rt(za, spec, inv_src, gate, HookRT{bw.fb, fscale, c.ctl, F, moved}, st);
            }
            k_decide<<<1, 1, 0, st>>>(c.ctl);                                              // K4
        } else if (fused) {
            {
                Prof p(c, kColFwdCheck, check_bytes);
                plan.col(za, -1, spec, spec, gate, HookFReduce{bw.fb, fscale, c.ctl}, st);   // K3a
            }
            k_decide<<<1, 1, 0, st>>>(c.ctl);                                              // K4
            {
                // clip pass 1 writes F densely (16 N_c); later passes write the 1-B clip map
                // where a clamp moved a component (counted as N_c: an upper bound)
                Prof p(c, kColClipInv, check_bytes + (nbody == 0 ? 16.0 * g.Nc() : 0.0) +
                                           (moved && nbody > 0 ? 1.0 * g.Nc() : 0.0));
                plan.col(za, +1, spec, spec, gate,
                         HookFClip<double>{bw.fb, fscale, F, c.ctl, moved}, st);          // K3b
            }
        }
        if (fused) {
            if (three_d) {
                Prof p(c, kColPass, pass_bytes);
                plan.col(mid, +1, inv_src, inv_src, gate, HookNone{}, st);
            }
            if (k1) {
                // K1: C2R -> s-clip (eps written, S) -> R2C in one row pass, from the inverse
                // chain's buffer into the forward chain's: half rows read + written, eps written,
                // S written densely by the first clip (later: read-modify-write where a clamp
                // moved, not counted), per-point E read
                Prof p(c, kRowFused, 32.0 * g.Nc() + (eps_late ? 0.0 : 8.0 * g.N) +
                                         (nbody == 0 ? 8.0 * g.N : 0.0) +
                                         (bw.sb.v ? 8.0 * g.N : 0.0));
                launch_row_fused<double>(g.n2, inv_src, g.P, g.rows, g.n2, invN, c.tw64, gate,
                                         HookSClip<double>{bw.sb, fscale, S,
                                                           eps_late ? nullptr : eps, c.ctl},
                                         st, inv_src == spec ? nullptr : spec);
            } else {   // K1 as C2R(+s-clip, eps written) then R2C
                Prof p(c, kRowC2R, 16.0 * g.Nc() + 8.0 * g.N + (bw.sb.v ? 8.0 * g.N : 0.0));
                launch_row_c2r_hook<double>(g.n2, inv_src, g.P, eps, g.n2, g.rows, invN, c.tw64,
                                            gate,
                                            HookSClip<double>{bw.sb, fscale, S, nullptr, c.ctl},
                                            st);
            }
            if (!k1) {
                Prof p(c, kRowR2C, 8.0 * g.N + 16.0 * g.Nc());
                launch_row_r2c<double>(g.n2, eps, g.n2, spec, g.P, g.rows, c.tw64, gate, st);
            }
            if (three_d) {
                Prof p(c, kColPass, pass_bytes);
                plan.col(mid, -1, spec, spec, gate, HookNone{}, st);
            }
            c.launches += (three_d ? 7 : 5) - (rt ? 1 : 0) - (k1 ? 1 : 0);
            ++nbody;
        } else {
            plan.r2c(eps, spec, gate, st);
            k_freduce<<<grid_for(g.Nc()), 256, 0, st>>>(spec, hg, bw.fb, fscale, c.ctl, gate);
            k_decide<<<1, 1, 0, st>>>(c.ctl);
            k_fclip<<<grid_for(g.Nc()), 256, 0, st>>>(spec, hg, bw.fb, fscale, F, gate);
            plan.c2r(spec, spec, tmp, invN, gate, st);
            k_sclip<<<grid_for(g.N), 256, 0, st>>>(tmp, eps, g.N, bw.sb, fscale, S, gate);
            c.launches += 10;
        }
        FFCZ_LAUNCH_CHECK();
    };

    if (fused) {
        if (!have_r2c) {  // (else the caller's fused eps0 + R2C already filled `spec`)
            Prof p(c, kRowR2C, 8.0 * g.N + 16.0 * g.Nc());
            launch_row_r2c<double>(g.n2, eps, g.n2, spec, g.P, g.rows, c.tw64, gate, st);
        }
        if (three_d) {
            Prof p(c, kColPass, pass_bytes);
            plan.col(mid, -1, spec, spec, gate, HookNone{}, st);
        }
        c.launches += three_d ? 2 : 1;
    }

    // pipelined speculative chunks: keep one chunk queued behind the one being polled
    struct Poll {
        cudaEvent_t ev;
        int slot;
    };
    static const int kChunk[] = {1, 1, 2, 4, 8};
    int ci = 0, issued = 0;
    std::vector<Poll> inflight;
    auto issue_chunk = [&]() {
        const int n = kChunk[std::min(ci++, 4)];
        for (int i = 0; i < n; ++i) body();
        const int slot = issued % 2;
        k_export_ctl<<<1, 32, 0, st>>>(c.ctl, &c.hctl_dev[1 + slot]);
        FFCZ_LAUNCH_CHECK();
        cudaEvent_t ev = c.ev[4 + slot];
        FFCZ_CUDA_CHECK(cudaEventRecord(ev, st));
        inflight.push_back({ev, slot});
        ++issued;
    };
    issue_chunk();
    for (;;) {
        issue_chunk();
        Poll p = inflight.front();
        inflight.erase(inflight.begin());
        FFCZ_CUDA_CHECK(cudaEventSynchronize(p.ev));
        if (c.hctl[1 + p.slot].done) break;
    }
    if (rt) {
        // the last check's clip never happened in the reference: re-form delta_final in `spec`
        // and clear the marks only that clip set (HookRT)
        Prof p(c, kColRoundTrip, check_bytes + 2.0 * g.Nc());
        HookRT hk{bw.fb, fscale, c.ctl, F, moved};
        hk.recover = 1;
        plan.col_rt(za, spec, spec, nullptr, hk, st);
        ++c.launches;
    }
    if (eps_late) {
        // the final epsilon = the s-clipped C2R of the last executed K1's input (body passes - 1;
        // with no clip at all eps still holds epsilon0)
        const unsigned long long passes = c.read_ctl().passes;
        if (passes >= 1) {
            Prof p(c, kRowC2R, 16.0 * g.Nc() + 8.0 * g.N + (bw.sb.v ? 8.0 * g.N : 0.0));
            HookSClip<double> hs{bw.sb, fscale, nullptr, eps, nullptr};
            hs.c2r_only = 1;
            launch_row_fused<double>(g.n2, ((passes - 1) & 1) ? spec_rt2 : spec_rt, g.P, g.rows,
                                     g.n2, invN, c.tw64, nullptr, hs, st, nullptr);
            ++c.launches;
        }
    }
    const Ctl h = c.read_ctl();
    if (fused && h.passes == 0) {  // converged at the first check: no clip ever wrote S / F
        FFCZ_CUDA_CHECK(cudaMemsetAsync(S, 0, g.N * sizeof(double), st));
        FFCZ_CUDA_CHECK(cudaMemsetAsync(F, 0, g.half_elems() * sizeof(double2), st));
    }
    LoopResult r;
    r.passes = h.passes;
    r.converged = h.converged;
    r.residual_f = h.residual_f;
    r.fused = fused;
    r.moved = moved;
    r.s_zero = fused && !h.s_any;
    return r;
}

} // namespace

// host-side bit cast
double bitsd_host(unsigned long long b);

namespace {

// bitmap -> ascending index list; returns the count
unsigned long long compact_bits(ffcz_cuda_ctx& c, const unsigned* words, long long nwords,
                                unsigned long long* idx) {
    const long long nblk = std::max<long long>(1, (nwords + 1023) / 1024);
    unsigned long long* counts = c.b<unsigned long long>("blk_counts", nblk + 1);
    {
        Prof p(c, kElemCompact, 0.0);
        k_popc_blocks<<<static_cast<unsigned>(nblk), 1024, 0, c.st>>>(words, nwords, counts);
        k_scan_blocks<<<1, 1024, 0, c.st>>>(counts, nblk, &c.ctl->count_a);
        k_compact<<<static_cast<unsigned>(nblk), 1024, 0, c.st>>>(words, nwords, counts, idx);
    }
    FFCZ_LAUNCH_CHECK();
    c.launches += 3;
    return c.read_ctl().count_a;
}

struct GateOut {
    unsigned long long n_keep_s = 0, n_keep_f = 0, n_esc_s = 0, n_esc_f = 0;
    unsigned long long rounds = 0;
    int verify_ok = 0;
    double vs = 0, vf = 0;
    unsigned long long act_s = 0, act_f = 0;
};

// whole-field FP64 transforms with one profiling record per pass
void r2c_p(ffcz_cuda_ctx& c, const FftPlan<double>& plan, const double* x, double2* half) {
    const Geometry& g = plan.g;
    {
        Prof p(c, kRowR2C, 8.0 * g.N + 16.0 * g.Nc());
        launch_row_r2c<double>(g.n2, x, g.n2, half, g.P, g.rows, c.tw64, nullptr, c.st);
    }
    for (int a : {1, 0})
        if (g.d[a] > 1) {
            Prof p(c, kColPass, 32.0 * g.Nc());
            plan.col(a, -1, half, half, nullptr, HookNone{}, c.st);
        }
    c.launches += 1 + (g.d[0] > 1) + (g.d[1] > 1);
}

void c2r_p(ffcz_cuda_ctx& c, const FftPlan<double>& plan, const double2* half, double2* work,
           double* x, double scale) {
    const Geometry& g = plan.g;
    const double2* src = half;
    for (int a : {0, 1})
        if (g.d[a] > 1) {
            Prof p(c, kColPass, 32.0 * g.Nc());
            plan.col(a, +1, src, work, nullptr, HookNone{}, c.st);
            src = work;
        }
    {
        Prof p(c, kRowC2R, 8.0 * g.N + 16.0 * g.Nc());
        launch_row_c2r<double>(g.n2, src, g.P, x, g.n2, g.rows, scale, c.tw64, nullptr, c.st);
    }
    c.launches += 1 + (g.d[0] > 1) + (g.d[1] > 1);
}

template <class TI>
GateOut run_gate(ffcz_cuda_ctx& c, const Geometry& g, const TI* orig, const TI* dec,
                 const Bounds& bo, int m, const LoopResult& lr, double* eps, double* S,
                 double2* F, double2* spec, double* corrected,
                 const std::function<void(unsigned long long, unsigned long long)>& on_codes) {
    cudaStream_t st = c.st;
    FftPlan<double> plan{g, &c.tw64};
    const HalfGeom hg = g.hg();
    const long long N = g.N, Nc = g.Nc();
    const long long ws = (N + 31) / 32, wf = (Nc + 31) / 32;
    double* spat_cur = c.b<double>("spat_cur", N);
    double2* freq_cur = c.b<double2>("freq_cur", g.half_elems());
    unsigned* keep_s = c.b<unsigned>("keep_s", ws);
    unsigned* esc_s = c.b<unsigned>("esc_s", ws);
    unsigned* keep_f = c.b<unsigned>("keep_f", wf);
    unsigned* esc_f = c.b<unsigned>("esc_f", wf);
    unsigned long long* idx = c.b<unsigned long long>("idx", std::max(N, Nc));
    int* codes_s = c.b<int>("codes_s", N);
    int* codes_f = c.b<int>("codes_f", 2 * Nc);
    double* eps_t = c.b<double>("eps_tilde", N);

    const bool converged = lr.converged, fused = lr.fused;
    if (lr.moved && lr.passes >= 2) {
        // F = mask(delta_final - FFT(eps0 + S)): one forward transform replaces the F
        // read-modify-writes of clip passes 2.. (HookFClip::moved); delta_final is `spec`
        const bool three_d = g.d[0] > 1;
        const int za = complete_axis(three_d, !bo.fb.re);
        double* x = eps_t;
        double2* work = freq_cur;  // free until k_gate_freq below
        bool fused_in = false;
        {   // eps0 + S formed inside the R2C (orig, dec, S rows in; no eps0 + S round trip)
            Prof p(c, kRowR2C, (2.0 * sizeof(TI) + 8.0) * N + 16.0 * Nc);
            fused_in = launch_row_r2c_eps0<TI>(g.n2, orig, dec, work, g.P, g.rows, c.tw64, bo.sb,
                                               1.0, 0.0, nullptr, st, S);
            if (!fused_in) p.bytes = 0.0;
        }
        if (!fused_in) {
            {
                Prof p(c, kElemPre, (2.0 * sizeof(TI) + 16.0) * N);
                k_eps0_plus_s<TI><<<grid_for(N), 256, 0, st>>>(orig, dec, S, x, N);
            }
            {
                Prof p(c, kRowR2C, 8.0 * g.N + 16.0 * Nc);
                launch_row_r2c<double>(g.n2, x, g.n2, work, g.P, g.rows, c.tw64, nullptr, st);
            }
        }
        if (three_d) {
            Prof p(c, kColPass, 32.0 * Nc);
            plan.col(1 - za, -1, work, work, nullptr, HookNone{}, st);
        }
        {
            Prof p(c, kColFwdCheck, 48.0 * Nc + Nc);
            if (plan.rt_ok(za) && loop_rt_enabled())  // marks + delta_final landed by TMA
                plan.col_frebuild(za, work, spec, F, lr.moved, st);
            else
                plan.col(za, -1, work, work, nullptr, HookFRebuild{spec, F, lr.moved}, st);
        }
        FFCZ_LAUNCH_CHECK();
        c.launches += three_d ? 4 : 3;
    }
    FFCZ_CUDA_CHECK(cudaMemsetAsync(&c.ctl->act_s, 0, 2 * sizeof(unsigned long long), st));
    const bool one_pass = gate_codes_one_pass();
    {
        Prof p(c, kElemGate, (lr.s_zero ? 0.0 : 16.0 * N) + (one_pass ? 0.0 : 32.0 * Nc));
        if (lr.s_zero) {
            // S is identically zero (no spatial clip moved a sample): no spatial edits, no
            // overflow escapes, spat_cur = 0 (editset.cpp:43-66 on an all-zero S)
            FFCZ_CUDA_CHECK(cudaMemsetAsync(spat_cur, 0, N * sizeof(double), st));
            FFCZ_CUDA_CHECK(cudaMemsetAsync(keep_s, 0, ws * sizeof(unsigned), st));
            FFCZ_CUDA_CHECK(cudaMemsetAsync(esc_s, 0, ws * sizeof(unsigned), st));
        } else {
            k_gate_spatial<<<grid_for(N), 256, 0, st>>>(S, N, bo.sb, m, spat_cur, keep_s, esc_s,
                                                        c.ctl);
            ++c.launches;
        }
        if (!one_pass)
            k_gate_freq<<<grid_for(Nc), 256, 0, st>>>(F, hg, bo.fb, m, freq_cur, keep_f, esc_f,
                                                       c.ctl);
    }
    if (one_pass) {
        Prof p(c, kElemGate, 32.0 * Nc + 8.0 * Nc);  // F + Delta in, freq_cur + codes out
        const long long nt = std::max<long long>(1, (Nc + kGateCodesTile - 1) / kGateCodesTile);
        unsigned long long* tstat = c.b<unsigned long long>("gc_status", nt + 1);
        unsigned* ticket = reinterpret_cast<unsigned*>(tstat + nt);
        FFCZ_CUDA_CHECK(cudaMemsetAsync(tstat, 0, (nt + 1) * sizeof(unsigned long long), st));
        k_gate_codes_freq<<<static_cast<unsigned>(nt), 256, 0, st>>>(
            F, hg, bo.fb, m, freq_cur, keep_f, esc_f, codes_f, tstat, ticket, nt, c.ctl);
    }
    FFCZ_LAUNCH_CHECK();
    ++c.launches;

    GateOut o;
    // counts + offsets of the keep bitmaps, then codes written straight from the bits
    auto codes_from = [&](const unsigned* words, long long nwords, const char* cname,
                          auto launch_codes) {
        const long long nblk = std::max<long long>(1, (nwords + 1023) / 1024);
        unsigned long long* counts = c.b<unsigned long long>(cname, nblk + 1);
        {
            Prof p(c, kElemCompact, 0.0);
            k_popc_blocks<<<static_cast<unsigned>(nblk), 1024, 0, st>>>(words, nwords, counts);
            k_scan_blocks<<<1, 1024, 0, st>>>(counts, nblk, &c.ctl->count_a);
        }
        {
            Prof p(c, kElemCodes, 0.0);
            launch_codes(static_cast<unsigned>(nblk), counts);
        }
        FFCZ_LAUNCH_CHECK();
        c.launches += 3;
        return c.read_ctl().count_a;
    };
    o.n_keep_s = lr.s_zero ? 0 : codes_from(keep_s, ws, "blk_counts_s", [&](unsigned nb, unsigned long long* off) {
        k_codes_spatial_bits<<<nb, 1024, 0, st>>>(keep_s, ws, off, S, bo.sb, m, codes_s);
    });
    if (one_pass)
        o.n_keep_f = c.read_ctl().count_b;  // count_a is the spatial compaction's
    else
        o.n_keep_f = codes_from(keep_f, wf, "blk_counts_f", [&](unsigned nb, unsigned long long* off) {
            k_codes_freq_bits<<<nb, 1024, 0, st>>>(keep_f, wf, off, F, hg, bo.fb, m, codes_f);
        });
    (void)idx;
    // flags and codes are final here (repair rounds only add escapes): hand them to the copy
    // stream so their D2H overlaps the repair / verify passes
    if (on_codes) on_codes(o.n_keep_s, o.n_keep_f);

    // delta_star = FFT(final_eps) is the spectrum the loop's last convergence check produced
    // (still in `spec`); S and F are consumed, so they become the round's real / half work buffers.
    double2* delta_star = spec;
    double* fpart = S;
    double2* work = F;
    const double invN = 1.0 / static_cast<double>(N);
    if (fused) {
        // fused rounds: [Z inv] [Y inv] [C2R -> repair_s -> R2C] [Y fwd] [Z fwd + mark] + sparse
        const bool three_d = g.d[0] > 1;
        const int za = complete_axis(three_d, !bo.fb.re);
        const int mid = 1 - za;
        const long long vw = (g.half_elems() + 31) / 32;
        unsigned* viol = c.b<unsigned>("viol", vw);
        const double pass = 32.0 * Nc;
        auto inverse_and_row = [&](auto row_hook, double row_bytes) {
            {
                Prof p(c, kColPass, pass);
                plan.col(za, +1, freq_cur, work, nullptr, HookNone{}, st);
            }
            if (three_d) {
                Prof p(c, kColPass, pass);
                plan.col(mid, +1, work, work, nullptr, HookNone{}, st);
            }
            bool fused_row = false;
            if constexpr (std::is_same_v<decltype(row_hook), HookRepairVerifyS<TI>>)
                fused_row = row_hook.dview && gate_row_fused() && plan.fused_ok();
            if (fused_row) {
                // C2R -> repair on the decoder view -> R2C in one row pass: v never leaves the SM
                Prof p(c, kRowC2R, row_bytes - 8.0 * N + 16.0 * Nc);
                if constexpr (std::is_same_v<decltype(row_hook), HookRepairVerifyS<TI>>)
                    launch_row_fused<double>(g.n2, work, g.P, g.rows, g.n2, invN, c.tw64, nullptr,
                                             row_hook, st);
                c.launches -= 1;
            } else {
                {
                    Prof p(c, kRowC2R, row_bytes);
                    launch_row_c2r_hook<double>(g.n2, work, g.P, eps_t, g.n2, g.rows, invN, c.tw64,
                                                nullptr, row_hook, st);
                }
                {
                    Prof p(c, kRowR2C, 8.0 * g.N + 16.0 * Nc);
                    launch_row_r2c<double>(g.n2, eps_t, g.n2, work, g.P, g.rows, c.tw64, nullptr,
                                           st);
                }
            }
            if (three_d) {
                Prof p(c, kColPass, pass);
                plan.col(mid, -1, work, work, nullptr, HookNone{}, st);
            }
            c.launches += three_d ? 5 : 3;
        };
        auto forward_row_mid = [&](const double* x) {
            {
                Prof p(c, kRowR2C, 8.0 * g.N + 16.0 * Nc);
                launch_row_r2c<double>(g.n2, x, g.n2, work, g.P, g.rows, c.tw64, nullptr, st);
            }
            if (three_d) {
                Prof p(c, kColPass, pass);
                plan.col(mid, -1, work, work, nullptr, HookNone{}, st);
            }
            c.launches += three_d ? 2 : 1;
        };
        bool verified = false;
        bool sc_zero = lr.s_zero;  // spat_cur stays zero until a spatial repair
        const bool dview = decoder_view_repair(c);
        if (converged) {
            double* eps_v = dview ? nullptr : c.b<double>("eps_verify", N);
            for (int round = 0; round < 32; ++round) {                   // pipeline.cpp:116
                FFCZ_CUDA_CHECK(cudaMemsetAsync(&c.ctl->dirty, 0, sizeof(int), st));
                FFCZ_CUDA_CHECK(cudaMemsetAsync(&c.ctl->dirty_s, 0, sizeof(int), st));
                FFCZ_CUDA_CHECK(cudaMemsetAsync(&c.ctl->vs_bits, 0, 2 * sizeof(unsigned long long), st));
                FFCZ_CUDA_CHECK(cudaMemsetAsync(viol, 0, vw * sizeof(unsigned), st));
                // inverse once: eps_tilde for the repair check (pipeline.cpp:125-136) and, in case
                // the round is clean, the decoder view for verify (pipeline.cpp:174-176)
                HookRepairVerifyS<TI> hk{orig, dec, spat_cur, eps, bo.sb, esc_s, corrected, eps_v,
                                         c.ctl};
                hk.sc_zero = sc_zero;
                hk.dview = dview;
                hk.keep_words = keep_s;
                // half spectrum in, orig + dec, spat_cur (unless still zero), the checked view
                // out (the R2C's input), eps_v (reference order), corrected, per-point E
                inverse_and_row(hk, 16.0 * Nc + 2.0 * sizeof(TI) * N + (sc_zero ? 0.0 : 8.0 * N) +
                                        8.0 * N + (dview ? 0.0 : 8.0 * N) +
                                        (corrected ? 8.0 * N : 0.0) + (bo.sb.v ? 8.0 * N : 0.0));
                {
                    Prof p(c, kColFwdCheck, pass);
                    plan.col(za, -1, work, work, nullptr, HookMarkViol{bo.fb, viol, c.ctl}, st);
                }
                k_repair_freq_sparse<<<grid_for(vw), 256, 0, st>>>(viol, vw, delta_star, work, hg,
                                                                   g.d[0], g.d[1], freq_cur, esc_f);
                FFCZ_LAUNCH_CHECK();
                c.launches += 2;
                ++o.rounds;
                const Ctl hr = c.read_ctl();
                if (hr.dirty_s) sc_zero = false;
                if (!hr.dirty && dview) {
                    // clean round on the decoder view: no sample exceeded E and no component of
                    // its spectrum exceeded Delta (both against the ORIGINAL bounds): that is
                    // verify_bounds (archive.cpp:275-297), so vs = vf = 0
                    verified = true;
                    break;
                }
                if (!hr.dirty) {                                         // :161
                    // clean round: spat_cur / freq_cur are final and eps_v is their decoder
                    // view, so its forward transform completes verify_bounds
                    forward_row_mid(eps_v);
                    {
                        Prof p(c, kColFwdCheck, 16.0 * Nc);
                        plan.col(za, -1, work, work, nullptr, HookVerifyF{bo.fb, c.ctl}, st);
                    }
                    ++c.launches;
                    verified = true;
                    break;
                }
            }
        }
        if (!verified) {
            // apply_edits + verify_bounds on the decoder view (pipeline.cpp:174-176)
            FFCZ_CUDA_CHECK(cudaMemsetAsync(&c.ctl->vs_bits, 0, 2 * sizeof(unsigned long long), st));
            // half spectrum in, orig + dec + spat_cur, the view out, corrected, per-point E
            inverse_and_row(HookVerifyS<TI>{orig, dec, spat_cur, corrected, bo.sb, c.ctl},
                            16.0 * Nc + 2.0 * sizeof(TI) * N + 16.0 * N +
                                (corrected ? 8.0 * N : 0.0) + (bo.sb.v ? 8.0 * N : 0.0));
            {
                Prof p(c, kColFwdCheck, 16.0 * Nc);
                plan.col(za, -1, work, work, nullptr, HookVerifyF{bo.fb, c.ctl}, st);
            }
            c.launches += 1;
        }
    } else {
        if (converged) {
            for (int round = 0; round < 32; ++round) {                   // pipeline.cpp:116
                FFCZ_CUDA_CHECK(cudaMemsetAsync(&c.ctl->dirty, 0, sizeof(int), st));
                c2r_p(c, plan, freq_cur, work, fpart, invN);             // :125-133
                k_repair_spatial<TI><<<grid_for(N), 256, 0, st>>>(orig, dec, fpart, eps, N, bo.sb,
                                                                  spat_cur, eps_t, esc_s, c.ctl);
                r2c_p(c, plan, eps_t, work);                             // :137-138
                k_repair_freq<<<grid_for(Nc), 256, 0, st>>>(delta_star, work, hg, g.ndim, g.d[0],
                                                            g.d[1], bo.fb, freq_cur, esc_f, c.ctl);
                FFCZ_LAUNCH_CHECK();
                c.launches += 2;
                ++o.rounds;
                if (!c.read_ctl().dirty) break;                          // :161
            }
        }
        // read_archive + apply_edits + verify_bounds (pipeline.cpp:174-176) on the decoder view
        c2r_p(c, plan, freq_cur, work, fpart, invN);
        k_verify_spatial<TI><<<grid_for(N), 256, 0, st>>>(orig, dec, spat_cur, fpart, N, bo.sb,
                                                          corrected, eps_t, c.ctl);
        r2c_p(c, plan, eps_t, work);
        k_verify_freq<<<grid_for(Nc), 256, 0, st>>>(work, hg, bo.fb, c.ctl);
        FFCZ_LAUNCH_CHECK();
        c.launches += 2;
    }
    const Ctl h = c.read_ctl();
    o.vs = bitsd_host(h.vs_bits);
    o.vf = bitsd_host(h.vf_bits);
    o.verify_ok = (o.vs == 0.0 && o.vf == 0.0);
    o.act_s = h.act_s;
    o.act_f = h.act_f;
    return o;
}

double event_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    FFCZ_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

// FFCZ_DEBUG_TIMING=1: host timestamps of the phases of correct() on stderr (syncs the stream).
struct DebugClock {
    bool on = std::getenv("FFCZ_DEBUG_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void mark(ffcz_cuda_ctx& c, const char* what) {
        if (!on) return;
        c.sync();
        std::fprintf(stderr, "[ffcz] %-28s %9.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
};

template <class TI>
void finish_typed(ffcz_cuda_ctx& c, const Geometry& g, const ffcz_field_desc& fd, const TI* orig,
                  const TI* dec, const ffcz_bounds_desc& bd, const Bounds& bo, int m,
                  const LoopResult& lr, double* eps, double* S, double2* F, double2* delta_star,
                  const ffcz_cuda_options& opt, ffcz_cuda_result* out);

// Mixed policy, FP32 phase: the fused loop in FP32 (spectrum and
// iterate in FP32, half the bytes per pass; S and F accumulate in FP64 inside the hooks) until
// max_excess <= tau * peak (k_decide32), then eps <- FP64(eps32) and the FP64 loop continues
// with the reference control flow (run_loop, keep_moved).  Returns false when the shape has no
// fused FP32 path (the FP64 loop then runs alone).
bool run_phase32(ffcz_cuda_ctx& c, const Geometry& g, double* eps, const Bounds& bw, double fscale,
                 double tau, double* S, double2* F) {
    cudaStream_t st = c.st;
    FftPlan<float> plan{g, &c.tw32};
    if (!plan.fused_ok()) return false;
    const bool three_d = g.d[0] > 1;
    const int za = complete_axis(three_d, !bw.fb.re), mid = 1 - za;
    float* eps32 = c.b<float>("eps32", g.N);
    float2* spec = c.b<float2>("spec32", g.half_elems());
    unsigned char* moved = c.b<unsigned char>("f_moved", g.half_elems());
    FFCZ_CUDA_CHECK(cudaMemsetAsync(moved, 0, g.half_elems(), st));
    FFCZ_CUDA_CHECK(cudaMemcpyAsync(&c.ctl->tau, &tau, sizeof(double), cudaMemcpyHostToDevice, st));
    const int* gate = &c.ctl->switch_now;
    const float invN = static_cast<float>(1.0 / static_cast<double>(g.N));
    k_cast_to_float<<<grid_for(g.N), 256, 0, st>>>(eps, eps32, g.N);
    launch_row_r2c<float>(g.n2, eps32, g.n2, spec, g.P, g.rows, c.tw32, gate, st);
    if (three_d) plan.col(mid, -1, spec, spec, gate, HookNone{}, st);
    FFCZ_LAUNCH_CHECK();
    c.launches += three_d ? 3 : 2;
    auto body = [&]() {
        plan.col(za, -1, spec, spec, gate, HookFReduce{bw.fb, fscale, c.ctl}, st);          // K3a
        k_decide32<<<1, 1, 0, st>>>(c.ctl);
        plan.col(za, +1, spec, spec, gate, HookFClip<float>{bw.fb, fscale, F, c.ctl, moved}, st);
        if (three_d) plan.col(mid, +1, spec, spec, gate, HookNone{}, st);
        launch_row_c2r_hook<float>(g.n2, spec, g.P, eps32, g.n2, g.rows, invN, c.tw32, gate,
                                   HookSClip<float>{bw.sb, fscale, S, nullptr, c.ctl}, st);
        launch_row_r2c<float>(g.n2, eps32, g.n2, spec, g.P, g.rows, c.tw32, gate, st);
        if (three_d) plan.col(mid, -1, spec, spec, gate, HookNone{}, st);
        FFCZ_LAUNCH_CHECK();
        c.launches += three_d ? 7 : 5;
    };
    static const int kChunk[] = {1, 1, 2, 4};
    int ci = 0, issued = 0;
    std::vector<std::pair<cudaEvent_t, int>> inflight;
    auto issue_chunk = [&]() {
        const int n = kChunk[std::min(ci++, 3)];
        for (int i = 0; i < n; ++i) body();
        const int slot = issued % 2;
        k_export_ctl<<<1, 32, 0, st>>>(c.ctl, &c.hctl_dev[1 + slot]);
        FFCZ_LAUNCH_CHECK();
        cudaEvent_t ev = c.ev[4 + slot];
        FFCZ_CUDA_CHECK(cudaEventRecord(ev, st));
        inflight.push_back({ev, slot});
        ++issued;
    };
    issue_chunk();
    for (;;) {
        issue_chunk();
        auto p = inflight.front();
        inflight.erase(inflight.begin());
        FFCZ_CUDA_CHECK(cudaEventSynchronize(p.first));
        if (c.hctl[1 + p.second].switch_now) break;
    }
    // hand over: the FP64 loop starts from the FP32 iterate (its next check is in FP64)
    k_cast_to_double<<<grid_for(g.N), 256, 0, st>>>(eps32, eps, g.N);
    FFCZ_LAUNCH_CHECK();
    ++c.launches;
    return true;
}

template <class TI>
void correct_typed(ffcz_cuda_ctx& c, const Geometry& g, const ffcz_field_desc& fd,
                   const void* orig_in, const void* dec_in, const ffcz_bounds_desc& bd, int m,
                   uint64_t max_iters, const ffcz_cuda_options& opt, ffcz_cuda_result* out) {
    cudaStream_t st = c.st;
    const bool on_dev = opt.flags & FFCZ_INPUTS_ON_DEVICE;
    const long long N = g.N;
    DebugClock dbg;
    dbg.mark(c, "enter");
    FFCZ_CUDA_CHECK(cudaEventRecord(c.ev[0], st));
    const TI* orig = static_cast<const TI*>(orig_in);
    const TI* dec = static_cast<const TI*>(dec_in);
    if (!on_dev) {
        TI* o = c.b<TI>("in_orig", N);
        TI* d = c.b<TI>("in_dec", N);
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(o, orig_in, N * sizeof(TI), cudaMemcpyHostToDevice, st));
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(d, dec_in, N * sizeof(TI), cudaMemcpyHostToDevice, st));
        orig = o;
        dec = d;
    }
    const Bounds bo = upload_bounds(c, g, bd, on_dev, !(opt.flags & FFCZ_BOUNDS_VALIDATED));
    FFCZ_CUDA_CHECK(cudaEventRecord(c.ev[1], st));  // inputs resident
    dbg.mark(c, "inputs resident");

    // compute_error + preconditions (pipeline.cpp:31-42)
    k_ctl_init<<<1, 1, 0, st>>>(c.ctl, max_iters);
    double* eps = c.b<double>("eps", N);
    const double f = 1.0 - std::ldexp(1.0, -m);
    const double slack = 1.0 / (1.0 - std::ldexp(1.0, -m)) - 1.0 + 0x1p-20;
    // FP64 fused loop: eps0 is formed inside the first R2C (it is never needed in HBM unless the
    // loop converges at its first check); otherwise materialise it
    bool eps0_in_r2c = false;
    if (opt.policy == FFCZ_POLICY_FP64 && !(opt.flags & FFCZ_FORCE_UNFUSED) &&
        FftPlan<double>{g, &c.tw64}.fused_ok() && eps0_fusion_enabled() && m >= 1 && m <= 24) {
        Prof p(c, kRowR2C, (2.0 * sizeof(TI)) * N + 16.0 * g.Nc());
        eps0_in_r2c = launch_row_r2c_eps0<TI>(g.n2, orig, dec, c.b<double2>("spec", g.half_elems()),
                                              g.P, g.rows, c.tw64, bo.sb, f, slack, c.ctl, st);
    }
    if (!eps0_in_r2c) {
        Prof p(c, kElemPre, (2.0 * sizeof(TI) + 8.0) * N);
        k_eps0<TI><<<grid_for(N), 256, 0, st>>>(orig, dec, eps, N, bo.sb, f, slack, 1, c.ctl);
    }
    FFCZ_LAUNCH_CHECK();
    c.launches += 2;
    Ctl h = c.read_ctl();
    if (h.bad1 != ~0ull)
        throw Error(kValidation, "correct: decompressed data violates the declared spatial bound "
                                 "at index " + std::to_string(h.bad1));
    if (m < 1 || m > 24) throw Error(kValidation, "shrink_bounds requires 1 <= m <= 24");
    if (max_iters < 1) throw Error(kValidation, "alternating_projection: max_iters must be >= 1");
    if (h.bad2 != ~0ull)
        throw Error(kValidation, "alternating_projection: epsilon0 violates the spatial bound at "
                                 "index " + std::to_string(h.bad2));

    double* S = c.b<double>("S", N);
    double2* F = c.b<double2>("F", g.half_elems());
    FFCZ_CUDA_CHECK(cudaEventRecord(c.ev[2], st));
    const bool mixed = opt.policy == FFCZ_POLICY_MIXED && !(opt.flags & FFCZ_FORCE_UNFUSED) &&
                       run_phase32(c, g, eps, bo, f, opt.tau_switch, S, F);
    LoopResult lr = run_loop(c, g, eps, bo, f, !(opt.flags & FFCZ_FORCE_UNFUSED), S, F, true,
                             mixed, eps0_in_r2c);
    if (mixed) lr.passes32 = c.read_ctl().passes32;
    if (eps0_in_r2c && lr.passes == 0) {  // the final epsilon is eps0 itself
        k_eps0<TI><<<grid_for(N), 256, 0, st>>>(orig, dec, eps, N, bo.sb, f, slack, 0, c.ctl);
        FFCZ_LAUNCH_CHECK();
        ++c.launches;
    }
    FFCZ_CUDA_CHECK(cudaEventRecord(c.ev[3], st));
    finish_typed<TI>(c, g, fd, orig, dec, bd, bo, m, lr, eps, S, F,
                     c.b<double2>("spec", g.half_elems()), opt, out);
    out->report.wall_time_s = event_ms(c.ev[2], c.ev[3]) * 1e-3;
    out->t_h2d_ms = event_ms(c.ev[0], c.ev[1]);
    out->t_loop_ms = event_ms(c.ev[2], c.ev[3]);
    out->t_feasible_ms = event_ms(c.ev[1], c.ev[6]);
}

// Engine buffers whose contents are dead once the escape records are on the host (the loop and
// gate state; every call re-initialises them before reading) lent to the archive encoder: at
// 1024^3 its sort / code-length / bit-packing scratch is ~55 GB, which would otherwise sit on top
// of the ~100 GB of engine state.  Requests by name are served first-fit from the donors (a name
// asked again with a size that fits gets the same region, as c.buf does); what does not fit
// falls back to engine buffers of its own.
struct DonorArena {
    ffcz_cuda_ctx& c;
    std::vector<std::pair<char*, size_t>> blocks;
    std::vector<size_t> used;
    std::map<std::string, std::pair<void*, size_t>> named;
    void donate(const char* name) {
        auto it = c.bufs.find(name);
        if (it == c.bufs.end()) return;
        blocks.emplace_back(static_cast<char*>(it->second.first), it->second.second);
        used.push_back(0);
    }
    void* get(const char* nm, size_t bytes) {
        auto it = named.find(nm);
        if (it != named.end() && it->second.second >= bytes) return it->second.first;
        bytes = round_up(std::max<size_t>(bytes, 256), 256);
        for (size_t i = 0; i < blocks.size(); ++i)
            if (blocks[i].second - used[i] >= bytes) {
                void* p = blocks[i].first + used[i];
                used[i] += bytes;
                named[nm] = {p, bytes};
                return p;
            }
        void* p = c.buf(std::string("arc_own_") + nm, bytes);
        named[nm] = {p, bytes};
        return p;
    }
};

// FFCZ_OUTER_DEVICE archives (archive_dev.cu) into the pinned result pool; `donors` names engine
// buffers that are dead at this point (DonorArena)
void device_archive(ffcz_cuda_ctx& c, const DevArchiveInput& ai, ffcz_cuda_result* r,
                    std::initializer_list<const char*> donors = {}) {
    DonorArena arena{c, {}, {}, {}};
    for (const char* d : donors) arena.donate(d);
    DevScratch ds{c.st, [&](const char* nm, size_t b) { return arena.get(nm, b); }};
    const auto t0 = std::chrono::steady_clock::now();
    std::uint64_t len = 0;
    write_archive_device(ds, ai, [](size_t n) { return pinned().get(n); }, &r->archive, &len);
    r->archive_len = len;
    r->t_archive_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// Residual, FP64 gate and products of one field whose projection loop has run (pipeline.cpp:
// 46-176): shared by correct() and the batched-frame path (each frame's state in the batch
// arrays).  Records ev[3] -> ev[6] around the gate.
template <class TI>
void finish_typed(ffcz_cuda_ctx& c, const Geometry& g, const ffcz_field_desc& fd, const TI* orig,
                  const TI* dec, const ffcz_bounds_desc& bd, const Bounds& bo, int m,
                  const LoopResult& lr, double* eps, double* S, double2* F, double2* delta_star,
                  const ffcz_cuda_options& opt, ffcz_cuda_result* out) {
    cudaStream_t st = c.st;
    const bool on_dev = opt.flags & FFCZ_INPUTS_ON_DEVICE;
    const long long N = g.N;
    const double f = 1.0 - std::ldexp(1.0, -m);
    DebugClock dbg;
    FFCZ_CUDA_CHECK(cudaEventRecord(c.ev[3], st));
    // residual_s (projection.cpp:129-133): after an FP64 s-clip every |eps| <= E exactly
    // (clamp), so it is 0 unless the final epsilon is eps0 or an FP32 iterate
    FFCZ_CUDA_CHECK(cudaMemsetAsync(&c.ctl->res_s_bits, 0, sizeof(unsigned long long), st));
    if (lr.passes == lr.passes32) {
        Prof p(c, kElemPre, 8.0 * N);
        k_residual_s<<<grid_for(N), 256, 0, st>>>(eps, N, bo.sb, f, c.ctl);
        ++c.launches;
    }

    // the FP64 corrected field is only materialised when the caller asks for it (the reference's
    // CorrectionResult carries no field; verify needs only its epsilon)
    double* corrected = (opt.flags & FFCZ_WANT_CORRECTED) ? c.b<double>("corrected", N) : nullptr;
    // flags / codes to the host: asked for, or the host archive writer needs them (the device
    // archive encodes them where they are); escapes go to the host for either archive
    const bool device_outer = opt.zlib_level == FFCZ_OUTER_DEVICE;
    const bool want_edits = (opt.flags & FFCZ_WANT_EDITS) ||
                            ((opt.flags & FFCZ_WANT_ARCHIVE) && !device_outer);
    const bool want_escapes = want_edits || (opt.flags & FFCZ_WANT_ARCHIVE);
    const long long ws = (N + 31) / 32, wf = (g.Nc() + 31) / 32;
    bool copy_pending = false;
    auto on_codes = [&](unsigned long long ns, unsigned long long nf) {
        if (!want_edits) return;
        out->spatial_flag_bytes = (N + 7) / 8;
        out->frequency_flag_bytes = (g.Nc() + 7) / 8;
        out->spatial_flags = static_cast<uint8_t*>(pinned().get(out->spatial_flag_bytes + 1));
        out->frequency_flags = static_cast<uint8_t*>(pinned().get(out->frequency_flag_bytes + 1));
        out->spatial_codes = static_cast<int32_t*>(pinned().get(ns * 4 + 4));
        out->frequency_codes = static_cast<int32_t*>(pinned().get(nf * 8 + 4));
        FFCZ_CUDA_CHECK(cudaEventRecord(c.ev_codes, st));
        FFCZ_CUDA_CHECK(cudaStreamWaitEvent(c.st_copy, c.ev_codes, 0));
        cudaStream_t cs = c.st_copy;
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(out->spatial_flags, c.b<unsigned>("keep_s", ws),
                                        out->spatial_flag_bytes, cudaMemcpyDeviceToHost, cs));
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(out->frequency_flags, c.b<unsigned>("keep_f", wf),
                                        out->frequency_flag_bytes, cudaMemcpyDeviceToHost, cs));
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(out->spatial_codes, c.b<int>("codes_s", N), ns * 4,
                                        cudaMemcpyDeviceToHost, cs));
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(out->frequency_codes, c.b<int>("codes_f", 2 * g.Nc()),
                                        nf * 8, cudaMemcpyDeviceToHost, cs));
        copy_pending = true;
    };
    const GateOut go = run_gate<TI>(c, g, orig, dec, bo, m, lr, eps, S, F, delta_star, corrected,
                                    on_codes);
    FFCZ_CUDA_CHECK(cudaEventRecord(c.ev[6], st));
    dbg.mark(c, "gate done");
    const Ctl h = c.read_ctl();

    out->report.iterations = std::max<unsigned long long>(lr.passes, 1);
    out->report.active_spatial = go.act_s;
    out->report.active_frequency = go.act_f;
    out->report.converged = lr.converged;
    out->report.residual_f = lr.residual_f;
    out->report.residual_s = bitsd_host(h.res_s_bits);
    out->iterations_fp32 = lr.passes32;
    out->iterations_fp64 = lr.passes - lr.passes32;
    out->escape_rounds = go.rounds;
    out->verify_ok = go.verify_ok;
    out->verify_max_spatial_excess = go.vs;
    out->verify_max_freq_excess = go.vf;
    out->n_spatial = go.n_keep_s;
    out->n_frequency = go.n_keep_f;
    out->t_gate_ms = event_ms(c.ev[3], c.ev[6]);

    // ---- products to the host -------------------------------------------------------------
    const auto t_d2h0 = std::chrono::steady_clock::now();
    const EscapeRec* escape_dev = nullptr;
    unsigned long long n_esc = 0;
    {
        unsigned long long* idx = c.b<unsigned long long>("idx", std::max(N, g.Nc()));
        dbg.mark(c, "escape section start");
        const unsigned long long ns = compact_bits(c, c.b<unsigned>("esc_s", ws), ws, idx);
        EscapeRec* recs = nullptr;
        if (ns) {
            recs = c.b<EscapeRec>("esc_recs", ns);
            k_escape_records_s<<<grid_for(ns), 256, 0, st>>>(idx, ns, c.b<double>("spat_cur", N), recs);
            FFCZ_LAUNCH_CHECK();
        }
        const unsigned long long nf = compact_bits(c, c.b<unsigned>("esc_f", wf), wf, idx);
        n_esc = ns + nf;
        if (n_esc) {
            // the spatial records may have to move when the buffer grows: rebuild them after
            EscapeRec* all = c.b<EscapeRec>("esc_recs_all", n_esc);
            if (ns) FFCZ_CUDA_CHECK(cudaMemcpyAsync(all, recs, ns * sizeof(EscapeRec), cudaMemcpyDeviceToDevice, st));
            if (nf) {
                k_escape_records_f<<<grid_for(nf), 256, 0, st>>>(
                    idx, nf, c.b<double2>("freq_cur", g.half_elems()), g.hg(), all + ns);
                FFCZ_LAUNCH_CHECK();
            }
            escape_dev = all;
        }
        dbg.mark(c, "escape records built");
    }
    std::vector<ffcz_cuda_escape> escapes;  // only for the archive writer below
    out->escape_count = n_esc;
    dbg.mark(c, "escapes compacted");
    if (want_escapes) {
        out->escapes = static_cast<ffcz_cuda_escape*>(
            pinned().get(sizeof(ffcz_cuda_escape) * (n_esc + 1)));
        if (n_esc)
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(out->escapes, escape_dev, n_esc * sizeof(EscapeRec),
                                            cudaMemcpyDeviceToHost, st));
    }
    dbg.mark(c, "edits to host");
    if (opt.flags & FFCZ_WANT_CORRECTED) {
        out->corrected = static_cast<double*>(pinned().get(N * sizeof(double)));
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(out->corrected, corrected, N * sizeof(double),
                                        cudaMemcpyDeviceToHost, st));
    }
    c.sync();
    if (copy_pending) FFCZ_CUDA_CHECK(cudaStreamSynchronize(c.st_copy));
    const auto t_d2h1 = std::chrono::steady_clock::now();
    out->t_d2h_ms = std::chrono::duration<double, std::milli>(t_d2h1 - t_d2h0).count();
    dbg.mark(c, "corrected to host");

    if ((opt.flags & FFCZ_WANT_ARCHIVE) && opt.zlib_level == FFCZ_OUTER_DEVICE) {
        // every stream from the resident flags / codes; bound arrays where the caller holds them
        DevArchiveInput ai{};
        ai.ndim = fd.ndim;
        for (int a = 0; a < fd.ndim; ++a) ai.dims[a] = fd.dims[a];
        ai.precision = fd.precision;
        ai.spatial_per_point = bd.spatial_per_point;
        ai.spatial_global = bd.spatial_global;
        ai.spatial_values = bd.spatial_values;
        ai.freq_per_component = bd.freq_per_component;
        ai.freq_global = bd.freq_global;
        ai.freq_re = bd.freq_re;
        ai.freq_im = bd.freq_im;
        ai.bounds_on_device = on_dev;
        ai.m = m;
        ai.converged = lr.converged;
        ai.spatial_flags = reinterpret_cast<const unsigned char*>(c.b<unsigned>("keep_s", ws));
        ai.spatial_flag_bytes = (N + 7) / 8;
        ai.frequency_flags = reinterpret_cast<const unsigned char*>(c.b<unsigned>("keep_f", wf));
        ai.frequency_flag_bytes = (g.Nc() + 7) / 8;
        ai.n_spatial = go.n_keep_s;
        ai.n_frequency = go.n_keep_f;
        ai.spatial_codes = c.b<int>("codes_s", N);
        ai.frequency_codes = c.b<int>("codes_f", 2 * g.Nc());
        ai.escapes = out->escapes;
        ai.n_escapes = n_esc;
        // (escape records and the corrected field are on the host: c.sync() above)
        device_archive(c, ai, out,
                       {"eps_tilde", "spat_cur", "freq_cur", "spec", "F", "S", "eps", "idx",
                        "eps_verify", "esc_recs", "esc_recs_all", "real_tmp"});
        return;
    }
    if (opt.flags & FFCZ_WANT_ARCHIVE) {
        // header bounds must be the caller's full arrays (host)
        std::vector<double> e_host, re_host, im_host;
        const double* e_vals = bd.spatial_values;
        const double* re_vals = bd.freq_re;
        const double* im_vals = bd.freq_im;
        if (on_dev) {
            if (bd.spatial_per_point) {
                e_host.resize(N);
                FFCZ_CUDA_CHECK(cudaMemcpy(e_host.data(), bd.spatial_values, N * 8, cudaMemcpyDeviceToHost));
                e_vals = e_host.data();
            }
            if (bd.freq_per_component) {
                re_host.resize(N);
                FFCZ_CUDA_CHECK(cudaMemcpy(re_host.data(), bd.freq_re, N * 8, cudaMemcpyDeviceToHost));
                re_vals = re_host.data();
                if (bd.freq_im == bd.freq_re) {
                    im_vals = re_vals;
                } else {
                    im_host.resize(N);
                    FFCZ_CUDA_CHECK(cudaMemcpy(im_host.data(), bd.freq_im, N * 8, cudaMemcpyDeviceToHost));
                    im_vals = im_host.data();
                }
            }
        }
        std::vector<ffcz_host::EscapeRec> er(n_esc);
        for (size_t i = 0; i < n_esc; ++i)
            er[i] = {out->escapes[i].frequency != 0, out->escapes[i].index, out->escapes[i].re,
                     out->escapes[i].im};
        ffcz_host::ArchiveInput ai{};
        ai.ndim = fd.ndim;
        for (int a = 0; a < fd.ndim; ++a) ai.dims[a] = fd.dims[a];
        ai.precision = fd.precision;
        ai.spatial_per_point = bd.spatial_per_point;
        ai.spatial_global = bd.spatial_global;
        ai.spatial_values = e_vals;
        ai.freq_per_component = bd.freq_per_component;
        ai.freq_global = bd.freq_global;
        ai.freq_re = re_vals;
        ai.freq_im = im_vals;
        ai.m = m;
        ai.converged = lr.converged;
        ai.spatial_flags = out->spatial_flags;
        ai.spatial_flag_bytes = out->spatial_flag_bytes;
        ai.frequency_flags = out->frequency_flags;
        ai.frequency_flag_bytes = out->frequency_flag_bytes;
        ai.n_spatial = go.n_keep_s;
        ai.n_frequency = go.n_keep_f;
        ai.spatial_codes = out->spatial_codes;
        ai.frequency_codes = out->frequency_codes;
        ai.escapes = er.data();
        ai.n_escapes = er.size();
        ai.zlib_level = opt.zlib_level;
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<uint8_t> sp, fp;
        if (opt.flags & FFCZ_DEVICE_ENCODE) {
            // Huffman payloads on the device from the resident codes; host does the outer stage
            DevScratch ds{st, [&](const char* nm, size_t b) { return c.buf(nm, b); }};
            auto enc = [&](const int* dcodes, unsigned long long n, std::vector<uint8_t>& dst) {
                unsigned char* dp = nullptr;
                const unsigned long long len = huffman_encode_device(ds, dcodes, n, &dp);
                dst.resize(len);
                FFCZ_CUDA_CHECK(cudaMemcpyAsync(dst.data(), dp, len, cudaMemcpyDeviceToHost, st));
                c.sync();
            };
            enc(c.b<int>("codes_s", N), go.n_keep_s, sp);
            enc(c.b<int>("codes_f", 2 * g.Nc()), 2 * go.n_keep_f, fp);
            ai.spatial_payload = sp.data();
            ai.spatial_payload_len = sp.size();
            ai.frequency_payload = fp.data();
            ai.frequency_payload_len = fp.size();
        }
        std::vector<uint8_t> bytes = ffcz_host::write_archive(ai);
        out->t_archive_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        out->archive_len = bytes.size();
        out->archive = static_cast<uint8_t*>(pinned().get(bytes.size() + 1));
        std::memcpy(out->archive, bytes.data(), bytes.size());
    }
}

} // namespace

double bitsd_host(unsigned long long b) {
    double d;
    std::memcpy(&d, &b, sizeof(d));
    return d;
}

template <class T>
static void r2c_dev(ffcz_cuda_ctx& c, Twiddles<T>& tw, const Geometry& g, const T* x, cplx<T>* out) {
    cplx<T>* half = static_cast<cplx<T>*>(c.buf("dev_half", g.half_elems() * sizeof(cplx<T>)));
    FftPlan<T> plan{g, &tw};
    plan.r2c(x, half, nullptr, c.st);
    FFCZ_CUDA_CHECK(cudaMemcpy2DAsync(out, g.H * sizeof(cplx<T>), half, g.P * sizeof(cplx<T>),
                                      g.H * sizeof(cplx<T>), g.rows, cudaMemcpyDeviceToDevice, c.st));
    c.sync();
}

template <class T>
static void c2r_dev(ffcz_cuda_ctx& c, Twiddles<T>& tw, const Geometry& g, const cplx<T>* in, T* x) {
    cplx<T>* half = static_cast<cplx<T>*>(c.buf("dev_half", g.half_elems() * sizeof(cplx<T>)));
    FFCZ_CUDA_CHECK(cudaMemcpy2DAsync(half, g.P * sizeof(cplx<T>), in, g.H * sizeof(cplx<T>),
                                      g.H * sizeof(cplx<T>), g.rows, cudaMemcpyDeviceToDevice, c.st));
    FftPlan<T> plan{g, &tw};
    plan.c2r(half, half, x, static_cast<T>(1.0 / static_cast<double>(g.N)), nullptr, c.st);
    c.sync();
}


// ================================ C-ABI ===========================================================

namespace {

// Runs fn(lane_ctx, item) for items [0, n) on `nl` lane sub-contexts (host threads, one stream
// each), ordered after the work already queued on ctx->st; ctx->st waits for every lane before
// returning.  The first exception of any lane is rethrown.
void ensure_lanes(ffcz_cuda_ctx* ctx, int nl) {
    while (static_cast<int>(ctx->lanes.size()) < nl) {
        ffcz_cuda_ctx* l = nullptr;
        if (ffcz_cuda_create(&l, ctx->device, nullptr) != kOk)
            throw Error(kCuda, std::string("lane context: ") + g_last_error);
        ctx->lanes.push_back(l);
    }
}

// start: event the lanes wait for (default: recorded now on ctx->st); join_stream: make ctx->st
// wait for the lanes at the end (off when the caller joins on the host instead)
void run_on_lanes(ffcz_cuda_ctx* ctx, int nl, uint64_t n,
                  const std::function<void(ffcz_cuda_ctx&, uint64_t)>& fn,
                  cudaEvent_t start = nullptr, bool join_stream = true) {
    ensure_lanes(ctx, nl);
    if (!start) {
        FFCZ_CUDA_CHECK(cudaEventRecord(ctx->ev[7], ctx->st));
        start = ctx->ev[7];
    }
    for (int i = 0; i < nl; ++i) {
        ffcz_cuda_ctx* l = ctx->lanes[i];
        FFCZ_CUDA_CHECK(cudaStreamWaitEvent(l->st, start, 0));
        l->call_flags = ctx->call_flags;
        if (l->prof_on != ctx->prof_on) {
            l->prof_on = ctx->prof_on;
            l->prof.clear();
            l->ev_used = 0;
        }
    }
    std::atomic<uint64_t> next{0};
    std::mutex err_mu;
    int err_status = kOk;
    std::string err_msg;
    auto work = [&](ffcz_cuda_ctx* l) {
        try {
            FFCZ_CUDA_CHECK(cudaSetDevice(l->device));
            std::lock_guard<std::mutex> lk(l->mu);
            for (;;) {
                const uint64_t i = next.fetch_add(1);
                if (i >= n) break;
                {
                    std::lock_guard<std::mutex> ek(err_mu);
                    if (err_status != kOk) break;
                }
                fn(*l, i);
            }
        } catch (const Error& e) {
            std::lock_guard<std::mutex> ek(err_mu);
            if (err_status == kOk) { err_status = e.status; err_msg = e.what(); }
        } catch (const std::exception& e) {
            std::lock_guard<std::mutex> ek(err_mu);
            if (err_status == kOk) { err_status = kCuda; err_msg = e.what(); }
        }
    };
    std::vector<std::thread> th;
    for (int i = 1; i < nl; ++i) th.emplace_back(work, ctx->lanes[i]);
    work(ctx->lanes[0]);
    for (auto& t : th) t.join();
    for (int i = 0; join_stream && i < nl; ++i) {
        ffcz_cuda_ctx* l = ctx->lanes[i];
        FFCZ_CUDA_CHECK(cudaEventRecord(l->ev[7], l->st));
        FFCZ_CUDA_CHECK(cudaStreamWaitEvent(ctx->st, l->ev[7], 0));
    }
    if (err_status != kOk) throw Error(err_status, "frame batch: " + err_msg);
}

// FFCZ_FRAMES_FUSED=0: always use per-frame correct() on lanes
inline bool frames_fused_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_FRAMES_FUSED");
        return !(e && e[0] == '0');
    }();
    return on;
}

// FFCZ_FRAMES_BATCHED_GATE=0: run each frame's FP64 gate on the lanes instead
inline bool frames_batched_gate_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FFCZ_FRAMES_BATCHED_GATE");
        return !(e && e[0] == '0');
    }();
    return on;
}

// The FP64 gate (pipeline.cpp:46-176) of every frame of a group at once: each pass of the
// single-field gate (run_gate, fused branch) runs over the stack with per-frame bounds and masks
// (kernels.cuh FrameGate / FrameMask hooks): F rebuild, quantisation + flags, codes, escape
// repair rounds (frames leave the rounds as they come clean; their verify runs on that round's
// decoder view), apply + verify for the rest, escapes; then per-frame products.
template <class TI>
void gate_frames(ffcz_cuda_ctx& c, const Geometry& gf, const ffcz_field_desc& fd, long long Gc,
                 uint64_t g0, const TI* orig, const TI* dec, const ffcz_bounds_desc* bd, int m,
                 const std::vector<FrameCtl>& hfc, const std::vector<double>& hE,
                 const std::vector<double>& hD, const double* dE, const double* dD, double* eps,
                 double* S, double2* F, double2* spec, const unsigned char* moved,
                 const ffcz_cuda_options& opt, double t_in, double t_loop, ffcz_cuda_result* out,
                 const std::function<std::string(const char*)>& nm) {
    cudaStream_t st = c.st;
    const long long Nf = gf.N, Hf = gf.half_elems(), n1 = gf.d[1], n2 = gf.n2;
    const long long Ncf = gf.Nc();                      // half-grid entries per frame
    const uint64_t dimsb[3] = {static_cast<uint64_t>(Gc), static_cast<uint64_t>(n1),
                               static_cast<uint64_t>(n2)};
    const Geometry gb = make_geometry(3, dimsb, kPitchAlign);
    const HalfGeom hg = gb.hg();
    FftPlan<double> plan{gb, &c.tw64};
    const long long N = Gc * Nf, Nc = Gc * Ncf;
    const long long ws = N / 32, wf = Nc / 32;          // frames are whole words (n1 >= 64)
    const double invN = 1.0 / static_cast<double>(Nf);
    FFCZ_CUDA_CHECK(cudaEventRecord(c.ev[3], st));
    // per-frame state and masks
    FrameGate* fg = c.b<FrameGate>(nm("fg_gate").c_str(), Gc);
    FFCZ_CUDA_CHECK(cudaMemsetAsync(fg, 0, sizeof(FrameGate) * Gc, st));
    int* mask = c.b<int>(nm("fg_mask").c_str(), Gc);
    std::vector<int> hmask(Gc);
    auto set_mask = [&](const std::function<bool(long long)>& pred) {
        bool any = false;
        for (long long i = 0; i < Gc; ++i) any |= (hmask[i] = pred(i) ? 1 : 0) != 0;
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(mask, hmask.data(), 4 * Gc, cudaMemcpyHostToDevice, st));
        c.sync();  // hmask is reused
        return any;
    };
    const FrameMask fmk{mask, n1};
    double* spat_cur = c.b<double>(nm("fg_spat").c_str(), N);
    double2* freq_cur = c.b<double2>(nm("fg_freq").c_str(), Gc * Hf);
    double2* work = c.b<double2>(nm("fg_work").c_str(), Gc * Hf);
    double* eps_t = c.b<double>(nm("fg_eps_t").c_str(), N);
    double* eps_v = c.b<double>(nm("fg_eps_v").c_str(), N);
    unsigned* keep_s = c.b<unsigned>(nm("fg_keep_s").c_str(), ws);
    unsigned* esc_s = c.b<unsigned>(nm("fg_esc_s").c_str(), ws);
    unsigned* keep_f = c.b<unsigned>(nm("fg_keep_f").c_str(), wf);
    unsigned* esc_f = c.b<unsigned>(nm("fg_esc_f").c_str(), wf);
    const long long vw = (Gc * Hf + 31) / 32;
    unsigned* viol = c.b<unsigned>(nm("fg_viol").c_str(), vw);
    int* codes_s = c.b<int>(nm("fg_codes_s").c_str(), N);
    int* codes_f = c.b<int>(nm("fg_codes_f").c_str(), 2 * Nc);
    double* corrected = (opt.flags & FFCZ_WANT_CORRECTED) ? c.b<double>(nm("fg_corr").c_str(), N) : nullptr;

    // F rebuild for the frames whose loop ran >= 2 clip passes (HookFRebuild)
    if (set_mask([&](long long i) { return hfc[i].passes >= 2; })) {
        k_eps0_plus_s<TI><<<grid_for(N), 256, 0, st>>>(orig, dec, S, eps_t, N);
        launch_row_r2c_hook<double>(n2, eps_t, n2, work, gb.P, gb.rows, c.tw64, nullptr,
                                    HookMaskB<true>{fmk}, st);
        plan.col(1, -1, work, work, nullptr, HookFRebuildB{fmk, spec, F, moved}, st);
        FFCZ_LAUNCH_CHECK();
        c.launches += 3;
    }
    // quantisation + flags + overflow escapes (editset.cpp:43-133, pipeline.cpp:57-106)
    k_gate_spatial_frames<<<grid_for(N), 256, 0, st>>>(S, N, Nf, dE, m, spat_cur, keep_s, esc_s, fg);
    k_gate_freq_frames<<<grid_for(Nc), 256, 0, st>>>(F, hg, n1, dD, m, freq_cur, keep_f, esc_f, fg);
    FFCZ_LAUNCH_CHECK();
    c.launches += 2;
    auto codes_stack = [&](const unsigned* words, long long nwords, const char* name, auto launch) {
        const long long nblk = std::max<long long>(1, (nwords + 1023) / 1024);
        unsigned long long* cnt = c.b<unsigned long long>(nm(name).c_str(), nblk + 1);
        k_popc_blocks<<<static_cast<unsigned>(nblk), 1024, 0, st>>>(words, nwords, cnt);
        k_scan_blocks<<<1, 1024, 0, st>>>(cnt, nblk, &c.ctl->count_a);
        launch(static_cast<unsigned>(nblk), cnt);
        FFCZ_LAUNCH_CHECK();
        c.launches += 3;
    };
    codes_stack(keep_s, ws, "fg_cnt_s", [&](unsigned nb, unsigned long long* o) {
        k_codes_spatial_frames<<<nb, 1024, 0, st>>>(keep_s, ws, o, S, Nf, dE, m, codes_s);
    });
    codes_stack(keep_f, wf, "fg_cnt_f", [&](unsigned nb, unsigned long long* o) {
        k_codes_freq_frames<<<nb, 1024, 0, st>>>(keep_f, wf, o, F, hg, n1, dD, m, codes_f);
    });
    // per-frame kept counts -> code offsets
    unsigned long long* pc = c.b<unsigned long long>(nm("fg_pc").c_str(), 2 * Gc);
    k_frame_popc<<<static_cast<unsigned>(std::min<long long>(Gc, 1184)), 256, 0, st>>>(keep_s, Nf / 32, Gc, pc);
    k_frame_popc<<<static_cast<unsigned>(std::min<long long>(Gc, 1184)), 256, 0, st>>>(keep_f, Ncf / 32, Gc, pc + Gc);
    FFCZ_LAUNCH_CHECK();
    std::vector<unsigned long long> hpc(2 * Gc);
    FFCZ_CUDA_CHECK(cudaMemcpyAsync(hpc.data(), pc, 16 * Gc, cudaMemcpyDeviceToHost, st));
    c.sync();
    std::vector<unsigned long long> off_s(Gc + 1, 0), off_f(Gc + 1, 0);
    for (long long i = 0; i < Gc; ++i) {
        off_s[i + 1] = off_s[i] + hpc[i];
        off_f[i + 1] = off_f[i] + hpc[Gc + i];
    }

    // escape-repair rounds (pipeline.cpp:111-163) for the converged frames
    std::vector<int> rounds(Gc, 0), verified(Gc, 0);
    const bool dview = decoder_view_repair(c);
    std::vector<double> vs(Gc, 0.0), vf(Gc, 0.0);
    std::vector<int> active(Gc);
    for (long long i = 0; i < Gc; ++i) active[i] = hfc[i].converged;
    std::vector<FrameGate> hg_gate(Gc);
    auto read_gate = [&]() {
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(hg_gate.data(), fg, sizeof(FrameGate) * Gc,
                                        cudaMemcpyDeviceToHost, st));
        c.sync();
    };
    auto reset_round = [&]() {  // dirty / dirty_s / vs / vf of every frame (act counts kept)
        k_frame_gate_reset<<<grid_for(Gc), 256, 0, st>>>(fg, Gc);
        FFCZ_LAUNCH_CHECK();
    };
    for (int round = 0; round < 32; ++round) {
        if (!set_mask([&](long long i) { return active[i] != 0; })) break;
        reset_round();
        FFCZ_CUDA_CHECK(cudaMemsetAsync(viol, 0, vw * sizeof(unsigned), st));
        plan.col(1, +1, freq_cur, work, nullptr, HookMaskB<false>{fmk}, st);
        HookRepairVerifySB<TI> hrv{fmk, dE, fg, orig, dec, spat_cur, eps, esc_s, corrected, eps_v};
        hrv.dview = dview;
        launch_row_c2r_hook<double>(n2, work, gb.P, eps_t, n2, gb.rows, invN, c.tw64, nullptr, hrv,
                                    st);
        launch_row_r2c_hook<double>(n2, eps_t, n2, work, gb.P, gb.rows, c.tw64, nullptr,
                                    HookMaskB<true>{fmk}, st);
        plan.col(1, -1, work, work, nullptr, HookMarkViolB{fmk, dD, fg, viol}, st);
        k_repair_freq_sparse_frames<<<grid_for(vw), 256, 0, st>>>(viol, vw, spec, work, hg, n1,
                                                                  freq_cur, esc_f);
        FFCZ_LAUNCH_CHECK();
        c.launches += 5;
        read_gate();
        bool any_clean = false;
        for (long long i = 0; i < Gc; ++i) {
            if (!active[i]) continue;
            ++rounds[i];
            if (!hg_gate[i].dirty) {          // clean round: its decoder view is final (:161)
                vs[i] = bitsd_host(hg_gate[i].vs_bits);
                active[i] = 0;
                // decoder-view repair: the clean round checked v and FFT(v) against the original
                // bounds, i.e. verify_bounds itself (vf = 0)
                verified[i] = dview ? 2 : 1;
                any_clean = true;
            }
        }
        if (any_clean && !dview) {  // verify the frames that came clean on this round's eps_v
            set_mask([&](long long i) { return verified[i] == 1; });
            launch_row_r2c_hook<double>(n2, eps_v, n2, work, gb.P, gb.rows, c.tw64, nullptr,
                                        HookMaskB<true>{fmk}, st);
            plan.col(1, -1, work, work, nullptr, HookVerifyFB{fmk, dD, fg}, st);
            FFCZ_LAUNCH_CHECK();
            c.launches += 2;
            read_gate();
            for (long long i = 0; i < Gc; ++i)
                if (verified[i] == 1) {
                    vf[i] = bitsd_host(hg_gate[i].vf_bits);
                    verified[i] = 2;
                }
        }
    }
    // apply_edits + verify_bounds for the rest (not converged, or 32 dirty rounds)
    if (set_mask([&](long long i) { return verified[i] == 0; })) {
        reset_round();
        plan.col(1, +1, freq_cur, work, nullptr, HookMaskB<false>{fmk}, st);
        launch_row_c2r_hook<double>(n2, work, gb.P, eps_v, n2, gb.rows, invN, c.tw64, nullptr,
            HookVerifySB<TI>{fmk, dE, fg, orig, dec, spat_cur, corrected}, st);
        launch_row_r2c_hook<double>(n2, eps_v, n2, work, gb.P, gb.rows, c.tw64, nullptr,
                                    HookMaskB<true>{fmk}, st);
        plan.col(1, -1, work, work, nullptr, HookVerifyFB{fmk, dD, fg}, st);
        FFCZ_LAUNCH_CHECK();
        c.launches += 4;
        read_gate();
        for (long long i = 0; i < Gc; ++i)
            if (verified[i] == 0) {
                vs[i] = bitsd_host(hg_gate[i].vs_bits);
                vf[i] = bitsd_host(hg_gate[i].vf_bits);
            }
    }
    read_gate();  // act counts
    // residual_s: 0 after an s-clip; frames that converged at their first check keep eps0
    std::vector<double> res_s(Gc, 0.0);
    for (long long i = 0; i < Gc; ++i)
        if (hfc[i].passes == 0) {
            FFCZ_CUDA_CHECK(cudaMemsetAsync(&c.ctl->res_s_bits, 0, 8, st));
            k_residual_s<<<grid_for(Nf), 256, 0, st>>>(eps + i * Nf, Nf, SpatialB{nullptr, hE[i]},
                                                       1.0 - std::ldexp(1.0, -m), c.ctl);
            FFCZ_LAUNCH_CHECK();
            res_s[i] = bitsd_host(c.read_ctl().res_s_bits);
        }
    FFCZ_CUDA_CHECK(cudaEventRecord(c.ev[6], st));

    // escapes of the whole stack (ascending global index: frame order, spatial then frequency
    // within a frame after the split below)
    unsigned long long* idx = c.b<unsigned long long>(nm("fg_idx").c_str(), std::max(N, Nc));
    const unsigned long long ns = compact_bits(c, esc_s, ws, idx);
    std::vector<EscapeRec> rs(ns), rf;
    if (ns) {
        EscapeRec* r = c.b<EscapeRec>(nm("fg_recs").c_str(), ns);
        k_escape_records_s<<<grid_for(ns), 256, 0, st>>>(idx, ns, spat_cur, r);
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(rs.data(), r, ns * sizeof(EscapeRec), cudaMemcpyDeviceToHost, st));
    }
    c.sync();
    const unsigned long long nf = compact_bits(c, esc_f, wf, idx);
    rf.resize(nf);
    if (nf) {
        EscapeRec* r = c.b<EscapeRec>(nm("fg_recs").c_str(), nf);
        k_escape_records_f<<<grid_for(nf), 256, 0, st>>>(idx, nf, freq_cur, hg, r);
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(rf.data(), r, nf * sizeof(EscapeRec), cudaMemcpyDeviceToHost, st));
    }
    c.sync();
    std::vector<std::vector<ffcz_cuda_escape>> esc(Gc);
    auto rec = [](int freq, uint64_t index, double re, double im) {
        ffcz_cuda_escape x;
        std::memset(&x, 0, sizeof(x));  // the padding after `frequency` travels to the caller
        x.frequency = freq;
        x.index = index;
        x.re = re;
        x.im = im;
        return x;
    };
    for (const EscapeRec& e : rs) {
        const long long f = static_cast<long long>(e.index / Nf);
        esc[f].push_back(rec(0, e.index - f * Nf, e.re, e.im));
    }
    for (const EscapeRec& e : rf) {
        const long long f = static_cast<long long>(e.index / Ncf);
        esc[f].push_back(rec(1, e.index - f * Ncf, e.re, e.im));
    }

    // per-frame products
    const bool want_edits = opt.flags & (FFCZ_WANT_EDITS | FFCZ_WANT_ARCHIVE);
    const double t_gate = event_ms(c.ev[3], c.ev[6]);
    for (long long i = 0; i < Gc; ++i) {
        ffcz_cuda_result* r = &out[g0 + i];
        r->report.iterations = std::max<unsigned long long>(hfc[i].passes, 1);
        r->report.active_spatial = hg_gate[i].act_s;
        r->report.active_frequency = hg_gate[i].act_f;
        r->report.converged = hfc[i].converged;
        r->report.residual_f = hfc[i].residual_f;
        r->report.residual_s = res_s[i];
        r->iterations_fp64 = hfc[i].passes;
        r->escape_rounds = rounds[i];
        r->escape_count = esc[i].size();
        r->verify_ok = vs[i] == 0.0 && vf[i] == 0.0;
        r->verify_max_spatial_excess = vs[i];
        r->verify_max_freq_excess = vf[i];
        r->n_spatial = hpc[i];
        r->n_frequency = hpc[Gc + i];
        r->t_h2d_ms = t_in / Gc;
        r->t_loop_ms = t_loop / Gc;
        r->t_gate_ms = t_gate / Gc;
        r->t_feasible_ms = r->t_loop_ms + r->t_gate_ms;
        r->report.wall_time_s = r->t_loop_ms * 1e-3;
        if (want_edits) {
            r->spatial_flag_bytes = Nf / 8;
            r->frequency_flag_bytes = Ncf / 8;
            r->spatial_flags = static_cast<uint8_t*>(pinned().get(Nf / 8 + 1));
            r->frequency_flags = static_cast<uint8_t*>(pinned().get(Ncf / 8 + 1));
            r->spatial_codes = static_cast<int32_t*>(pinned().get(hpc[i] * 4 + 4));
            r->frequency_codes = static_cast<int32_t*>(pinned().get(hpc[Gc + i] * 8 + 4));
            r->escapes = static_cast<ffcz_cuda_escape*>(
                pinned().get(sizeof(ffcz_cuda_escape) * (esc[i].size() + 1)));
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(r->spatial_flags, reinterpret_cast<const uint8_t*>(keep_s) + i * (Nf / 8),
                                            Nf / 8, cudaMemcpyDeviceToHost, st));
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(r->frequency_flags, reinterpret_cast<const uint8_t*>(keep_f) + i * (Ncf / 8),
                                            Ncf / 8, cudaMemcpyDeviceToHost, st));
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(r->spatial_codes, codes_s + off_s[i], hpc[i] * 4,
                                            cudaMemcpyDeviceToHost, st));
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(r->frequency_codes, codes_f + 2 * off_f[i], hpc[Gc + i] * 8,
                                            cudaMemcpyDeviceToHost, st));
            if (!esc[i].empty())
                std::memcpy(r->escapes, esc[i].data(), sizeof(ffcz_cuda_escape) * esc[i].size());
        }
        if (corrected) {
            r->corrected = static_cast<double*>(pinned().get(Nf * sizeof(double)));
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(r->corrected, corrected + i * Nf, Nf * sizeof(double),
                                            cudaMemcpyDeviceToHost, st));
        }
    }
    c.sync();
    if ((opt.flags & FFCZ_WANT_ARCHIVE) && opt.zlib_level == FFCZ_OUTER_DEVICE) {
        for (long long i = 0; i < Gc; ++i) {
            ffcz_cuda_result* r = &out[g0 + i];
            DevArchiveInput ai{};
            ai.ndim = fd.ndim;
            for (int a = 0; a < fd.ndim; ++a) ai.dims[a] = fd.dims[a];
            ai.precision = fd.precision;
            ai.spatial_global = hE[i];
            ai.freq_global = hD[i];
            ai.m = m;
            ai.converged = hfc[i].converged;
            ai.spatial_flags = reinterpret_cast<const unsigned char*>(keep_s) + i * (Nf / 8);
            ai.spatial_flag_bytes = Nf / 8;
            ai.frequency_flags = reinterpret_cast<const unsigned char*>(keep_f) + i * (Ncf / 8);
            ai.frequency_flag_bytes = Ncf / 8;
            ai.n_spatial = r->n_spatial;
            ai.n_frequency = r->n_frequency;
            ai.spatial_codes = codes_s + off_s[i];
            ai.frequency_codes = codes_f + 2 * off_f[i];
            ai.escapes = r->escapes;
            ai.n_escapes = esc[i].size();
            device_archive(c, ai, r);
        }
    } else if (opt.flags & FFCZ_WANT_ARCHIVE) {
        for (long long i = 0; i < Gc; ++i) {
            ffcz_cuda_result* r = &out[g0 + i];
            std::vector<ffcz_host::EscapeRec> er(esc[i].size());
            for (size_t k = 0; k < er.size(); ++k)
                er[k] = {esc[i][k].frequency != 0, esc[i][k].index, esc[i][k].re, esc[i][k].im};
            ffcz_host::ArchiveInput ai{};
            ai.ndim = fd.ndim;
            for (int a = 0; a < fd.ndim; ++a) ai.dims[a] = fd.dims[a];
            ai.precision = fd.precision;
            ai.spatial_global = hE[i];
            ai.freq_global = hD[i];
            ai.m = m;
            ai.converged = hfc[i].converged;
            ai.spatial_flags = r->spatial_flags;
            ai.spatial_flag_bytes = r->spatial_flag_bytes;
            ai.frequency_flags = r->frequency_flags;
            ai.frequency_flag_bytes = r->frequency_flag_bytes;
            ai.n_spatial = r->n_spatial;
            ai.n_frequency = r->n_frequency;
            ai.spatial_codes = r->spatial_codes;
            ai.frequency_codes = r->frequency_codes;
            ai.escapes = er.data();
            ai.n_escapes = er.size();
            ai.zlib_level = opt.zlib_level;
            const auto t0 = std::chrono::steady_clock::now();
            std::vector<uint8_t> bytes = ffcz_host::write_archive(ai);
            r->t_archive_ms =
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            r->archive_len = bytes.size();
            r->archive = static_cast<uint8_t*>(pinned().get(bytes.size() + 1));
            std::memcpy(r->archive, bytes.data(), bytes.size());
        }
    }
    (void)bd;
}

// Batched frames with ONE projection loop over the whole stack (config 3): every pass covers
// all frames (axis-1 column passes with planes = frames, row passes over all rows), each frame
// has its own control block / bounds / decision, and the tiles of converged frames are skipped
// so each frame's state stops exactly where its own loop would (kernels.cuh, FrameBatch).  The
// FP64 gate of each frame then runs on the lanes (finish_typed on the frame's slices).  Frames
// are processed in groups sized to a device-memory budget.
template <class TI>
void correct_frames_fused(ffcz_cuda_ctx& c, const ffcz_field_desc& fd, uint64_t nframes,
                          const void* orig_in, const void* dec_in, const ffcz_bounds_desc* bd,
                          int m, uint64_t max_iters, const ffcz_cuda_options& opt, int nl,
                          ffcz_cuda_result* out) {
    if (m < 1 || m > 24) throw Error(kValidation, "shrink_bounds requires 1 <= m <= 24");
    if (max_iters < 1) throw Error(kValidation, "alternating_projection: max_iters must be >= 1");
    cudaStream_t st = c.st;
    const bool on_dev = opt.flags & FFCZ_INPUTS_ON_DEVICE;
    const Geometry gf = make_geometry(fd.ndim, fd.dims, kPitchAlign);
    const long long Nf = gf.N, Hf = gf.half_elems(), n1 = gf.d[1], n2 = gf.n2;
    const double fw = 1.0 - std::ldexp(1.0, -m);
    const double slack = 1.0 / (1.0 - std::ldexp(1.0, -m)) - 1.0 + 0x1p-20;
    const double per_frame = 16.0 * Nf + 33.0 * Hf + (on_dev ? 0.0 : 2.0 * sizeof(TI) * Nf);
    // two buffer sets: the per-frame gates of group k run on the lanes (background thread) while
    // the loop of group k+1 runs on the context stream
    // (the batched gate runs in the main thread: one buffer set, its own stack buffers)
    const bool batched_gate = frames_batched_gate_enabled();
    const double per_frame_all = per_frame + (batched_gate ? 36.0 * Nf + 32.0 * Hf + 12.0 * Nf : 0.0);
    static const double budget_env = [] {  // FFCZ_FRAMES_BUDGET_GB: group-size sweeps
        const char* e = std::getenv("FFCZ_FRAMES_BUDGET_GB");
        return e ? std::atof(e) * 1e9 : 0.0;
    }();
    const double budget = budget_env > 0 ? budget_env : (batched_gate ? 60e9 : 24e9);
    uint64_t G = std::max<uint64_t>(1, std::min<uint64_t>(
        nframes, static_cast<uint64_t>(budget / per_frame_all)));
    if (!batched_gate && nframes >= 64 && G >= nframes) G = (nframes + 1) / 2;  // overlap
    const uint64_t dims3[3] = {G, static_cast<uint64_t>(n1), static_cast<uint64_t>(n2)};
    ensure_lanes(&c, nl);
    std::thread gate_thread;
    std::exception_ptr gate_err;
    cudaEvent_t loop_done[2];
    for (auto& e : loop_done) FFCZ_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    struct Joiner {
        std::thread& t;
        cudaEvent_t* evs;
        ~Joiner() {
            if (t.joinable()) t.join();
            for (int i = 0; i < 2; ++i) cudaEventDestroy(evs[i]);
        }
    } joiner{gate_thread, loop_done};
    auto join_gates = [&]() {
        if (gate_thread.joinable()) gate_thread.join();
        if (gate_err) std::rethrow_exception(gate_err);
    };
    int parity = 0;
    for (uint64_t g0 = 0; g0 < nframes; g0 += G, parity = batched_gate ? 0 : parity ^ 1) {
        auto nm = [&](const char* base) { return std::string(base) + (parity ? "1" : "0"); };
        const long long Gc = static_cast<long long>(std::min<uint64_t>(G, nframes - g0));
        const uint64_t dimsc[3] = {static_cast<uint64_t>(Gc), dims3[1], dims3[2]};
        const Geometry gb = make_geometry(3, dimsc, kPitchAlign);
        FFCZ_CUDA_CHECK(cudaEventRecord(c.ev[0], st));
        const TI* orig = static_cast<const TI*>(orig_in) + g0 * Nf;
        const TI* dec = static_cast<const TI*>(dec_in) + g0 * Nf;
        if (!on_dev) {
            TI* o = c.b<TI>(nm("fr_orig"), Gc * Nf);
            TI* d = c.b<TI>(nm("fr_dec"), Gc * Nf);
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(o, orig, Gc * Nf * sizeof(TI), cudaMemcpyHostToDevice, st));
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(d, dec, Gc * Nf * sizeof(TI), cudaMemcpyHostToDevice, st));
            orig = o;
            dec = d;
        }
        std::vector<double> hE(Gc), hD(Gc);
        for (long long i = 0; i < Gc; ++i) {
            hE[i] = bd[g0 + i].spatial_global;
            hD[i] = bd[g0 + i].freq_global;
            if (!(hE[i] > 0.0) || !std::isfinite(hE[i]))
                throw Error(kValidation, "spatial bound E must be strictly positive and finite");
            if (!(hD[i] > 0.0) || !std::isfinite(hD[i]))
                throw Error(kValidation, "frequency bound Delta must be strictly positive and finite");
        }
        double* dE = c.b<double>(nm("fr_E"), Gc);
        double* dD = c.b<double>(nm("fr_D"), Gc);
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(dE, hE.data(), 8 * Gc, cudaMemcpyHostToDevice, st));
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(dD, hD.data(), 8 * Gc, cudaMemcpyHostToDevice, st));
        FFCZ_CUDA_CHECK(cudaEventRecord(c.ev[1], st));
        // compute_error + preconditions of every frame (pipeline.cpp:31-42)
        FrameCtl* fc = c.b<FrameCtl>(nm("fr_ctl"), Gc);
        k_frames_init<<<grid_for(Gc), 256, 0, st>>>(fc, Gc, max_iters);
        k_ctl_init<<<1, 1, 0, st>>>(c.ctl, max_iters);
        double* eps = c.b<double>(nm("fr_eps"), Gc * Nf);
        k_eps0_frames<TI><<<grid_for(Gc * Nf), 256, 0, st>>>(orig, dec, eps, Gc * Nf, Nf, dE, fw,
                                                             slack, c.ctl);
        FFCZ_LAUNCH_CHECK();
        const Ctl h0 = c.read_ctl();  // also orders the pageable hE / hD copies
        if (h0.bad1 != ~0ull)
            throw Error(kValidation, "correct: decompressed data violates the declared spatial "
                                     "bound at index " + std::to_string(h0.bad1 % Nf) +
                                     " (frame " + std::to_string(g0 + h0.bad1 / Nf) + ")");
        if (h0.bad2 != ~0ull)
            throw Error(kValidation, "alternating_projection: epsilon0 violates the spatial bound "
                                     "at index " + std::to_string(h0.bad2 % Nf) + " (frame " +
                                     std::to_string(g0 + h0.bad2 / Nf) + ")");
        double* S = c.b<double>(nm("fr_S"), Gc * Nf);
        double2* F = c.b<double2>(nm("fr_F"), Gc * Hf);
        double2* spec = c.b<double2>(nm("fr_spec"), Gc * Hf);
        unsigned char* moved = c.b<unsigned char>(nm("fr_moved"), Gc * Hf);
        FFCZ_CUDA_CHECK(cudaMemsetAsync(moved, 0, Gc * Hf, st));
        const FrameBatch fbt{fc, dE, dD, fw, n1};
        FftPlan<double> plan{gb, &c.tw64};
        const int* gate = &c.ctl->done;
        const double invN = 1.0 / static_cast<double>(Nf);
        FFCZ_CUDA_CHECK(cudaEventRecord(c.ev[2], st));
        launch_row_r2c_hook<double>(n2, eps, n2, spec, gb.P, gb.rows, c.tw64, nullptr,
                                    HookSkipB<true>{fbt}, st);
        c.launches += 3;
        auto body = [&]() {
            plan.col(1, -1, spec, spec, gate, HookFReduceB{fbt}, st);                  // K3a
            k_decide_frames<<<grid_for(Gc), 256, 0, st>>>(fc, Gc, c.ctl);              // K4
            plan.col(1, +1, spec, spec, gate, HookFClipB<double>{fbt, F, moved}, st);  // K3b
            launch_row_c2r_hook<double>(n2, spec, gb.P, eps, n2, gb.rows, invN, c.tw64, gate,
                                        HookSClipB<double>{fbt, S}, st);               // K1a
            launch_row_r2c_hook<double>(n2, eps, n2, spec, gb.P, gb.rows, c.tw64, gate,
                                        HookSkipB<true>{fbt}, st);                     // K1b
            FFCZ_LAUNCH_CHECK();
            c.launches += 5;
        };
        static const int kChunk[] = {1, 1, 2, 4, 8};
        int ci = 0, issued = 0;
        std::vector<std::pair<cudaEvent_t, int>> inflight;
        auto issue_chunk = [&]() {
            const int k = kChunk[std::min(ci++, 4)];
            for (int i = 0; i < k; ++i) body();
            const int slot = issued % 2;
            k_export_ctl<<<1, 32, 0, st>>>(c.ctl, &c.hctl_dev[1 + slot]);
            FFCZ_LAUNCH_CHECK();
            cudaEvent_t ev = c.ev[4 + slot];
            FFCZ_CUDA_CHECK(cudaEventRecord(ev, st));
            inflight.push_back({ev, slot});
            ++issued;
        };
        issue_chunk();
        for (;;) {
            issue_chunk();
            auto p = inflight.front();
            inflight.erase(inflight.begin());
            FFCZ_CUDA_CHECK(cudaEventSynchronize(p.first));
            if (c.hctl[1 + p.second].done) break;
        }
        FFCZ_CUDA_CHECK(cudaEventRecord(c.ev[3], st));
        std::vector<FrameCtl> hfc(Gc);
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(hfc.data(), fc, sizeof(FrameCtl) * Gc, cudaMemcpyDeviceToHost, st));
        c.sync();
        for (long long i = 0; i < Gc; ++i)
            if (hfc[i].passes == 0) {  // converged at the first check: no clip wrote S / F
                FFCZ_CUDA_CHECK(cudaMemsetAsync(S + i * Nf, 0, 8 * Nf, st));
                FFCZ_CUDA_CHECK(cudaMemsetAsync(F + i * Hf, 0, 16 * Hf, st));
            }
        const double t_in = event_ms(c.ev[0], c.ev[1]);
        const double t_loop = event_ms(c.ev[2], c.ev[3]);
        FFCZ_CUDA_CHECK(cudaEventRecord(loop_done[parity], st));
        // the previous group's gates must be done before its buffers are reused (next trip)
        join_gates();
        if (batched_gate) {  // the whole group's gate in stack passes
            gate_frames<TI>(c, gf, fd, Gc, g0, orig, dec, bd, m, hfc, hE, hD, dE, dD, eps, S, F,
                            spec, moved, opt, t_in, t_loop, out,
                            [&](const char* b) { return nm(b); });
            continue;
        }
        // per-frame FP64 gate on the lanes, in the background
        auto gate_group = [&c, &gate_err, nl, Gc, g0, Nf, Hf, gf, fd, bd, m, opt, out, hfc,
                           hE, hD, orig, dec, eps, S, F, spec, moved, t_loop, t_in,
                           start = loop_done[parity]]() {
          try {
            FFCZ_CUDA_CHECK(cudaSetDevice(c.device));
            run_on_lanes(&c, nl, static_cast<uint64_t>(Gc), [&](ffcz_cuda_ctx& l, uint64_t i) {
            LoopResult lr;
            lr.passes = hfc[i].passes;
            lr.converged = hfc[i].converged;
            lr.residual_f = hfc[i].residual_f;
            lr.fused = true;
            lr.moved = moved + i * Hf;
            Bounds bo;
            bo.sb.g = hE[i];
            bo.fb.g = hD[i];
            ffcz_cuda_result* r = &out[g0 + i];
            const unsigned long long l0 = l.launches;
            finish_typed<TI>(l, gf, fd, orig + i * Nf, dec + i * Nf, bd[g0 + i], bo, m, lr,
                             eps + i * Nf, S + i * Nf, F + i * Hf, spec + i * Hf, opt, r);
            r->kernel_launches = l.launches - l0;
            r->report.wall_time_s = t_loop / Gc * 1e-3;   // the loop is shared by the group
            r->t_loop_ms = t_loop / Gc;
            r->t_h2d_ms = t_in / Gc;
            r->t_feasible_ms = r->t_loop_ms + r->t_gate_ms;
            }, start, false);
          } catch (...) {
            gate_err = std::current_exception();
          }
        };
        gate_thread = std::thread(gate_group);
    }
    join_gates();
}

} // namespace

namespace {
// the field as FP64 on the device (host buffers copied in; f32 widened)
const double* metric_field(ffcz_cuda_ctx& c, const std::string& name, const Geometry& g,
                           int dtype, const void* p, int on_device) {
    if (!p) throw Error(kValidation, "null field buffer");
    if (dtype == FFCZ_F64 && on_device) return static_cast<const double*>(p);
    double* d = c.b<double>(name, g.N);
    if (dtype == FFCZ_F64) {
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(d, p, g.N * 8, cudaMemcpyHostToDevice, c.st));
        return d;
    }
    const float* f = static_cast<const float*>(p);
    if (!on_device) {
        float* t = c.b<float>(name + "_f32", g.N);
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(t, p, g.N * 4, cudaMemcpyHostToDevice, c.st));
        f = t;
    }
    k_cast_to_double<<<grid_for(g.N), 256, 0, c.st>>>(f, d, g.N);
    FFCZ_LAUNCH_CHECK();
    return d;
}
template <class S>
S read_stats(ffcz_cuda_ctx& c, const S* d) {
    S h;
    FFCZ_CUDA_CHECK(cudaMemcpyAsync(&h, d, sizeof(S), cudaMemcpyDeviceToHost, c.st));
    c.sync();
    return h;
}
FieldStats* fresh_field_stats(ffcz_cuda_ctx& c) {
    FieldStats* d = c.b<FieldStats>("m_fstats", 1);
    FieldStats z{};
    z.lo = ~0ull;
    FFCZ_CUDA_CHECK(cudaMemcpyAsync(d, &z, sizeof z, cudaMemcpyHostToDevice, c.st));
    return d;
}
SpecStats* fresh_spec_stats(ffcz_cuda_ctx& c) {
    SpecStats* d = c.b<SpecStats>("m_sstats", 1);
    FFCZ_CUDA_CHECK(cudaMemsetAsync(d, 0, sizeof(SpecStats), c.st));
    return d;
}
double bits_to_d(unsigned long long u) {
    double d;
    std::memcpy(&d, &u, 8);
    return d;
}
} // namespace

extern "C" {

int ffcz_cuda_abi_version(void) { return FFCZ_CUDA_ABI_VERSION; }
const char* ffcz_cuda_last_error(void) { return g_last_error.c_str(); }

void ffcz_cuda_default_options(ffcz_cuda_options* opt) {
    opt->flags = FFCZ_WANT_EDITS;
    opt->policy = FFCZ_POLICY_FP64;
    opt->tau_switch = 1e-4;
    opt->zlib_level = FFCZ_OUTER_DEVICE;
}

int ffcz_cuda_create(ffcz_cuda_ctx** out, int device, void* stream) {
    try {
        if (!out) return fail(kValidation, "null output pointer");
        auto* c = new ffcz_cuda_ctx;
        c->device = device;
        FFCZ_CUDA_CHECK(cudaSetDevice(device));
        if (stream) {
            c->st = static_cast<cudaStream_t>(stream);
        } else {
            FFCZ_CUDA_CHECK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
            c->own_stream = true;
        }
        FFCZ_CUDA_CHECK(cudaMalloc(&c->ctl, sizeof(Ctl)));
        FFCZ_CUDA_CHECK(cudaHostAlloc(&c->hctl, 4 * sizeof(Ctl), cudaHostAllocMapped));
        FFCZ_CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->hctl_dev), c->hctl, 0));
        for (auto& e : c->ev) FFCZ_CUDA_CHECK(cudaEventCreate(&e));
        FFCZ_CUDA_CHECK(cudaStreamCreateWithFlags(&c->st_copy, cudaStreamNonBlocking));
        FFCZ_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_codes, cudaEventDisableTiming));
        c->tw64.init();
        c->tw32.init();
        *out = c;
        return kOk;
    } catch (const Error& e) {
        return fail(e.status, e.what());
    } catch (const std::exception& e) {
        return fail(kCuda, e.what());
    }
}

void ffcz_cuda_destroy(ffcz_cuda_ctx* c) {
    if (!c) return;
    for (ffcz_cuda_ctx* l : c->lanes) ffcz_cuda_destroy(l);
    c->lanes.clear();
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->st);
    if (c->st_copy) cudaStreamSynchronize(c->st_copy);
    for (auto& kv : c->bufs) cudaFree(kv.second.first);
    if (c->ctl) cudaFree(c->ctl);
    if (c->hctl) cudaFreeHost(c->hctl);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->ev_codes) cudaEventDestroy(c->ev_codes);
    if (c->st_copy) cudaStreamDestroy(c->st_copy);
    if (c->own_stream) cudaStreamDestroy(c->st);
    delete c;
}

void ffcz_cuda_result_free(ffcz_cuda_result* r) {
    if (!r) return;
    pinned().put(r->spatial_flags);
    pinned().put(r->frequency_flags);
    pinned().put(r->spatial_codes);
    pinned().put(r->frequency_codes);
    pinned().put(r->escapes);
    pinned().put(r->corrected);
    pinned().put(r->archive);
    std::memset(r, 0, sizeof(*r));
}

int ffcz_cuda_correct(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, const void* original,
                      const void* decompressed, const ffcz_bounds_desc* bounds_original, int m,
                      uint64_t max_iters, const ffcz_cuda_options* opt_in, ffcz_cuda_result* out) {
    return guarded(ctx, [&] {
        if (!field || !original || !decompressed || !bounds_original || !out)
            throw Error(kValidation, "null argument");
        std::memset(out, 0, sizeof(*out));
        ffcz_cuda_options opt;
        ffcz_cuda_default_options(&opt);
        if (opt_in) opt = *opt_in;
        if (opt.policy != FFCZ_POLICY_FP64 && opt.policy != FFCZ_POLICY_MIXED)
            throw Error(kValidation, "unknown precision policy");
        if (opt.policy == FFCZ_POLICY_MIXED && !(opt.tau_switch > 0.0 && opt.tau_switch < 1.0))
            throw Error(kValidation, "mixed policy: tau_switch must be in (0, 1)");
        const Geometry g = make_geometry(field->ndim, field->dims, kPitchAlign);
        const unsigned long long l0 = ctx->launches;
        ctx->call_flags = opt.flags;
        if (field->dtype == FFCZ_F32)
            correct_typed<float>(*ctx, g, *field, original, decompressed, *bounds_original, m,
                                 max_iters, opt, out);
        else
            correct_typed<double>(*ctx, g, *field, original, decompressed, *bounds_original, m,
                                  max_iters, opt, out);
        out->kernel_launches = ctx->launches - l0;
    });
}


// Batched frames (BASELINE config 3): every frame is an independent ffcz::correct() call
// (pipeline.cpp:26-178), with its own bounds, iterations and edit set.  Power-of-two 2-D frames
// (>= 64 x 64) with global bounds run ONE projection loop over the whole stack
// (correct_frames_fused) and their per-frame gates on the lanes; anything else runs whole
// per-frame correct() calls on the lanes (host threads, one sub-context and stream each).  Results
// equal one ffcz_cuda_correct() per frame (FFT round-off of the batched passes aside).  The
// batch is ordered on the context stream.
int ffcz_cuda_correct_batch(ffcz_cuda_ctx* ctx, const ffcz_field_desc* frame, uint64_t nframes,
                            const void* original, const void* decompressed,
                            const ffcz_bounds_desc* bounds, int m, uint64_t max_iters,
                            const ffcz_cuda_options* opt_in, int lanes, ffcz_cuda_result* out) {
    return guarded(ctx, [&] {
        if (!frame || !original || !decompressed || !bounds || !out)
            throw Error(kValidation, "null argument");
        ffcz_cuda_options opt;
        ffcz_cuda_default_options(&opt);
        if (opt_in) opt = *opt_in;
        if (opt.policy != FFCZ_POLICY_FP64 && opt.policy != FFCZ_POLICY_MIXED)
            throw Error(kValidation, "unknown precision policy");
        for (uint64_t i = 0; i < nframes; ++i) std::memset(&out[i], 0, sizeof(out[i]));
        if (nframes == 0) return;
        ctx->call_flags = opt.flags;
        const Geometry g = make_geometry(frame->ndim, frame->dims, kPitchAlign);
        const size_t esz = frame->dtype == FFCZ_F32 ? 4 : 8;
        if (lanes <= 0) lanes = 8;
        const int nl = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(lanes), nframes));
        bool fused = frames_fused_enabled() && frame->ndim == 2 &&
                     opt.policy == FFCZ_POLICY_FP64 &&
                     !(opt.flags & FFCZ_FORCE_UNFUSED) && g.d[1] >= 64 && g.n2 >= 64 &&
                     radix_col_ok(g.d[1]) && radix_row_ok(g.n2);
        for (uint64_t i = 0; fused && i < nframes; ++i)
            fused = !bounds[i].spatial_per_point && !bounds[i].freq_per_component;
        try {
            if (fused) {
                // kernel launches of the shared loop and gate (context + lanes), spread over the
                // frames' results so that their sum is the batch's total
                auto all_launches = [&] {
                    unsigned long long t = ctx->launches;
                    for (auto* l : ctx->lanes) t += l->launches;
                    return t;
                };
                const unsigned long long L0 = all_launches();
                if (frame->dtype == FFCZ_F32)
                    correct_frames_fused<float>(*ctx, *frame, nframes, original, decompressed,
                                                bounds, m, max_iters, opt, nl, out);
                else
                    correct_frames_fused<double>(*ctx, *frame, nframes, original, decompressed,
                                                 bounds, m, max_iters, opt, nl, out);
                unsigned long long tot = all_launches() - L0, given = 0;
                for (uint64_t i = 0; i < nframes; ++i) given += out[i].kernel_launches;
                if (tot > given) {
                    const unsigned long long extra = tot - given;
                    for (uint64_t i = 0; i < nframes; ++i)
                        out[i].kernel_launches += extra / nframes + (i < extra % nframes ? 1 : 0);
                }
                return;
            }
            run_on_lanes(ctx, nl, nframes, [&](ffcz_cuda_ctx& l, uint64_t i) {
                const char* o = static_cast<const char*>(original) + i * g.N * esz;
                const char* d = static_cast<const char*>(decompressed) + i * g.N * esz;
                const unsigned long long l0 = l.launches;
                if (frame->dtype == FFCZ_F32)
                    correct_typed<float>(l, g, *frame, o, d, bounds[i], m, max_iters, opt, &out[i]);
                else
                    correct_typed<double>(l, g, *frame, o, d, bounds[i], m, max_iters, opt, &out[i]);
                out[i].kernel_launches = l.launches - l0;
            });
        } catch (...) {
            for (uint64_t i = 0; i < nframes; ++i) ffcz_cuda_result_free(&out[i]);
            throw;
        }
    });
}

// apply_edits(decompressed, read_archive(bytes)) (archive.cpp:137-273) on the device: the host
// parses the container (header, CRC-32C, zlib outer stages), the device decodes the Huffman
// index streams, dequantises + scatters the edits and escapes, inverts the half spectrum and adds.
int ffcz_cuda_apply_archive(ffcz_cuda_ctx* ctx, const uint8_t* archive, uint64_t len,
                            const ffcz_field_desc* field, const void* decompressed, uint32_t flags,
                            double* corrected) {
    return guarded(ctx, [&] {
        if (!archive || !field || !decompressed || !corrected) throw Error(kValidation, "null argument");
        DebugClock dbg;
        ffcz_host::ParsedArchive a;
        try {
            a = ffcz_host::parse_archive(archive, len);
        } catch (const std::runtime_error& e) {
            throw Error(kFormat, e.what());
        }
        dbg.mark(*ctx, "apply: container parsed");
        bool same = field->ndim == a.ndim;
        for (int i = 0; same && i < a.ndim; ++i) same = field->dims[i] == a.dims[i];
        if (!same) throw Error(kValidation, "apply_edits: field dims do not match archive dims");
        ffcz_cuda_ctx& c = *ctx;
        cudaStream_t st = c.st;
        const Geometry g = make_geometry(a.ndim, a.dims, kPitchAlign);
        const HalfGeom hg = g.hg();
        const long long N = g.N, Nc = g.Nc();
        const bool on_dev = flags & FFCZ_INPUTS_ON_DEVICE;
        const size_t esz = field->dtype == FFCZ_F32 ? 4 : 8;
        const void* dec = decompressed;
        if (!on_dev) {
            void* d = c.buf("ap_dec", N * esz);
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(d, decompressed, N * esz, cudaMemcpyHostToDevice, st));
            dec = d;
        }
        ffcz_bounds_desc bd{};
        bd.spatial_per_point = a.spatial_per_point;
        bd.spatial_global = a.spatial_global;
        bd.spatial_values = reinterpret_cast<const double*>(a.spatial_values);
        bd.freq_per_component = a.freq_per_component;
        bd.freq_global = a.freq_global;
        bd.freq_re = reinterpret_cast<const double*>(a.freq_re);
        bd.freq_im = reinterpret_cast<const double*>(a.freq_im);
        const Bounds b = upload_bounds(c, g, bd, false);
        dbg.mark(c, "apply: bounds uploaded");
        const long long ws = (N + 31) / 32, wf = (Nc + 31) / 32;
        unsigned* ks = c.b<unsigned>("ap_keep_s", ws);
        unsigned* kf = c.b<unsigned>("ap_keep_f", wf);
        // BitVector semantics (bitvector.hpp:24-29): only bits < nbits exist, so padding bits of
        // the last flag byte are cleared; the flag count must equal the code count before any
        // scatter is launched (archive.cpp:205-208), so a malformed archive never indexes past
        // N / Nc or past the decoded codes
        auto clean_flags = [&](std::vector<uint8_t>& f, long long nbits, unsigned long long want) {
            if (static_cast<long long>(f.size()) != (nbits + 7) / 8)
                throw Error(kFormat, "read_archive: flag stream size mismatch");
            if ((nbits & 7) && !f.empty()) f.back() &= static_cast<uint8_t>((1u << (nbits & 7)) - 1);
            unsigned long long pc = 0;
            for (uint8_t v : f) pc += static_cast<unsigned>(__builtin_popcount(v));
            if (pc != want) throw Error(kFormat, "read_archive: edit count mismatch");
        };
        clean_flags(a.spatial_flags, N, a.n_spatial);
        clean_flags(a.frequency_flags, Nc, a.n_frequency);
        FFCZ_CUDA_CHECK(cudaMemsetAsync(ks, 0, 4 * ws, st));
        FFCZ_CUDA_CHECK(cudaMemsetAsync(kf, 0, 4 * wf, st));
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(ks, a.spatial_flags.data(), a.spatial_flags.size(),
                                        cudaMemcpyHostToDevice, st));
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(kf, a.frequency_flags.data(), a.frequency_flags.size(),
                                        cudaMemcpyHostToDevice, st));
        DevScratch ds{st, [&](const char* nm, size_t bytes) { return c.buf(nm, bytes); }};
        auto decode = [&](const std::vector<uint8_t>& payload, unsigned long long want,
                          const char* name) {
            std::vector<std::uint64_t> off, first;
            unsigned long long total = 0;
            try {
                total = ffcz_host::huffman_blocks(payload, off, first);
            } catch (const std::runtime_error& e) {
                throw Error(kFormat, e.what());
            }
            if (total != want) throw Error(kFormat, "read_archive: edit count mismatch");
            int* codes = c.b<int>(name, std::max<unsigned long long>(total, 1));
            huffman_decode_device(ds, payload.data(), payload.size(),
                                  reinterpret_cast<const unsigned long long*>(off.data()),
                                  reinterpret_cast<const unsigned long long*>(first.data()),
                                  static_cast<long long>(off.size()), codes);
            return codes;
        };
        dbg.mark(c, "apply: flags uploaded");
        int* cs = decode(a.spatial_payload, a.n_spatial, "ap_codes_s");
        int* cf = decode(a.frequency_payload, 2 * a.n_frequency, "ap_codes_f");
        dbg.mark(c, "apply: huffman decoded");
        double* spat = c.b<double>("ap_spat", N);
        double2* freq = c.b<double2>("ap_freq", g.half_elems());
        FFCZ_CUDA_CHECK(cudaMemsetAsync(spat, 0, 8 * N, st));
        FFCZ_CUDA_CHECK(cudaMemsetAsync(freq, 0, 16 * g.half_elems(), st));
        auto scatter = [&](const unsigned* words, long long nwords, unsigned long long want,
                           const char* name, auto launch) {
            const long long nblk = std::max<long long>(1, (nwords + 1023) / 1024);
            unsigned long long* cnt = c.b<unsigned long long>(name, nblk + 1);
            k_popc_blocks<<<static_cast<unsigned>(nblk), 1024, 0, st>>>(words, nwords, cnt);
            k_scan_blocks<<<1, 1024, 0, st>>>(cnt, nblk, &c.ctl->count_a);
            launch(static_cast<unsigned>(nblk), cnt);
            FFCZ_LAUNCH_CHECK();
            (void)want;  // checked on the host flags above
        };
        scatter(ks, ws, a.n_spatial, "ap_cnt_s", [&](unsigned nb, unsigned long long* o) {
            k_dequant_spatial_bits<<<nb, 1024, 0, st>>>(ks, ws, o, cs, b.sb, a.m, spat);
        });
        scatter(kf, wf, a.n_frequency, "ap_cnt_f", [&](unsigned nb, unsigned long long* o) {
            k_dequant_freq_bits<<<nb, 1024, 0, st>>>(kf, wf, o, cf, hg, b.fb, a.m, freq);
        });
        if (!a.escapes.empty()) {
            std::vector<EscapeRec> er(a.escapes.size());
            for (size_t i = 0; i < er.size(); ++i)
                er[i] = {a.escapes[i].frequency ? 1 : 0, 0, a.escapes[i].index, a.escapes[i].re,
                         a.escapes[i].im};
            EscapeRec* de = c.b<EscapeRec>("ap_esc", er.size());
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(de, er.data(), er.size() * sizeof(EscapeRec),
                                            cudaMemcpyHostToDevice, st));
            k_scatter_escapes<<<grid_for(er.size()), 256, 0, st>>>(de, er.size(), spat, freq, hg);
            FFCZ_LAUNCH_CHECK();
            c.sync();  // `er` is pageable and goes out of scope
        }
        dbg.mark(c, "apply: edits scattered");
        FftPlan<double> plan{g, &c.tw64};
        double* fpart = c.b<double>("ap_fpart", N);
        double2* work = c.b<double2>("ap_work", g.half_elems());
        c2r_p(c, plan, freq, work, fpart, 1.0 / static_cast<double>(N));
        double* out = on_dev ? corrected : c.b<double>("ap_out", N);
        if (field->dtype == FFCZ_F32)
            k_apply_sum<float><<<grid_for(N), 256, 0, st>>>(static_cast<const float*>(dec), spat,
                                                             fpart, out, N);
        else
            k_apply_sum<double><<<grid_for(N), 256, 0, st>>>(static_cast<const double*>(dec), spat,
                                                              fpart, out, N);
        FFCZ_LAUNCH_CHECK();
        if (!on_dev)
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(corrected, out, 8 * N, cudaMemcpyDeviceToHost, st));
        c.sync();
    });
}

uint64_t ffcz_cuda_slab_pitch(uint64_t n2) { return round_up(n2 / 2 + 1, kPitchAlign); }

// CUDA IPC for the slab path's fused all-to-all: each rank exports its receive buffers, every
// other rank maps them (NVLink peer memory on a multi-GPU node; the same device across processes
// in the tests) and the scattering passes store into them directly.
int ffcz_cuda_ipc_handle(ffcz_cuda_ctx* ctx, const void* ptr, unsigned char handle[64],
                         uint64_t* offset) {
    return guarded(ctx, [&] {
        if (!ptr || !handle || !offset) throw Error(kValidation, "ipc_handle: null argument");
        // the handle names the whole allocation (a torch cache block may start inside it)
        using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
        static GetRange get_range = [] {
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) !=
                    cudaSuccess || q != cudaDriverEntryPointSuccess)
                fn = nullptr;
            return reinterpret_cast<GetRange>(fn);
        }();
        if (!get_range) throw Error(kCuda, "ipc_handle: cuMemGetAddressRange unavailable");
        CUdeviceptr base = 0;
        size_t size = 0;
        if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
            throw Error(kValidation, "ipc_handle: not a device allocation");
        cudaIpcMemHandle_t h;
        FFCZ_CUDA_CHECK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
        static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
        std::memcpy(handle, &h, 64);
        *offset = reinterpret_cast<uint64_t>(ptr) - static_cast<uint64_t>(base);
    });
}

int ffcz_cuda_ipc_open(ffcz_cuda_ctx* ctx, const unsigned char handle[64], void** base) {
    return guarded(ctx, [&] {
        if (!handle || !base) throw Error(kValidation, "ipc_open: null argument");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, 64);
        FFCZ_CUDA_CHECK(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

int ffcz_cuda_ipc_close(ffcz_cuda_ctx* ctx, void* base) {
    return guarded(ctx, [&] { FFCZ_CUDA_CHECK(cudaIpcCloseMemHandle(base)); });
}

// One per-rank device step of the slab-decomposed correction (paper_2601_01596_b200/slab.py).
namespace {
// device-resident slab loop (slab.py): this rank's (peak, excess) of the check pass, unless the
// loop is already done
__global__ void k_slab_export(const Ctl* __restrict__ ctl, double* red, const int* gate) {
    if (gated(gate)) return;
    red[0] = bitsd(ctl->peak_bits);
    red[1] = bitsd(ctl->exc_bits);
}
// the decision of alternating_projection (projection.cpp:106-116) on the all-reduced
// (peak, excess): state = (passes, residual_f), gate = (done, converged)
__global__ void k_slab_decide(const double* __restrict__ red, double* state, int* gate,
                              unsigned long long max_iters) {
    if (gate[0]) return;
    const double peak = red[0], ex = red[1];
    if (!(ex > 1e-11 * peak)) {                                   // projection.cpp:40,106-111
        gate[1] = 1;
        state[1] = 0.0;
        gate[0] = 1;
    } else if (state[0] >= static_cast<double>(max_iters)) {     // :112-116
        gate[1] = 0;
        state[1] = ex;
        gate[0] = 1;
    } else {
        state[0] += 1.0;
    }
}
}  // namespace

int ffcz_cuda_slab(ffcz_cuda_ctx* ctx, const ffcz_cuda_slab_op* op, double out[4]) {
    return guarded(ctx, [&] {
        if (!op) throw Error(kValidation, "null op");
        ffcz_cuda_ctx& c = *ctx;
        cudaStream_t st = c.st;
        const uint64_t dims[3] = {op->d0, op->d1, op->n2};
        const Geometry g = make_geometry(3, dims, kPitchAlign);
        FftPlan<double> plan{g, &c.tw64};
        const HalfGeom hg = g.hg();
        const long long N = g.N, Nc = g.Nc();
        const double invN = 1.0 / static_cast<double>(op->n_total);
        // per-point E (natural slab layout) / per-component Delta lanes (the pitched half layout
        // of the buffer the op works on) when given, else the global values
        const SpatialB sb{op->e_arr, op->e};
        const FreqB fb{op->d_re, op->d_im ? op->d_im : op->d_re, op->delta};
        auto P = [&](int i) { return op->p[i]; };
        auto d2 = [&](int i) { return static_cast<double2*>(op->p[i]); };
        auto dd = [&](int i) { return static_cast<double*>(op->p[i]); };
        auto ww = [&](int i) { return static_cast<unsigned*>(op->p[i]); };
        double o4[4] = {0, 0, 0, 0};
        const unsigned long long ticks0 = launch_ticks();  // launches of this op (c.launches)
        auto reset_ctl = [&] { k_ctl_init<<<1, 1, 0, st>>>(c.ctl, 1); FFCZ_LAUNCH_CHECK(); };
        // loop ops of the device-resident slab loop: p9 = the loop's done flag (NULL: ungated)
        const bool loop_op = op->op == FFCZ_SLAB_FWD_LOCAL || op->op == FFCZ_SLAB_COL0_CHECK ||
                             op->op == FFCZ_SLAB_COL0_CLIP_INV || op->op == FFCZ_SLAB_INV_SCLIP ||
                             op->op == FFCZ_SLAB_FWD_LOCAL_PEER ||
                             op->op == FFCZ_SLAB_COL0_CLIP_INV_PEER;
        const int* gate = loop_op ? static_cast<const int*>(P(9)) : nullptr;
        // FFCZ_SLAB_SWAP_AXES (a one-rank slab: the B layout is the natural one): the "axis-0"
        // ops transform the middle axis and the local ops the outer one, the fused engine's
        // order (check / clip hooks on the middle axis, where they run ~2x faster at 1024^3)
        const int ax0 = (op->pad & FFCZ_SLAB_SWAP_AXES) ? 1 : 0, axl = 1 - ax0;
        const bool f32 = op->in_dtype == FFCZ_F32;
        switch (op->op) {
        case FFCZ_SLAB_EPS0: {
            reset_ctl();
            if (f32)
                k_eps0<float><<<grid_for(N), 256, 0, st>>>(static_cast<const float*>(P(0)),
                    static_cast<const float*>(P(1)), dd(2), N, sb, op->fscale, op->slack, 1, c.ctl);
            else
                k_eps0<double><<<grid_for(N), 256, 0, st>>>(static_cast<const double*>(P(0)),
                    static_cast<const double*>(P(1)), dd(2), N, sb, op->fscale, op->slack, 1, c.ctl);
            FFCZ_LAUNCH_CHECK();
            const Ctl h = c.read_ctl();
            o4[0] = h.bad1 == ~0ull ? -1.0 : static_cast<double>(h.bad1);
            o4[1] = h.bad2 == ~0ull ? -1.0 : static_cast<double>(h.bad2);
            break;
        }
        case FFCZ_SLAB_FWD_LOCAL:
            launch_row_r2c<double>(g.n2, dd(0), g.n2, d2(1), g.P, g.rows, c.tw64, gate, st);
            plan.col(axl, -1, d2(1), d2(1), gate, HookNone{}, st);
            break;
        case FFCZ_SLAB_COL0_CHECK: {
            reset_ctl();
            plan.col(ax0, -1, d2(0), d2(0), gate, HookFReduce{fb, op->fscale, c.ctl}, st);
            if (P(1)) {  // device-resident loop: (peak, excess) stay on the device
                k_slab_export<<<1, 1, 0, st>>>(c.ctl, dd(1), gate);
                FFCZ_LAUNCH_CHECK();
                break;
            }
            const Ctl h = c.read_ctl();
            o4[0] = bitsd_host(h.peak_bits);
            o4[1] = bitsd_host(h.exc_bits);
            break;
        }
        case FFCZ_SLAB_DECIDE:
            k_slab_decide<<<1, 1, 0, st>>>(dd(0), dd(1), static_cast<int*>(P(9)), op->n_total);
            FFCZ_LAUNCH_CHECK();
            break;
        case FFCZ_SLAB_COL0_CLIP_INV: {
            HookFClip<double> hk{fb, op->fscale, d2(1), nullptr, static_cast<unsigned char*>(P(2))};
            hk.first = op->first != 0;
            plan.col(ax0, +1, d2(0), d2(0), gate, hk, st);
            break;
        }
        case FFCZ_SLAB_FWD_LOCAL_PEER:
        case FFCZ_SLAB_COL0_CLIP_INV_PEER: {
            // fused all-to-all (kernels.cuh PeerScatter): the pass stores into the receive
            // buffers of the ranks that own its outputs in the other layout
            const unsigned W = static_cast<unsigned>(op->world), r = static_cast<unsigned>(op->rank);
            if (op->world < 2 || op->rank < 0 || r >= W || !P(8) || (op->pad & FFCZ_SLAB_SWAP_AXES))
                throw Error(kValidation, "slab peer op: needs world >= 2, 0 <= rank < world, p8");
            if (g.half_elems() >= (1LL << 32))
                throw Error(kUnsupported, "slab peer op: slab above 2^32 half-spectrum elements");
            const bool fwd = op->op == FFCZ_SLAB_FWD_LOCAL_PEER;
            // forward: this buffer is A (c0, n1, P); backward: B (n0, c1, P)
            const unsigned d0 = static_cast<unsigned>(g.d[0]), d1 = static_cast<unsigned>(g.d[1]);
            if ((fwd ? d1 : d0) % W)
                throw Error(kValidation, "slab peer op: the exchanged axis must divide by world");
            auto lg2 = [](unsigned v) {
                if (!v || (v & (v - 1)))
                    throw Error(kUnsupported, "slab peer op: power-of-two slab extents only");
                int l = 0;
                while ((1u << l) < v) ++l;
                return l;
            };
            PeerScatter ps;
            ps.peers = static_cast<double2* const*>(P(8));
            ps.row = FastDiv::make(static_cast<unsigned>(g.P));
            ps.d1_sh = lg2(d1);
            ps.fwd = fwd ? 1 : 0;
            if (fwd) {   // (c0, n1) -> (n0, c1): c1 = n1 / W
                ps.part_sh = lg2(d1 / W);
                ps.width_sh = lg2(d1 / W);
                ps.base = r * d0;
                if (P(0))  // (p0 NULL: the rows of A were transformed by INV_SCLIP's fused pass)
                    launch_row_r2c<double>(g.n2, dd(0), g.n2, d2(1), g.P, g.rows, c.tw64, gate, st);
                plan.col(1, -1, d2(1), d2(1), gate, HookScatter{ps}, st);
            } else {     // (n0, c1) -> (c0, n1): c0 = n0 / W, n1 = W c1
                ps.part_sh = lg2(d0 / W);
                ps.width_sh = lg2(W * d1);
                ps.base = r * d1;
                HookFClipScatter<double> hk;
                hk.fb = fb;
                hk.fscale = op->fscale;
                hk.F = d2(1);
                hk.moved = static_cast<unsigned char*>(P(2));
                hk.first = op->first != 0;
                hk.ps = ps;
                plan.col(0, +1, d2(0), d2(0), gate, hk, st);
            }
            break;
        }
        case FFCZ_SLAB_COL0_PLAIN:
            plan.col(ax0, op->dir < 0 ? -1 : +1, d2(0), d2(1), nullptr, HookNone{}, st);
            break;
        case FFCZ_SLAB_COL0_REBUILD:
            plan.col(ax0, -1, d2(0), d2(0), nullptr,
                     HookFRebuild{d2(1), d2(3), static_cast<const unsigned char*>(P(2))}, st);
            break;
        case FFCZ_SLAB_COL0_MARK: {
            reset_ctl();
            FFCZ_CUDA_CHECK(cudaMemsetAsync(P(1), 0, ((g.half_elems() + 31) / 32) * 4, st));
            plan.col(ax0, -1, d2(0), d2(0), nullptr, HookMarkViol{fb, ww(1), c.ctl}, st);
            o4[0] = c.read_ctl().dirty;
            break;
        }
        case FFCZ_SLAB_COL0_VERIFY: {
            reset_ctl();
            plan.col(ax0, -1, d2(0), d2(0), nullptr, HookVerifyF{fb, c.ctl}, st);
            o4[0] = bitsd_host(c.read_ctl().vf_bits);
            break;
        }
        case FFCZ_SLAB_INV_SCLIP: {
            plan.col(axl, +1, d2(0), d2(0), gate, HookNone{}, st);
            HookSClip<double> hk{sb, op->fscale, dd(2), nullptr, nullptr};
            hk.first = op->first != 0;
            if (P(3)) {
                // + the forward row step into p3 (the single-volume loop's fused K1: C2R ->
                // s-clip -> R2C in one row pass, eps still written), and the forward local pass
                // on p3 when p4 is set (else the caller's peer pass follows)
                if (radix_row_ok(g.n2)) {
                    hk.eps = dd(1);
                    launch_row_fused<double>(g.n2, d2(0), g.P, g.rows, g.n2, invN, c.tw64, gate,
                                             hk, st, P(3) == P(0) ? nullptr : d2(3));
                } else {
                    launch_row_c2r_hook<double>(g.n2, d2(0), g.P, dd(1), g.n2, g.rows, invN,
                                                c.tw64, gate, hk, st);
                    launch_row_r2c<double>(g.n2, dd(1), g.n2, d2(3), g.P, g.rows, c.tw64, gate,
                                           st);
                }
                if (P(4)) plan.col(axl, -1, d2(3), d2(3), gate, HookNone{}, st);
                break;
            }
            launch_row_c2r_hook<double>(g.n2, d2(0), g.P, dd(1), g.n2, g.rows, invN, c.tw64,
                                        gate, hk, st);
            break;
        }
        case FFCZ_SLAB_INV_REPAIR_VERIFY:
        case FFCZ_SLAB_INV_VERIFY: {
            reset_ctl();
            plan.col(axl, +1, d2(0), d2(0), nullptr, HookNone{}, st);
            auto run = [&](auto tag) {
                using TI = decltype(tag);
                const TI* o = static_cast<const TI*>(P(2));
                const TI* d = static_cast<const TI*>(P(3));
                if (op->op == FFCZ_SLAB_INV_REPAIR_VERIFY) {
                    HookRepairVerifyS<TI> hk{o, d, dd(4), dd(5), sb, ww(6), dd(7), dd(8), c.ctl};
                    hk.dview = P(8) == nullptr;  // no eps_v buffer: decoder-view repair
                    launch_row_c2r_hook<double>(g.n2, d2(0), g.P, dd(1), g.n2, g.rows, invN, c.tw64,
                                                nullptr, hk, st);
                }
                else
                    launch_row_c2r_hook<double>(g.n2, d2(0), g.P, dd(1), g.n2, g.rows, invN, c.tw64,
                        nullptr, HookVerifyS<TI>{o, d, dd(4), dd(5), sb, c.ctl}, st);
            };
            if (f32) run(float{}); else run(double{});
            const Ctl h = c.read_ctl();
            o4[0] = h.dirty;
            o4[1] = bitsd_host(h.vs_bits);
            break;
        }
        case FFCZ_SLAB_RESIDUAL_S: {
            reset_ctl();
            k_residual_s<<<grid_for(N), 256, 0, st>>>(dd(0), N, sb, op->fscale, c.ctl);
            FFCZ_LAUNCH_CHECK();
            o4[0] = bitsd_host(c.read_ctl().res_s_bits);
            break;
        }
        case FFCZ_SLAB_EPS0_PLUS_S:
            if (f32)
                k_eps0_plus_s<float><<<grid_for(N), 256, 0, st>>>(static_cast<const float*>(P(0)),
                    static_cast<const float*>(P(1)), dd(2), dd(3), N);
            else
                k_eps0_plus_s<double><<<grid_for(N), 256, 0, st>>>(static_cast<const double*>(P(0)),
                    static_cast<const double*>(P(1)), dd(2), dd(3), N);
            FFCZ_LAUNCH_CHECK();
            break;
        case FFCZ_SLAB_GATE: {
            reset_ctl();
            const long long ws = (N + 31) / 32, wf = (Nc + 31) / 32;
            k_gate_spatial<<<grid_for(N), 256, 0, st>>>(dd(0), N, sb, op->m, dd(2), ww(4), ww(5), c.ctl);
            k_gate_freq<<<grid_for(Nc), 256, 0, st>>>(d2(1), hg, fb, op->m, d2(3), ww(6), ww(7), c.ctl);
            FFCZ_LAUNCH_CHECK();
            auto codes = [&](const unsigned* words, long long nwords, const char* name,
                             auto launch) {
                const long long nblk = std::max<long long>(1, (nwords + 1023) / 1024);
                unsigned long long* cnt = c.b<unsigned long long>(name, nblk + 1);
                k_popc_blocks<<<static_cast<unsigned>(nblk), 1024, 0, st>>>(words, nwords, cnt);
                k_scan_blocks<<<1, 1024, 0, st>>>(cnt, nblk, &c.ctl->count_a);
                launch(static_cast<unsigned>(nblk), cnt);
                FFCZ_LAUNCH_CHECK();
                return c.read_ctl().count_a;
            };
            o4[2] = static_cast<double>(codes(ww(4), ws, "slab_cnt_s", [&](unsigned nb, unsigned long long* off) {
                k_codes_spatial_bits<<<nb, 1024, 0, st>>>(ww(4), ws, off, dd(0), sb, op->m,
                                                          static_cast<int*>(P(8)));
            }));
            o4[3] = static_cast<double>(codes(ww(6), wf, "slab_cnt_f", [&](unsigned nb, unsigned long long* off) {
                k_codes_freq_bits<<<nb, 1024, 0, st>>>(ww(6), wf, off, d2(1), hg, fb, op->m,
                                                       static_cast<int*>(P(9)));
            }));
            const Ctl h = c.read_ctl();
            o4[0] = static_cast<double>(h.act_s);
            o4[1] = static_cast<double>(h.act_f);
            break;
        }
        default:
            throw Error(kValidation, "unknown slab op " + std::to_string(op->op));
        }
        FFCZ_CUDA_CHECK(cudaGetLastError());
        c.launches += launch_ticks() - ticks0;
        if (out) std::memcpy(out, o4, sizeof(o4));
    });
}

uint64_t ffcz_cuda_launch_count(ffcz_cuda_ctx* ctx) { return ctx ? ctx->launches : 0; }

int ffcz_cuda_alternating_projection(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field,
                                     const void* eps0_in, const ffcz_bounds_desc* bw_desc,
                                     uint64_t max_iters, double precondition_slack,
                                     const ffcz_cuda_options* opt_in, double* spatial_edits,
                                     double* frequency_edits, double* final_epsilon,
                                     ffcz_cuda_report* report) {
    return guarded(ctx, [&] {
        if (!field || !eps0_in || !bw_desc || !report) throw Error(kValidation, "null argument");
        ffcz_cuda_options opt;
        ffcz_cuda_default_options(&opt);
        if (opt_in) opt = *opt_in;
        if (max_iters < 1) throw Error(kValidation, "alternating_projection: max_iters must be >= 1");
        const Geometry g = make_geometry(field->ndim, field->dims, kPitchAlign);
        ffcz_cuda_ctx& c = *ctx;
        cudaStream_t st = c.st;
        const bool on_dev = opt.flags & FFCZ_INPUTS_ON_DEVICE;
        const long long N = g.N;
        c.call_flags = opt.flags;
        const Bounds bw = upload_bounds(c, g, *bw_desc, on_dev, !(opt.flags & FFCZ_BOUNDS_VALIDATED));
        double* eps = c.b<double>("eps", N);
        const size_t esz = field->dtype == FFCZ_F32 ? 4 : 8;
        const void* src = eps0_in;
        if (!on_dev) {
            void* d = c.buf("in_eps0", N * esz);
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(d, eps0_in, N * esz, cudaMemcpyHostToDevice, st));
            src = d;
        }
        // eps = eps0 (widened); precondition vs working bounds + slack (projection.cpp:88-94)
        double* zeros = c.b<double>("zeros_in", 1);
        (void)zeros;
        k_ctl_init<<<1, 1, 0, st>>>(c.ctl, max_iters);
        if (field->dtype == FFCZ_F32) {
            float* z = c.b<float>("zero_f", N);
            FFCZ_CUDA_CHECK(cudaMemsetAsync(z, 0, N * sizeof(float), st));
            k_eps0<float><<<grid_for(N), 256, 0, st>>>(z, static_cast<const float*>(src), eps, N,
                                                        bw.sb, 1.0, precondition_slack, 0, c.ctl);
        } else {
            double* z = c.b<double>("zero_d", N);
            FFCZ_CUDA_CHECK(cudaMemsetAsync(z, 0, N * sizeof(double), st));
            k_eps0<double><<<grid_for(N), 256, 0, st>>>(z, static_cast<const double*>(src), eps, N,
                                                         bw.sb, 1.0, precondition_slack, 0, c.ctl);
        }
        FFCZ_LAUNCH_CHECK();
        const Ctl h0 = c.read_ctl();
        if (h0.bad2 != ~0ull)
            throw Error(kValidation, "alternating_projection: epsilon0 violates the spatial bound "
                                     "at index " + std::to_string(h0.bad2));
        double* S = c.b<double>("S", N);
        double2* F = c.b<double2>("F", g.half_elems());
        FFCZ_CUDA_CHECK(cudaEventRecord(c.ev[2], st));
        // F is returned: accumulate it in every clip pass (no gate-side rebuild here)
        const LoopResult lr = run_loop(c, g, eps, bw, 1.0, !(opt.flags & FFCZ_FORCE_UNFUSED), S, F,
                                       false);
        FFCZ_CUDA_CHECK(cudaEventRecord(c.ev[3], st));
        k_residual_s<<<grid_for(N), 256, 0, st>>>(eps, N, bw.sb, 1.0, c.ctl);
        FFCZ_CUDA_CHECK(cudaMemsetAsync(&c.ctl->act_s, 0, 2 * sizeof(unsigned long long), st));
        k_count_spatial<<<grid_for(N), 256, 0, st>>>(S, N, c.ctl);
        k_count_freq<<<grid_for(g.Nc()), 256, 0, st>>>(F, g.hg(), c.ctl);
        FFCZ_LAUNCH_CHECK();
        const Ctl h = c.read_ctl();
        report->iterations = std::max<unsigned long long>(lr.passes, 1);
        report->active_spatial = h.act_s;
        report->active_frequency = h.act_f;
        report->converged = lr.converged;
        report->residual_f = lr.residual_f;
        report->residual_s = bitsd_host(h.res_s_bits);
        report->wall_time_s = event_ms(c.ev[2], c.ev[3]) * 1e-3;
        if (spatial_edits)
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(spatial_edits, S, N * 8, cudaMemcpyDeviceToHost, st));
        if (final_epsilon)
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(final_epsilon, eps, N * 8, cudaMemcpyDeviceToHost, st));
        if (frequency_edits) {
            double2* full = c.b<double2>("full_tmp", N);
            k_expand_full<<<grid_for(N), 256, 0, st>>>(F, full, g.ndim, g.d[0], g.d[1], g.d[2], g.P);
            FFCZ_LAUNCH_CHECK();
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(frequency_edits, full, N * 16, cudaMemcpyDeviceToHost, st));
        }
        c.sync();
    });
}

// ---- device metrics (metrics.cu; metrics.cpp) -------------------------------------------------

int ffcz_cuda_spectrum_bound(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, const void* original,
                             int on_device, double rho, double* delta_out) {
    return guarded(ctx, [&] {
        if (!(rho >= 0.0) || !std::isfinite(rho))
            throw Error(kValidation, "spectrum_bound_to_freq_bounds: rho must be >= 0");
        const Geometry g = make_geometry(field->ndim, field->dims, kPitchAlign);
        ffcz_cuda_ctx& c = *ctx;
        const double* x = metric_field(c, "m_x", g, field->dtype, original, on_device);
        double2* X = c.b<double2>("m_half", g.half_elems());
        FftPlan<double>{g, &c.tw64}.r2c(x, X, nullptr, c.st);
        SpecStats* ss = fresh_spec_stats(c);
        k_spec_sums<<<grid_for(g.Nc()), 256, 0, c.st>>>(X, nullptr, nullptr, g.hg(), ss);
        FFCZ_LAUNCH_CHECK();
        const double max_mag = bits_to_d(read_stats(c, ss).max_abs_X);
        const double floor_v = std::max(1e-12 * max_mag, 1e-300);
        const double scale = (std::sqrt(1.0 + rho) - 1.0) / std::sqrt(2.0);
        double* out = on_device ? delta_out : c.b<double>("m_delta", g.N);
        k_spectrum_bound<<<grid_for(g.Nc()), 256, 0, c.st>>>(X, g.d[0], g.d[1], g.n2, g.P, scale,
                                                            floor_v, out);
        FFCZ_LAUNCH_CHECK();
        if (!on_device)
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(delta_out, out, g.N * 8, cudaMemcpyDeviceToHost, c.st));
        c.sync();
    });
}

int ffcz_cuda_metrics(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, const void* original,
                      const void* reconstructed, int on_device, ffcz_cuda_metrics_out* out) {
    return guarded(ctx, [&] {
        if (!out) throw Error(kValidation, "null metrics output");
        const Geometry g = make_geometry(field->ndim, field->dims, kPitchAlign);
        ffcz_cuda_ctx& c = *ctx;
        cudaStream_t st = c.st;
        const double* x = metric_field(c, "m_x", g, field->dtype, original, on_device);
        const double* y = metric_field(c, "m_y", g, field->dtype, reconstructed, on_device);
        double* e = c.b<double>("m_eps", g.N);
        FieldStats* fs = fresh_field_stats(c);
        k_field_stats<double><<<grid_for(g.N), 256, 0, st>>>(x, y, g.N, e, fs);
        FFCZ_LAUNCH_CHECK();
        FftPlan<double> plan{g, &c.tw64};
        double2* X = c.b<double2>("m_half", g.half_elems());
        double2* Y = c.b<double2>("m_half2", g.half_elems());
        double2* D = c.b<double2>("m_half3", g.half_elems());
        plan.r2c(x, X, nullptr, st);
        plan.r2c(y, Y, nullptr, st);
        plan.r2c(e, D, nullptr, st);
        SpecStats* ss = fresh_spec_stats(c);
        k_spec_sums<<<grid_for(g.Nc()), 256, 0, st>>>(X, Y, D, g.hg(), ss);
        FFCZ_LAUNCH_CHECK();
        const FieldStats hf = read_stats(c, fs);
        const SpecStats hs = read_stats(c, ss);
        const double inf = std::numeric_limits<double>::infinity();
        out->max_spatial = bits_to_d(hf.max_abs_eps);
        // psnr (metrics.cpp:64-79): zero error wins over a zero range
        const double se = hf.sum[0];
        if (se == 0.0) {
            out->psnr_db = inf;
        } else {
            const double lo = ord_bits_decode(hf.lo), hi = ord_bits_decode(hf.hi);
            if (hi == lo) throw Error(kUndefined, "psnr: constant original has no defined range");
            out->psnr_db = 20.0 * std::log10((hi - lo) / std::sqrt(se / static_cast<double>(g.N)));
        }
        // ssnr (metrics.cpp:81-93)
        if (hs.sum[0] == 0.0) throw Error(kUndefined, "ssnr: zero-energy original spectrum");
        out->ssnr_db = hs.sum[1] == 0.0 ? inf : 10.0 * std::log10(hs.sum[0] / hs.sum[1]);
        // max over rfe (metrics.cpp:95-105)
        const double mx = bits_to_d(hs.max_abs_X);
        if (mx == 0.0) throw Error(kUndefined, "rfe: all-zero original spectrum");
        out->max_rfe = bits_to_d(hs.max_abs_D) / mx;
    });
}

int ffcz_cuda_power_spectrum(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, const void* x_in,
                             int on_device, uint64_t capacity, double* power, uint64_t* counts,
                             uint64_t* nbins_out, double* mean_out, int* mean_fallback_out) {
    return guarded(ctx, [&] {
        const Geometry g = make_geometry(field->ndim, field->dims, kPitchAlign);
        double r2 = 0.0;
        for (int a = 0; a < 3; ++a) {
            const double cc = static_cast<double>(g.d[a] / 2);
            r2 += cc * cc;
        }
        const uint64_t nbins = static_cast<uint64_t>(std::llround(std::sqrt(r2))) + 1;
        if (nbins_out) *nbins_out = nbins;
        if (!power) return;  // size query
        if (capacity < nbins || !counts)
            throw Error(kValidation, "power_spectrum: output capacity " + std::to_string(capacity) +
                                         " < " + std::to_string(nbins) + " bins");
        ffcz_cuda_ctx& c = *ctx;
        cudaStream_t st = c.st;
        const double* x = metric_field(c, "m_x", g, field->dtype, x_in, on_device);
        FieldStats* fs = fresh_field_stats(c);
        k_field_stats<double><<<grid_for(g.N), 256, 0, st>>>(x, nullptr, g.N, nullptr, fs);
        FFCZ_LAUNCH_CHECK();
        const FieldStats hf = read_stats(c, fs);
        const double mean = hf.sum[1] / static_cast<double>(g.N);
        const double max_abs = bits_to_d(hf.max_abs_x);
        const bool fallback = std::abs(mean) <= 1e-12 * max_abs;  // metrics.cpp:21-24
        double* fl = c.b<double>("m_eps", g.N);
        k_fluct<double><<<grid_for(g.N), 256, 0, st>>>(x, g.N, mean, fallback ? 1 : 0, fl);
        FFCZ_LAUNCH_CHECK();
        double2* X = c.b<double2>("m_half", g.half_elems());
        FftPlan<double>{g, &c.tw64}.r2c(fl, X, nullptr, st);
        double* dp = c.b<double>("m_power", nbins);
        unsigned long long* dc = c.b<unsigned long long>("m_counts", nbins);
        FFCZ_CUDA_CHECK(cudaMemsetAsync(dp, 0, nbins * 8, st));
        FFCZ_CUDA_CHECK(cudaMemsetAsync(dc, 0, nbins * 8, st));
        const int nb = static_cast<int>(nbins);
        const size_t smem = nbins <= static_cast<uint64_t>(kShellSmemBins) ? nbins * 16 : 0;
        k_shell_power<<<grid_for(g.Nc()), 256, smem, st>>>(X, g.d[0], g.d[1], g.n2, g.P, nb, dp, dc);
        FFCZ_LAUNCH_CHECK();
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(power, dp, nbins * 8, cudaMemcpyDeviceToHost, st));
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(counts, dc, nbins * 8, cudaMemcpyDeviceToHost, st));
        c.sync();
        if (mean_out) *mean_out = mean;
        if (mean_fallback_out) *mean_fallback_out = fallback ? 1 : 0;
    });
}

int ffcz_cuda_forward_dft(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, const double* x,
                          double* spectrum_out) {
    return guarded(ctx, [&] {
        const Geometry g = make_geometry(field->ndim, field->dims, kPitchAlign);
        ffcz_cuda_ctx& c = *ctx;
        double* dx = c.b<double>("fx", g.N);
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(dx, x, g.N * 8, cudaMemcpyHostToDevice, c.st));
        double2* half = c.b<double2>("fhalf", g.half_elems());
        FftPlan<double> plan{g, &c.tw64};
        plan.r2c(dx, half, nullptr, c.st);
        double2* full = c.b<double2>("full_tmp", g.N);
        k_expand_full<<<grid_for(g.N), 256, 0, c.st>>>(half, full, g.ndim, g.d[0], g.d[1], g.d[2], g.P);
        FFCZ_LAUNCH_CHECK();
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(spectrum_out, full, g.N * 16, cudaMemcpyDeviceToHost, c.st));
        c.sync();
    });
}

int ffcz_cuda_inverse_dft(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, const double* spectrum,
                          int out_precision, double* x_out) {
    return guarded(ctx, [&] {
        const Geometry g = make_geometry(field->ndim, field->dims, kPitchAlign);
        ffcz_cuda_ctx& c = *ctx;
        cudaStream_t st = c.st;
        double2* full = c.b<double2>("full_tmp", g.N);
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(full, spectrum, g.N * 16, cudaMemcpyHostToDevice, st));
        double2* Hh = c.b<double2>("fhalf", g.half_elems());
        double2* Ah = c.b<double2>("fhalf2", g.half_elems());
        k_split_hermitian<<<grid_for(g.Nc()), 256, 0, st>>>(full, Hh, Ah, g.hg(), g.d[0], g.d[1]);
        FFCZ_LAUNCH_CHECK();
        double* re = c.b<double>("fx", g.N);
        double* im = c.b<double>("fx2", g.N);
        FftPlan<double> plan{g, &c.tw64};
        const double invN = 1.0 / static_cast<double>(g.N);
        plan.c2r(Hh, Hh, re, invN, nullptr, st);
        plan.c2r(Ah, Ah, im, invN, nullptr, st);
        FFCZ_CUDA_CHECK(cudaMemsetAsync(&c.ctl->vs_bits, 0, 2 * sizeof(unsigned long long), st));
        k_maxabs<<<grid_for(g.N), 256, 0, st>>>(re, g.N, &c.ctl->vs_bits);
        k_maxabs<<<grid_for(g.N), 256, 0, st>>>(im, g.N, &c.ctl->vf_bits);
        FFCZ_LAUNCH_CHECK();
        const Ctl h = c.read_ctl();
        const double max_re = bitsd_host(h.vs_bits), max_im = bitsd_host(h.vf_bits);
        // transform.cpp:64-80
        const double tol = (out_precision == FFCZ_PRECISION_F32 ? 1e-6 : 1e-10) * std::max(max_re, 1e-300);
        if (max_im > tol)
            throw Error(kSymmetry, "inverse_dft: imaginary residue " + std::to_string(max_im) +
                                       " exceeds tolerance (non-Hermitian input?)");
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(x_out, re, g.N * 8, cudaMemcpyDeviceToHost, st));
        c.sync();
    });
}

int ffcz_cuda_r2c_device(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, const void* x_dev,
                         void* half_dev) {
    return guarded(ctx, [&] {
        const Geometry g = make_geometry(field->ndim, field->dims, kPitchAlign);
        if (field->dtype == FFCZ_F32)
            r2c_dev<float>(*ctx, ctx->tw32, g, static_cast<const float*>(x_dev), static_cast<float2*>(half_dev));
        else
            r2c_dev<double>(*ctx, ctx->tw64, g, static_cast<const double*>(x_dev), static_cast<double2*>(half_dev));
    });
}

int ffcz_cuda_c2r_device(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, const void* half_dev,
                         void* x_dev) {
    return guarded(ctx, [&] {
        const Geometry g = make_geometry(field->ndim, field->dims, kPitchAlign);
        if (field->dtype == FFCZ_F32)
            c2r_dev<float>(*ctx, ctx->tw32, g, static_cast<const float2*>(half_dev), static_cast<float*>(x_dev));
        else
            c2r_dev<double>(*ctx, ctx->tw64, g, static_cast<const double2*>(half_dev), static_cast<double*>(x_dev));
    });
}

uint32_t ffcz_cuda_crc32c(const uint8_t* data, size_t len) { return ffcz_host::crc32c(data, len); }

int ffcz_cuda_huffman_encode(ffcz_cuda_ctx* ctx, const int32_t* codes, uint64_t n, uint8_t* out,
                             uint64_t cap, uint64_t* len) {
    return guarded(ctx, [&] {
        if ((!codes && n) || !len) throw Error(kValidation, "null argument");
        ffcz_cuda_ctx& c = *ctx;
        int* d = c.b<int>("he_codes", std::max<uint64_t>(n, 1));
        if (n) FFCZ_CUDA_CHECK(cudaMemcpyAsync(d, codes, 4 * n, cudaMemcpyHostToDevice, c.st));
        DevScratch ds{c.st, [&](const char* nm, size_t b) { return c.buf(nm, b); }};
        unsigned char* dp = nullptr;
        const unsigned long long l = huffman_encode_device(ds, d, n, &dp);
        *len = l;
        if (out && cap >= l)
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(out, dp, l, cudaMemcpyDeviceToHost, c.st));
        c.sync();
        if (out && cap < l) throw Error(kValidation, "output buffer too small");
    });
}

int ffcz_cuda_outer_compress(ffcz_cuda_ctx* ctx, const uint8_t* data, uint64_t n, uint8_t* out,
                             uint64_t cap, uint64_t* len) {
    return guarded(ctx, [&] {
        if ((!data && n) || !len) throw Error(kValidation, "null argument");
        ffcz_cuda_ctx& c = *ctx;
        auto* d = c.b<unsigned char>("oc_in", std::max<uint64_t>(n, 1));
        if (n) FFCZ_CUDA_CHECK(cudaMemcpyAsync(d, data, n, cudaMemcpyHostToDevice, c.st));
        DevScratch ds{c.st, [&](const char* nm, size_t b) { return c.buf(nm, b); }};
        auto* dl = c.b<unsigned long long>("oc_len", 1);
        unsigned char* dp = nullptr;
        deflate_device(ds, "oc_out", d, n, &dp, dl);
        unsigned long long l = 0;
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(&l, dl, 8, cudaMemcpyDeviceToHost, c.st));
        c.sync();
        *len = l;
        if (out && cap < l) throw Error(kValidation, "output buffer too small");
        if (out) {
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(out, dp, l, cudaMemcpyDeviceToHost, c.st));
            c.sync();
        }
    });
}

int ffcz_cuda_crc32c_device(ffcz_cuda_ctx* ctx, const uint8_t* data, uint64_t n, int on_device,
                            uint32_t* crc) {
    return guarded(ctx, [&] {
        if ((!data && n) || !crc) throw Error(kValidation, "null argument");
        ffcz_cuda_ctx& c = *ctx;
        const unsigned char* d = data;
        if (!on_device && n) {
            auto* t = c.b<unsigned char>("crc_in", n);
            FFCZ_CUDA_CHECK(cudaMemcpyAsync(t, data, n, cudaMemcpyHostToDevice, c.st));
            d = t;
        }
        auto* acc = c.b<unsigned>("crc_acc", 1);
        FFCZ_CUDA_CHECK(cudaMemsetAsync(acc, 0, 4, c.st));
        crc32c_raw_device(c.st, d, n, acc);
        unsigned raw = 0;
        FFCZ_CUDA_CHECK(cudaMemcpyAsync(&raw, acc, 4, cudaMemcpyDeviceToHost, c.st));
        c.sync();
        *crc = ffcz_host::crc32c_from_raw(raw, n);
    });
}

int ffcz_cuda_profile_enable(ffcz_cuda_ctx* ctx, int enable) {
    return guarded(ctx, [&] {
        std::vector<ffcz_cuda_ctx*> all{ctx};
        all.insert(all.end(), ctx->lanes.begin(), ctx->lanes.end());
        for (ffcz_cuda_ctx* c : all) {
            if (enable) {
                c->sync();
                c->prof.clear();
                c->ev_used = 0;
            }
            c->prof_on = enable != 0;
        }
    });
}

int ffcz_cuda_profile_read(ffcz_cuda_ctx* ctx, ffcz_cuda_kernel_stat* out, int max, int* n) {
    return guarded(ctx, [&] {
        ctx->sync();
        ffcz_cuda_kernel_stat st[kNumProf];
        std::memset(st, 0, sizeof(st));
        for (int k = 0; k < kNumProf; ++k)
            std::strncpy(st[k].name, kProfNames[k], sizeof(st[k].name) - 1);
        // launches that returned at the convergence gate run for a small fraction of a real
        // pass: anything under 20% of the longest launch of the same class and byte count
        // records of the context and of its batch lanes
        std::vector<ffcz_cuda_ctx::ProfRec> recs = ctx->prof;
        for (ffcz_cuda_ctx* l : ctx->lanes) {
            l->sync();
            recs.insert(recs.end(), l->prof.begin(), l->prof.end());
        }
        std::vector<float> dur(recs.size());
        std::map<std::pair<int, double>, float> longest;
        for (size_t i = 0; i < recs.size(); ++i) {
            const auto& r = recs[i];
            FFCZ_CUDA_CHECK(cudaEventElapsedTime(&dur[i], r.a, r.b));
            float& l = longest[{r.cls, r.bytes}];
            l = std::max(l, dur[i]);
        }
        for (size_t i = 0; i < recs.size(); ++i) {
            const auto& r = recs[i];
            if (dur[i] < 0.2f * longest[{r.cls, r.bytes}]) {
                ++st[r.cls].gated;
                continue;
            }
            ++st[r.cls].launches;
            st[r.cls].total_ms += dur[i];
            st[r.cls].bytes += r.bytes;
        }
        int k = 0;
        for (; k < kNumProf && k < max; ++k) out[k] = st[k];
        *n = k;
    });
}

// Per-pass micro-benchmark (tools/passbench.py): every pass kind of the engine on a field of the
// given geometry and dtype, `reps` back-to-back launches each, CUDA-event timed.
int ffcz_cuda_bench_passes(ffcz_cuda_ctx* ctx, const ffcz_field_desc* field, int reps,
                           ffcz_cuda_kernel_stat* out, int max, int* n) {
    return guarded(ctx, [&] {
        const Geometry g = make_geometry(field->ndim, field->dims, kPitchAlign);
        ffcz_cuda_ctx& c = *ctx;
        cudaStream_t st = c.st;
        int k = 0;
        auto timed = [&](const char* name, double bytes, auto&& launch) {
            launch();  // warm (tables, attributes)
            FFCZ_CUDA_CHECK(cudaEventRecord(c.ev[0], st));
            for (int r = 0; r < reps; ++r) launch();
            FFCZ_CUDA_CHECK(cudaEventRecord(c.ev[1], st));
            FFCZ_CUDA_CHECK(cudaEventSynchronize(c.ev[1]));
            if (k < max) {
                std::memset(&out[k], 0, sizeof(out[k]));
                std::strncpy(out[k].name, name, sizeof(out[k].name) - 1);
                out[k].launches = reps;
                out[k].total_ms = event_ms(c.ev[0], c.ev[1]);
                out[k].bytes = bytes * reps;
                ++k;
            }
        };
        const double Nc = static_cast<double>(g.Nc()), N = static_cast<double>(g.N);
        if (field->dtype == FFCZ_F64) {
            double* x = c.b<double>("pb_x", g.N);
            double* S = c.b<double>("pb_S", g.N);
            double2* h = c.b<double2>("pb_h", g.half_elems());
            double2* F = c.b<double2>("pb_F", g.half_elems());
            FFCZ_CUDA_CHECK(cudaMemsetAsync(x, 0x3f, g.N * 8, st));
            FFCZ_CUDA_CHECK(cudaMemsetAsync(S, 0, g.N * 8, st));
            FFCZ_CUDA_CHECK(cudaMemsetAsync(F, 0, g.half_elems() * 16, st));
            FftPlan<double> plan{g, &c.tw64};
            Bounds b;
            b.sb.g = 0.25;
            b.fb.g = 1e-3;
            k_ctl_init<<<1, 1, 0, st>>>(c.ctl, 1000);
            timed("row_r2c", 8 * N + 16 * Nc, [&] {
                launch_row_r2c<double>(g.n2, x, g.n2, h, g.P, g.rows, c.tw64, nullptr, st); });
            timed("row_c2r", 8 * N + 16 * Nc, [&] {
                launch_row_c2r<double>(g.n2, h, g.P, x, g.n2, g.rows, 1.0, c.tw64, nullptr, st); });
            launch_row_r2c<double>(g.n2, x, g.n2, h, g.P, g.rows, c.tw64, nullptr, st);
            if (plan.fused_ok())
                timed("row_c2r_sclip_r2c (K1)", 32 * Nc + 8 * N, [&] {
                    launch_row_fused<double>(g.n2, h, g.P, g.rows, g.n2, 1.0 / N, c.tw64, nullptr,
                                             HookSClip<double>{b.sb, 1.0, S, x}, st); });
            for (int a : {1, 0}) {
                if (g.d[a] == 1) continue;
                const std::string ax = a == 1 ? "axis_mid" : "axis_first";
                timed(("col_fwd " + ax).c_str(), 32 * Nc, [&] {
                    plan.col(a, -1, h, h, nullptr, HookNone{}, st); });
                timed(("col_inv " + ax).c_str(), 32 * Nc, [&] {
                    plan.col(a, +1, h, h, nullptr, HookNone{}, st); });
            }
            const int za = complete_axis(g.d[0] > 1, true);
            if (g.d[za] > 1 && plan.fused_ok()) {
                timed("K3a col_fwd_check", 32 * Nc, [&] {
                    plan.col(za, -1, h, h, nullptr, HookFReduce{b.fb, 1.0, c.ctl}, st); });
                timed("K3b col_clip_inv (F rmw)", 64 * Nc, [&] {
                    plan.col(za, +1, h, h, nullptr, HookFClip<double>{b.fb, 1.0, F}, st); });
            }
        } else {
            float* x = c.b<float>("pb_x32", g.N);
            float2* h = c.b<float2>("pb_h32", g.half_elems());
            FFCZ_CUDA_CHECK(cudaMemsetAsync(x, 0x3f, g.N * 4, st));
            FftPlan<float> plan{g, &c.tw32};
            timed("f32 row_r2c", 4 * N + 8 * Nc, [&] {
                launch_row_r2c<float>(g.n2, x, g.n2, h, g.P, g.rows, c.tw32, nullptr, st); });
            timed("f32 row_c2r", 4 * N + 8 * Nc, [&] {
                launch_row_c2r<float>(g.n2, h, g.P, x, g.n2, g.rows, 1.0f, c.tw32, nullptr, st); });
            for (int a : {1, 0}) {
                if (g.d[a] == 1) continue;
                const std::string ax = a == 1 ? "axis_mid" : "axis_first";
                timed(("f32 col_fwd " + ax).c_str(), 16 * Nc, [&] {
                    plan.col(a, -1, h, h, nullptr, HookNone{}, st); });
            }
        }
        *n = k;
    });
}

} // extern "C"
