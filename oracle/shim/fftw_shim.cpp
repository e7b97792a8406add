// FFTW3-API provider for the CPU reference build (oracle/_ref).  TEST INFRASTRUCTURE ONLY.
//
// Implements the three FFTW entry points the reference uses
// (/root/reference/proj/core/src/transform.cpp:20-41): an N-d complex<double> DFT,
// unnormalised, sign -1 forward / +1 backward, row-major extents, out-of-place,
// input preserved.  Separable: one 1-D transform per axis over every line.
// Power-of-two lines use an iterative radix-2 FFT with per-index twiddles
// (no recurrences); other lengths use Bluestein's chirp-z through a power-of-two
// FFT with exact (k^2 mod 2n) chirp phases, which keeps errors at ~1e-15 of the
// peak (the reference's own test bound is 1e-9, proj/tests/test_transform.cpp:25-33).
//
// FFCZ_SHIM_THREADS=<k> (default 1) splits the lines of each axis across k
// threads; the reference itself is single-threaded, so the
// default reproduces it and k>1 is the "FFT-threaded" CPU figure.

#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

namespace {

using cd = std::complex<double>;

bool is_pow2(std::size_t n) { return n && !(n & (n - 1)); }

struct Radix2 {
    std::size_t n = 0;
    int logn = 0;
    std::vector<cd> tw;            // exp(sign*2*pi*i*k/n), k < n/2
    std::vector<std::uint32_t> rev;

    void init(std::size_t n_, int sign) {
        n = n_;
        logn = 0;
        while ((std::size_t(1) << logn) < n) ++logn;
        tw.resize(n / 2);
        for (std::size_t k = 0; k < n / 2; ++k) {
            double a = 2.0 * M_PI * double(k) / double(n);
            tw[k] = cd(std::cos(a), sign * std::sin(a));
        }
        rev.resize(n);
        for (std::size_t i = 0; i < n; ++i) {
            std::uint32_t r = 0;
            for (int b = 0; b < logn; ++b)
                if (i & (std::size_t(1) << b)) r |= 1u << (logn - 1 - b);
            rev[i] = r;
        }
    }

    void run(cd* a) const {
        for (std::size_t i = 0; i < n; ++i)
            if (i < rev[i]) std::swap(a[i], a[rev[i]]);
        for (std::size_t len = 2; len <= n; len <<= 1) {
            std::size_t half = len / 2, step = n / len;
            for (std::size_t s = 0; s < n; s += len) {
                for (std::size_t j = 0; j < half; ++j) {
                    cd w = tw[j * step];
                    cd u = a[s + j], v = a[s + j + half] * w;
                    a[s + j] = u + v;
                    a[s + j + half] = u - v;
                }
            }
        }
    }
};

struct Line1D {
    std::size_t n = 0;
    int sign = -1;
    bool pow2 = true;
    Radix2 fft;         // pow2: length n; Bluestein: length m, sign -1
    Radix2 ifft;        // Bluestein inverse, sign +1
    std::vector<cd> chirp, bhat;

    void init(std::size_t n_, int sign_) {
        n = n_;
        sign = sign_;
        pow2 = is_pow2(n);
        if (pow2) {
            fft.init(n, sign);
            return;
        }
        std::size_t m = 1;
        while (m < 2 * n - 1) m <<= 1;
        fft.init(m, -1);
        ifft.init(m, +1);
        chirp.resize(n);
        for (std::size_t k = 0; k < n; ++k) {
            std::size_t k2 = (k * k) % (2 * n);
            double a = M_PI * double(k2) / double(n);
            chirp[k] = cd(std::cos(a), sign * std::sin(a));
        }
        bhat.assign(m, cd(0, 0));
        bhat[0] = std::conj(chirp[0]);
        for (std::size_t k = 1; k < n; ++k) bhat[k] = bhat[m - k] = std::conj(chirp[k]);
        fft.run(bhat.data());
    }

    // in-place on a contiguous line; work must hold fft.n entries
    void run(cd* x, cd* work) const {
        if (n == 1) return;
        if (pow2) {
            fft.run(x);
            return;
        }
        std::size_t m = fft.n;
        for (std::size_t k = 0; k < n; ++k) work[k] = x[k] * chirp[k];
        for (std::size_t k = n; k < m; ++k) work[k] = cd(0, 0);
        fft.run(work);
        for (std::size_t k = 0; k < m; ++k) work[k] *= bhat[k];
        ifft.run(work);
        const double inv = 1.0 / double(m);
        for (std::size_t k = 0; k < n; ++k) x[k] = work[k] * inv * chirp[k];
    }
};

int shim_threads() {
    const char* s = std::getenv("FFCZ_SHIM_THREADS");
    int k = s ? std::atoi(s) : 1;
    return k < 1 ? 1 : k;
}

} // namespace

struct ffcz_shim_plan_s {
    std::vector<std::size_t> dims;
    cd* in;
    cd* out;
    std::vector<Line1D> axes;
};

extern "C" fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out,
                                   int sign, unsigned /*flags*/) {
    auto* p = new ffcz_shim_plan_s;
    p->dims.assign(n, n + rank);
    p->in = reinterpret_cast<cd*>(in);
    p->out = reinterpret_cast<cd*>(out);
    p->axes.resize(rank);
    for (int a = 0; a < rank; ++a) p->axes[a].init(std::size_t(n[a]), sign);
    return p;
}

extern "C" void fftw_execute(const fftw_plan p) {
    std::size_t total = 1;
    for (auto d : p->dims) total *= d;
    if (p->out != p->in) std::memcpy(p->out, p->in, total * sizeof(cd));
    const int nthreads = shim_threads();
    for (std::size_t a = 0; a < p->dims.size(); ++a) {
        const std::size_t len = p->dims[a];
        std::size_t stride = 1;
        for (std::size_t b = a + 1; b < p->dims.size(); ++b) stride *= p->dims[b];
        const std::size_t lines = total / len;
        const Line1D& plan = p->axes[a];
        auto work_range = [&](std::size_t l0, std::size_t l1) {
            std::vector<cd> line(len), work(plan.pow2 ? 0 : plan.fft.n);
            for (std::size_t l = l0; l < l1; ++l) {
                std::size_t outer = l / stride, inner = l % stride;
                cd* base = p->out + outer * len * stride + inner;
                for (std::size_t i = 0; i < len; ++i) line[i] = base[i * stride];
                plan.run(line.data(), work.data());
                for (std::size_t i = 0; i < len; ++i) base[i * stride] = line[i];
            }
        };
        if (nthreads == 1 || lines < 64) {
            work_range(0, lines);
        } else {
            std::vector<std::thread> pool;
            std::size_t chunk = (lines + nthreads - 1) / nthreads;
            for (int t = 0; t < nthreads; ++t) {
                std::size_t l0 = t * chunk, l1 = std::min(lines, l0 + chunk);
                if (l0 < l1) pool.emplace_back(work_range, l0, l1);
            }
            for (auto& th : pool) th.join();
        }
    }
}

extern "C" void fftw_destroy_plan(fftw_plan p) { delete p; }
